"""Where the host time of the C1 cp_als call goes (perf_counter around each step, device idle between)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np, torch
import paper_2105_01170_b200 as bt
from paper_2105_01170_b200 import configs, decomp, _dev, _native as N
from paper_2105_01170_b200.tensor import fro_norm_dev
pat, a = configs.c1_matrix()
init = configs.normal_init((32, 32, 32), 8, 0)
t = bt.mat_to_tensor(a, pat)
td = t if torch.is_tensor(t) else torch.from_numpy(t).cuda()
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
for _ in range(5):
    decomp.cp_als(td, 8, 50, 0.0)
torch.cuda.synchronize()
acc = {}
def lap(name, t0):
    t1 = time.perf_counter(); acc[name] = acc.get(name, 0.0) + (t1 - t0); return t1
REP = 50
for _ in range(REP):
    t0 = time.perf_counter()
    xd = _dev.to_device(td); t0 = lap("to_device", t0)
    nrm = fro_norm_dev(xd); t0 = lap("fro_norm", t0)
    ini = decomp._cp_init(td, 8); t0 = lap("init hook (3 H2D)", t0)
    f = [_dev.to_device(x).clone() for x in ini]; t0 = lap("clones", t0)
    lam = _dev.empty((8,)); t0 = lap("lam", t0)
    res = decomp.cp_als_device(xd, 8, f, lam, 50, 0.0, "auto", nrm); t0 = lap("cp_als_device (C call)", t0)
    rep = [_dev.like_input(td, v) for v in f]; t0 = lap("like_input", t0)
tot = sum(acc.values())
for k, v in acc.items():
    print(f"{k:28s} {1e6 * v / REP:8.1f} us")
print(f"{'total':28s} {1e6 * tot / REP:8.1f} us")
