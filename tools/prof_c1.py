"""C1 CP-ALS (32^3, R=8, 50 sweeps) timing: wall vs in-library phase events."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import configs, decomp, _dev
import paper_2105_01170_b200 as bt

pat, a = configs.c1_matrix()
t = bt.mat_to_tensor(a, pat)
init = configs.normal_init((32, 32, 32), 8, 0)
f0 = [torch.from_numpy(v).cuda() for v in init]
xd = t if torch.is_tensor(t) else torch.from_numpy(t).cuda()
for rep in range(3):
    f = [v.clone() for v in f0]
    lam = _dev.empty((8,))
    pm = [0.0] * 4
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hist, n, conv = decomp.cp_als_device(xd, 8, f, lam, 50, 0.0, "auto", 0.0, phase_ms=pm)
    torch.cuda.synchronize()
    print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms, phases {[round(v, 2) for v in pm]}, fit {hist[-1]}")
    f = [v.clone() for v in f0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hist, n, conv = decomp.cp_als_device(xd, 8, f, lam, 50, 0.0, "auto", 0.0)
    torch.cuda.synchronize()
    print(f"  no phase events (graph replay unless BT_CP_GRAPH=0): wall {1e3 * (time.perf_counter() - t0):.2f} ms, fit {hist[-1]}")
