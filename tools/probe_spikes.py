"""Attribute the slow outliers of single cp_als calls (C1, C4): host wall
time of each sub-step (each followed by a synchronize) over 20 calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp, multilevel, _dev
from paper_2105_01170_b200.tensor import fro_norm_dev
import paper_2105_01170_b200 as bt

x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255).contiguous()
init4 = [torch.from_numpy(f).cuda() for f in configs.normal_init((255, 255, 255), 16, 2)]
pat, a = configs.c1_matrix()
t1 = bt.mat_to_tensor(a, pat)
init1 = [torch.from_numpy(f).cuda() for f in configs.normal_init((32, 32, 32), 8, 0)]


def run(name, xd, init, r, iters, n=20):
    rows = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nt = fro_norm_dev(xd)
        t1_ = time.perf_counter()
        f = [g.clone() for g in init]
        lam = _dev.empty((r,))
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        decomp.cp_als_device(xd, r, f, lam, iters, 0.0, "auto", nt)
        e1.record()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rows.append((round((t1_ - t0) * 1e3, 2), round((t2 - t1_) * 1e3, 2),
                     round((t3 - t2) * 1e3, 2), round(e0.elapsed_time(e1), 2)))
    print(name, "(norm, init, als wall, als events) ms:", rows, flush=True)


for _ in range(2):
    run("c4", x3, init4, 16, 30)
    run("c1", t1, init1, 8, 50)
