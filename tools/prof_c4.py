"""C4 CP-ALS (255^3, R=16, 30 sweeps) phase timing + launch list helper."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp, multilevel, _dev

x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255).contiguous()
init = configs.normal_init((255, 255, 255), 16, 2)
f0 = [torch.from_numpy(v).cuda() for v in init]
for rep in range(3):
    f = [v.clone() for v in f0]
    lam = _dev.empty((16,))
    pm = [0.0] * 4
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hist, n, conv = decomp.cp_als_device(x3, 16, f, lam, 30, 0.0, "auto", 0.0, phase_ms=pm)
    torch.cuda.synchronize()
    print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms, phases/sweep {[round(v / 30, 3) for v in pm]}")
    f = [v.clone() for v in f0]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hist, n, conv = decomp.cp_als_device(x3, 16, f, lam, 30, 0.0, "auto", 0.0)
    torch.cuda.synchronize()
    print(f"  graph: wall {1e3 * (time.perf_counter() - t0):.2f} ms")
