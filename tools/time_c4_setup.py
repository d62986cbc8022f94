"""C4 CP-ALS call overhead: time of 1-, 2- and 30-sweep calls (setup = intercept)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp, multilevel
x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init = configs.normal_init((255, 255, 255), 16, 2)
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
for n in (1, 2, 30, 1, 2, 30):
    ts = []
    for rep in range(7):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); decomp.cp_als(x3, 16, n, 0.0); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{n:2d} sweeps: median {ts[3]:.3f} ms (min {ts[0]:.3f})")
