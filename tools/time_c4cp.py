"""C4 CP-ALS (255^3, R=16, 30 sweeps) timing, repeated (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp, multilevel

x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init = configs.normal_init((255, 255, 255), 16, 2)
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
for rep in range(6):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = decomp.cp_als(x3, 16, 30, 0.0)
    e1.record()
    torch.cuda.synchronize()
    print(f"c4 cp_als: {e0.elapsed_time(e1):.2f} ms  fit {res.fit:.12f}")
