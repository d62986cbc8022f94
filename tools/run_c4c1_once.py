"""One C4 CP-ALS (255^3, R=16, 30 sweeps) and one C1 CP-ALS (32^3, R=8, 50
sweeps) after a warm-up each: the command behind the r02 C4/C1 ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_01170_b200 as bt
from paper_2105_01170_b200 import configs, decomp, multilevel

x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init4 = configs.normal_init((255, 255, 255), 16, 2)
pat, a = configs.c1_matrix()
init1 = configs.normal_init((32, 32, 32), 8, 0)
t1 = bt.mat_to_tensor(a, pat)
t1 = t1 if torch.is_tensor(t1) else torch.from_numpy(t1).cuda()
for rep in range(2):
    decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init4]
    r4 = decomp.cp_als(x3, 16, 30, 0.0)
    decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init1]
    r1 = decomp.cp_als(t1, 8, 50, 0.0)
    torch.cuda.synchronize()
print("c4 fit", r4.fit, "c1 fit", r1.fit)
