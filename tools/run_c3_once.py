"""One C3 ST-HOSVD + 5 HOOI sweeps after a warm-up call (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp

pat, t = configs.c3_build()
rep = decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3))
decomp.hooi(t, rep, 1, shared=(1, 3))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured")
rep = decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3))
h = decomp.hooi(t, rep, 5, shared=(1, 3))
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("core norm ratio", float(torch.linalg.norm(h.core) / torch.linalg.norm(t)))
