"""Host-side profile of one C3 HOOI sweep (where the idle ~2 ms per sweep goes)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp
pat, t = configs.c3_build()
rep = decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3))
decomp.hooi(t, rep, 1, shared=(1, 3)); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    decomp.hooi(t, rep, 1, shared=(1, 3))
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
