"""C3 ST-HOSVD and +5 HOOI timings (median of 5, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp

pat, t = configs.c3_build()
def timed(fn, reps=5):
    fn(); ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); out = fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2], out
a, rep = timed(lambda: decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3)))
b, _ = timed(lambda: decomp.hooi(t, rep, 5, shared=(1, 3)))
print(f"c3 st_hosvd {a:.2f} ms, 5 hooi {b:.2f} ms, BT_RR_ROUGH={os.environ.get('BT_RR_ROUGH')}")
