"""Every kernel of one C3 HOOI sweep inside a time window (ms), in launch order."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2105_01170_b200 import configs, decomp
lo, hi = float(sys.argv[1]), float(sys.argv[2])
pat, t = configs.c3_build()
rep = decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3))
decomp.hooi(t, rep, 1, shared=(1, 3)); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    decomp.hooi(t, rep, 1, shared=(1, 3)); torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = None
for e in ev:
    s = (e.time_range.start - t0) / 1e3
    if lo <= s <= hi:
        gap = 0.0 if prev_end is None else e.time_range.start - prev_end
        print(f"{s:8.3f} ms  {e.device_time_total:7.1f} us  gap {gap:6.1f}  {e.name[:80]}")
    prev_end = e.time_range.end
