"""The C3 ST-HOSVD kernel by kernel (>= 30 us) in launch order (torch.profiler)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2105_01170_b200 import configs, decomp

pat, t = configs.c3_build()
decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3)); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3)); torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
thr = float(sys.argv[1]) if len(sys.argv) > 1 else 30.0
for e in ev:
    d = e.device_time_total
    if d >= thr:
        print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  {d:8.1f} us  {e.name[:100]}")
print(f"total span {(ev[-1].time_range.end - t0) / 1e3:.2f} ms, kernels {len(ev)}, "
      f"sum {sum(e.device_time_total for e in ev) / 1e3:.2f} ms")
