"""The C2 HOSVD kernel by kernel, in launch order (torch.profiler): the
sequence with durations, to attribute the full-tensor TTMs and the basis
passes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2105_01170_b200 import configs, decomp

pat, t = configs.c2_build(configs.c2_markov())
rep = None
decomp.hosvd(t, [32, 400, 32])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    decomp.hosvd(t, [32, 400, 32])
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    d = e.device_time_total
    if d >= 30:
        print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  {d:8.1f} us  {e.name[:100]}")
print(f"total span {(ev[-1].time_range.end - t0) / 1e3:.2f} ms, kernels {len(ev)}, "
      f"sum {sum(e.device_time_total for e in ev) / 1e3:.2f} ms")
