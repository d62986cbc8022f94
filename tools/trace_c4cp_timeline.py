"""Timeline (start, duration) of the kernels of two C4 CP-ALS sweeps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2105_01170_b200 import configs, decomp, multilevel

x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init = configs.normal_init((255, 255, 255), 16, 2)
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
fn = lambda: decomp.cp_als(x3, 16, 6, 0.0)
fn(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fn(); torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev[-40:]:
    print(f"{e.time_range.start - t0:9.1f} us  +{e.device_time_total:7.1f}  {e.name[:60]}")
