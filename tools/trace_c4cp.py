"""Kernel breakdown of the C4 CP-ALS (255^3, R=16, 30 sweeps)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2105_01170_b200 import configs, decomp, multilevel

x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init = configs.normal_init((255, 255, 255), 16, 2)
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
fn = lambda: decomp.cp_als(x3, 16, 30, 0.0)
fn(); torch.cuda.synchronize()
t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fn(); torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    k = e.name[:90]
    c, s = tot.get(k, (0, 0.0))
    tot[k] = (c + 1, s + e.device_time_total / 1e3)
print(f"GPU {sum(s for _, s in tot.values()):.2f} ms")
for k, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {s:8.3f} ms  {c:4d}x  {k}")
