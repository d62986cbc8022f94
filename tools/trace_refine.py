"""Kernel sequence of one warm basis refinement (C3 HOOI V-step shape:
y (64, 512, 64), mode 2, r = 32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2105_01170_b200 import _linalg as L

y = torch.randn(64, 512, 64, dtype=torch.float64, device="cuda")
y = y * torch.logspace(0, -12, 512, dtype=torch.float64, device="cuda")[None, :, None]
v0 = L.gaussian_dev(512, 32, 5)
L._refine_basis_qr(y, 2, 32, v0)
torch.cuda.synchronize()
t0 = time.perf_counter()
L._refine_basis_qr(y, 2, 32, v0)
torch.cuda.synchronize()
print(f"refine wall {1e3 * (time.perf_counter() - t0):.2f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    L._refine_basis_qr(y, 2, 32, v0)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  {e.device_time_total:8.1f} us  {e.name[:90]}")
