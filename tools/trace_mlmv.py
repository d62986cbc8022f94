"""Kernel breakdown of the C4-shaped multilevel matvec (16 terms, 32 volumes of 128^3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2105_01170_b200 import multilevel
class T:
    def __init__(self, mats):
        self.level_mats = mats
        self.block = np.ones((1, 1))
g = torch.Generator(device="cuda").manual_seed(0)
terms = [T([torch.randn(128, 128, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]) for _ in range(16)]
stacks = multilevel.stack_level_mats(terms)
vols = torch.randn(128 ** 3, 32, dtype=torch.float64, device="cuda", generator=g)
multilevel.ml_matvec(terms, vols, stacks); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    multilevel.ml_matvec(terms, vols, stacks); torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA: continue
    c, s = tot.get(e.name[:110], (0, 0.0)); tot[e.name[:110]] = (c + 1, s + e.device_time_total / 1e3)
for k, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:8]:
    print(f"  {s:8.3f} ms  {c:4d}x  {k}")
