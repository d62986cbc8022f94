"""C4-shaped multilevel matvec alone (16 random 3-level terms of 128x128
factors, 32 volumes of 128^3) for timing and ncu (-k regex:bt_gemm)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import multilevel


class T:
    def __init__(self, mats):
        self.level_mats = mats
        self.block = np.ones((1, 1))


g = torch.Generator(device="cuda").manual_seed(0)
terms = [T([torch.randn(128, 128, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)])
         for _ in range(16)]
stacks = multilevel.stack_level_mats(terms)
vols = torch.randn(128 ** 3, 32, dtype=torch.float64, device="cuda", generator=g)
reps = int(os.environ.get("REPS", "3"))
multilevel.ml_matvec(terms, vols, stacks)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    multilevel.ml_matvec(terms, vols, stacks)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / max(reps, 1)
print(f"ml_matvec 32 vols: {ms:.2f} ms, {16 * 32 * 3 * 2 * 128**4 / ms / 1e9:.2f} TFLOP/s")
