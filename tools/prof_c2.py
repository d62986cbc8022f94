"""Stage timing of the C2 HOSVD (mode bases, passes, completion)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import configs, _linalg as L, decomp

params = configs.c2_markov()
pat, t = configs.c2_build(params)
torch.cuda.synchronize()
orig = {name: getattr(L, name) for name in ("unfold_gram_dev", "eigh_dev", "_residual", "_complete", "_orth_normalize", "qr_thin_dev", "_leading_subspace", "gemm_dev")}
stats = {}
def wrap(name, fn):
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        s = stats.setdefault(name, [0, 0.0]); s[0] += 1; s[1] += time.perf_counter() - t0
        return out
    return g
for name, fn in orig.items():
    setattr(L, name, wrap(name, fn))
decomp.hosvd(t, [32, 400, 32])
stats.clear()
torch.cuda.synchronize(); t0 = time.perf_counter()
decomp.hosvd(t, [32, 400, 32])
torch.cuda.synchronize()
print("total ms", (time.perf_counter() - t0) * 1e3)
for k, (c, s) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:20s} calls {c:3d} ms {s * 1e3:9.2f}")
