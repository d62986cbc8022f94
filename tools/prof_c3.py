"""Stage timing of the C3 ST-HOSVD (+1 HOOI sweep): mode bases, deflation
passes, Grams, eigensolves, TTMs.  BT_BASIS_DEBUG=1 prints the passes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, _linalg as L, decomp, tensor as T

pat, t = configs.c3_build()
torch.cuda.synchronize()
stats = {}


def wrap(mod, name):
    fn = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        s = stats.setdefault(name, [0, 0.0]); s[0] += 1; s[1] += time.perf_counter() - t0
        return out
    setattr(mod, name, g)


for name in ("unfold_gram_dev", "eigh_dev", "_residual", "_complete", "_orth_normalize", "_axpby", "_leading_subspace", "gemm_dev"):
    wrap(L, name)
wrap(decomp, "ttm_dev")
rep = decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3))
for label, fn in (("st_hosvd", lambda: decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3))),
                  ("hooi_1", lambda: decomp.hooi(t, rep, 1, shared=(1, 3)))):
    stats.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    print(f"== {label} total ms {(time.perf_counter() - t0) * 1e3:.1f}")
    for k, (c, s) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:20s} calls {c:3d} ms {s * 1e3:9.2f}")
