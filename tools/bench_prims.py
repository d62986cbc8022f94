"""Latency of the small dense primitives behind the Tucker mode bases:
one-CTA Jacobi (eigh_dev, b <= 96), bt_syevx (leading pairs), bt_syevd
(full spectrum), CholeskyQR2, SVQB, engine GEMMs, Cholesky."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import _linalg as L, decomp


def tm(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def spd(n, decay=True, seed=0):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-np.linspace(0, 12, n)) if decay else rng.uniform(0.5, 1.0, n)
    a = (q * lam) @ q.T
    return torch.from_numpy((a + a.T) / 2).cuda()


for b in (16, 32, 48, 64, 80, 96):
    a = spd(b)
    near = torch.diag(torch.linspace(1, 2, b, dtype=torch.float64, device="cuda")) + 1e-6 * spd(b, False)
    print(f"jacobi b={b:3d}: random {tm(lambda: L.eigh_dev(a)):7.3f} ms   near-diag {tm(lambda: L.eigh_dev(near)):7.3f} ms")
for n in (128, 192, 256):
    a = spd(n)
    print(f"syevd n={n}: {tm(lambda: L.eigh_dev(a), 2):8.3f} ms")
for n, k in ((512, 32), (1024, 64), (1024, 80), (2047, 400), (2047, 96)):
    a = spd(n)
    print(f"syevx n={n} nvec={k}: {tm(lambda: L.eigh_dev(a, nvec=k, tau=1e-6), 2):8.3f} ms")
for m, k in ((1024, 80), (2047, 96), (512, 48)):
    y = torch.randn(m, k, dtype=torch.float64, device="cuda")
    g = spd(m)
    print(f"m={m} k={k}: qr_thin {tm(lambda: L.qr_thin_dev(y)):7.3f}  "
          f"gemm GQ {tm(lambda: L.gemm_dev(g, y)):7.3f}  gemm YtY {tm(lambda: L.gemm_dev(y, y, ta=True)):7.3f} ms")
for n in (48, 80, 96):
    a = spd(n, False)
    print(f"cholesky n={n}: {tm(lambda: decomp.cholesky(a)):7.3f} ms")
