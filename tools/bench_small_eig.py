"""Small dense symmetric eigensolvers on one CTA: Jacobi (bt_syevd_f64 small
path) vs tridiagonal + bisection + inverse iteration (bt_syevx_f64, nvec=n)."""
import ctypes as C
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import _linalg as L, _dev
from paper_2105_01170_b200 import _native as N


def syevx_full(ad):
    n = int(ad.shape[0])
    w = _dev.empty((n,)); v = _dev.empty((n, n))
    ws = _dev.workspace(N.load().bt_syevx_ws_bytes(n, n))
    N.call("bt_syevx_f64", _dev.ptr(ad), n, n, -1.0, _dev.ptr(w), _dev.ptr(v), _dev.ptr(ws),
           int(ws.numel()) * 8, _dev.stream())
    return w, v


cases = []
for n in (16, 32, 48, 64, 80, 96, 128):
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-np.linspace(0, 12, n))
    cases.append((n, "graded", (q * lam) @ q.T))
    g = rng.standard_normal((n, n))
    cases.append((n, "wishart", g @ g.T))
    e = np.diag(lam) + 1e-9 * (lambda m: (m + m.T) / 2)(rng.standard_normal((n, n))) * np.sqrt(np.outer(lam, lam))
    cases.append((n, "near_diag", e))
for n, kind, a in cases:
    a = (a + a.T) / 2
    ad = torch.from_numpy(a).cuda()
    row = {"n": n, "kind": kind}
    for name, fn in (("jacobi", lambda: L.eigh_dev(ad) if n <= 96 else None), ("syevx", lambda: syevx_full(ad))):
        r = fn()
        if r is None:
            continue
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            w, v = fn()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / 5
        w, v = w.cpu().numpy(), v.cpu().numpy()
        row[name + "_ms"] = ms
        row[name + "_resid"] = float(np.max(np.abs(a @ v - v * w)))
        row[name + "_orth"] = float(np.max(np.abs(v.T @ v - np.eye(n))))
    print(json.dumps(row), flush=True)
