"""Leading-eigenpair solver (tridiagonal path) vs numpy: time + accuracy."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import _linalg as L

for n, nvec in ((200, 20), (512, 64), (1024, 64), (2047, 400), (1024, 1023)):
    rng = np.random.default_rng(n)
    for kind in ("decay", "wishart", "lowrank"):
        if kind == "decay":
            q, _ = np.linalg.qr(rng.standard_normal((n, n)))
            lam = 10.0 ** (-np.linspace(0, 14, n))
            a = (q * lam) @ q.T
        elif kind == "wishart":
            g = rng.standard_normal((n, n))
            a = g @ g.T
        else:
            g = rng.standard_normal((n, 40))
            a = g @ g.T
        a = (a + a.T) / 2
        ad = torch.from_numpy(a).cuda()
        L.eigh_dev(ad, nvec=nvec); torch.cuda.synchronize()
        t0 = time.perf_counter()
        w, v = L.eigh_dev(ad, nvec=nvec); torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        w, v = w.cpu().numpy(), v.cpu().numpy()
        ref = np.linalg.eigvalsh(a)[::-1][:nvec]
        print(json.dumps({"n": n, "nvec": nvec, "kind": kind, "ms": round(ms, 2),
                          "eig_err": float(np.max(np.abs(w - ref)) / ref[0]),
                          "orth": float(np.max(np.abs(v.T @ v - np.eye(nvec)))),
                          "resid": float(np.max(np.abs(a @ v - v * w)) / ref[0])}), flush=True)
