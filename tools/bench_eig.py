"""Time + accuracy of the device eigensolver on Gram-like matrices."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import _linalg as L

out = []
for n in (512, 1024, 2047):
    rng = np.random.default_rng(n)
    # fast-decaying spectrum (like the configs' Grams) + a dense random case
    for kind in ("decay", "wishart"):
        if kind == "decay":
            q, _ = np.linalg.qr(rng.standard_normal((n, n)))
            lam = 10.0 ** (-np.linspace(0, 14, n))
            a = (q * lam) @ q.T
        else:
            g = rng.standard_normal((n, n))
            a = g @ g.T
        a = (a + a.T) / 2
        ad = torch.from_numpy(a).cuda()
        L.eigh_dev(ad); torch.cuda.synchronize()
        t0 = time.perf_counter()
        w, v = L.eigh_dev(ad); torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        w, v = w.cpu().numpy(), v.cpu().numpy()
        ref = np.linalg.eigvalsh(a)[::-1]
        out.append({"n": n, "kind": kind, "ms": ms,
                    "eig_err": float(np.max(np.abs(w - ref)) / ref[0]),
                    "orth": float(np.max(np.abs(v.T @ v - np.eye(n)))),
                    "resid": float(np.max(np.abs(a @ v - v * w)) / ref[0])})
        print(json.dumps(out[-1]), flush=True)
