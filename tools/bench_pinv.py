"""bt_pinv_sym_f64 timing for small R on identity / diagonal / random SPD."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import _dev
from paper_2105_01170_b200 import _native as N

for R in (8, 16, 64):
    rng = np.random.default_rng(R)
    g = rng.standard_normal((R, 3 * R))
    cases = {"identity": np.eye(R), "diag": np.diag(np.linspace(1, 2, R)), "spd": g @ g.T}
    for dec in (8, 16, 20):
        q, _ = np.linalg.qr(rng.standard_normal((R, R)))
        lam = 10.0 ** (-np.linspace(0, dec, R))
        cases[f"cond1e{dec}"] = (q * lam) @ q.T
    # Hadamard of two nearly collinear Grams (C4-like factors)
    base = rng.standard_normal((255, 1))
    fa = base + 1e-6 * rng.standard_normal((255, R))
    fa /= np.linalg.norm(fa, axis=0)
    ga = fa.T @ fa
    cases["collinear"] = ga * ga
    for name, v in cases.items():
        vd = torch.from_numpy(v).cuda()
        out = torch.empty_like(vd)
        N.call("bt_pinv_sym_f64", _dev.ptr(vd), R, _dev.ptr(out), _dev.stream())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            N.call("bt_pinv_sym_f64", _dev.ptr(vd), R, _dev.ptr(out), _dev.stream())
        e1.record()
        torch.cuda.synchronize()
        v = (v + v.T) / 2
        err = np.abs(out.cpu().numpy() - np.linalg.pinv(v)).max() / np.abs(np.linalg.pinv(v)).max()
        import ctypes
        lib = N.load()
        lib.bt_debug_pinv1s.restype = ctypes.c_int64
        sw, cyc = lib.bt_debug_pinv1s(0), lib.bt_debug_pinv1s(1)
        print(f"R={R:3d} {name:9s} {e0.elapsed_time(e1) * 10:.1f} us/launch  err {err:.1e}  "
              f"(1-sided: {sw} sweeps, {cyc} cycles)")
