"""C4's R=16 normal matrices V = (G_a o G_b) along the first ALS sweeps (numpy
oracle trajectory): their spectra, and bt_pinv_sym_f64 time / Jacobi sweeps
on each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from scipy.linalg import khatri_rao
from paper_2105_01170_b200 import _dev
from paper_2105_01170_b200 import _native as N
from oracle import configs as oc, port

x = oc.c4_tensor().reshape(255, 255, 255)
f = [v.copy() for v in oc.normal_init((255, 255, 255), 16, 2)]
lib = N.load()
us = [port.unfold(x, k + 1) for k in range(3)]
for sweep in range(3):
    for k in range(3):
        o = [j for j in range(3) if j != k]
        v = (f[o[0]].T @ f[o[0]]) * (f[o[1]].T @ f[o[1]])
        vd = torch.from_numpy(v).cuda()
        out = torch.empty_like(vd)
        N.call("bt_pinv_sym_f64", _dev.ptr(vd), 16, _dev.ptr(out), _dev.stream())
        torch.cuda.synchronize()
        sw = lib.bt_debug_jacobi_sweeps()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            N.call("bt_pinv_sym_f64", _dev.ptr(vd), 16, _dev.ptr(out), _dev.stream())
        e1.record()
        torch.cuda.synchronize()
        from torch.profiler import profile, ProfilerActivity
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(5):
                N.call("bt_pinv_sym_f64", _dev.ptr(vd), 16, _dev.ptr(out), _dev.stream())
            torch.cuda.synchronize()
        dev = [e.device_time_total for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        w = np.linalg.eigvalsh(v)
        vs = (v + v.T) / 2
        ref = np.linalg.pinv(v)
        err = np.abs(out.cpu().numpy() - ref).max() / np.abs(ref).max()
        print(f"   device us per launch: {[round(d, 1) for d in dev]}, max rel err vs numpy pinv {err:.2e}")
        print(f"sweep {sweep} mode {k + 1}: {e0.elapsed_time(e1) * 50:.1f} us/launch, jacobi sweeps {sw}, "
              f"eig range {w[0]:.2e}..{w[-1]:.2e}", flush=True)
        kr = khatri_rao(f[o[1]], f[o[0]])
        f[k] = us[k] @ kr @ np.linalg.pinv(v)
        f[k] /= np.linalg.norm(f[k], axis=0)
