"""Jacobi sweeps / cycles of every R=16 pinv call along the C4 CP-ALS run
(the ring log of pinv_jacobi1_kernel)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp, multilevel, _native as N

x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init = configs.normal_init((255, 255, 255), 16, 2)
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
lib = N.load()
lib.bt_debug_pinv1s_log.restype = C.c_int64
buf = (C.c_longlong * 512)()
n0 = lib.bt_debug_pinv1s_log(buf)
res = decomp.cp_als(x3, 16, 30, 0.0)
n1 = lib.bt_debug_pinv1s_log(buf)
print("calls", n1 - n0, "fit", res.fit)
ent = [buf[i & 511] for i in range(n0, n1)]
for i, e in enumerate(ent):
    print(f"jacobi call {i:3d}: sweeps {e >> 56:3d}, rank {(e >> 48) & 255:2d}, dmin/d0 1e-{(e >> 40) & 255:<3d} {(e & 0xffffffff) / 1.965e3:7.1f} us")
