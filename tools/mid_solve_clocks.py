"""Phase clocks of the last one-CTA factor update of the small-rank CP path."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, decomp, multilevel, _native as N
x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init = configs.normal_init((255, 255, 255), 16, 2)
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
decomp.cp_als(x3, 16, 5, 0.0)
buf = (C.c_longlong * 12)()
N.load().bt_debug_mid_clocks(buf)
c = list(buf)
print([c[i + 1] - c[i] for i in range(10)])
