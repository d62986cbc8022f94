import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_01170_b200 import configs, decomp, multilevel
from oracle import configs as oc, port
x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
xg = x.reshape(255, 255, 255).cpu().numpy()
xo = oc.c4_tensor().reshape(255, 255, 255)
print("tensor max diff", np.abs(xg - xo).max(), "norm", np.linalg.norm(xo))
init = oc.normal_init((255, 255, 255), 16, 2)
for iters in (1, 2):
    ro = port.cp_als(xo, 16, iters, 0.0, init=lambda t, r: init)
    saved = decomp._cp_init
    decomp._cp_init = lambda _t, _r: [torch.from_numpy(f.copy()).cuda() for f in init]
    try:
        rg = decomp.cp_als(torch.from_numpy(xo).cuda(), 16, iters, 0.0, fit="explicit")
    finally:
        decomp._cp_init = saved
    print(iters, "fit oracle", ro.fit_history, "gpu", rg.fit_history)
    for name, a, b in (("x", ro.x, rg.rep.x), ("y", ro.y, rg.rep.y), ("z", ro.z, rg.rep.z)):
        b = b.cpu().numpy()
        print("  ", name, "rel diff", np.linalg.norm(a - b) / np.linalg.norm(a))
