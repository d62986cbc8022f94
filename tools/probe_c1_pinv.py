import sys; sys.path.insert(0,'.')
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from oracle import configs as oc, port
from paper_2105_01170_b200 import _dev
from paper_2105_01170_b200 import _native as N
pat, a = oc.c1_inputs()
t = port.gather(a, pat)
init = oc.normal_init((32, 32, 32), 8, 0)
res = port.cp_als(t, 8, 1, 0.0, init=lambda _t, _r: [f.copy() for f in init])
f = [res.x / np.linalg.norm(res.x, axis=0), res.y, res.z]
vs = {"mode1": (f[1].T @ f[1]) * (f[2].T @ f[2]), "mode2": (f[0].T @ f[0]) * (f[2].T @ f[2]), "mode3": (f[0].T @ f[0]) * (f[1].T @ f[1])}
for name, v in vs.items():
    vd = torch.from_numpy(v).cuda(); out = torch.empty_like(vd)
    N.call("bt_pinv_sym_f64", _dev.ptr(vd), 8, _dev.ptr(out), _dev.stream()); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3): N.call("bt_pinv_sym_f64", _dev.ptr(vd), 8, _dev.ptr(out), _dev.stream())
        torch.cuda.synchronize()
    dev = [e.device_time_total for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    w = np.linalg.eigvalsh(v)
    print(name, 'device us', [round(d,1) for d in dev], 'eig', w[0], w[-1], 'min |v|', np.abs(v).min(), flush=True)
