"""Kernel-level breakdown of the C2 HOSVD / C3 ST-HOSVD / C3 HOOI sweep via
torch.profiler (CUPTI sees every kernel of libbt200.so): wall time vs summed
GPU kernel time, top kernels by total time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2105_01170_b200 import configs, decomp

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
if which == "c1":
    import numpy as np
    import paper_2105_01170_b200 as bt
    from paper_2105_01170_b200 import reconstruct
    pat, a = configs.c1_matrix()
    init = configs.normal_init((32, 32, 32), 8, 0)
    rhs = torch.from_numpy(np.random.default_rng(1001).standard_normal((1024, 16))).cuda()

    def c1():
        t = bt.mat_to_tensor(a, pat)
        saved = decomp._cp_init
        decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
        try:
            res = decomp.cp_als(t, 8, 50, 0.0)
        finally:
            decomp._cp_init = saved
        ks = reconstruct.kron_sum_from_kruskal(res.rep, pat)
        err = reconstruct.error_fro(a, ks)
        return reconstruct.matvec(ks, rhs), err
    runs = {"c1_pipeline": c1}
elif which == "c2":
    params = configs.c2_markov()
    pat, t = configs.c2_build(params)
    runs = {"c2_hosvd": lambda: decomp.hosvd(t, [32, 400, 32])}
else:
    pat, t = configs.c3_build()
    rep = decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3))
    runs = {"c3_st_hosvd": lambda: decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3)),
            "c3_hooi_1": lambda: decomp.hooi(t, rep, 1, shared=(1, 3))}
for name, fn in runs.items():
    fn(); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    tot = {}
    for e in evs:
        k = e.name[:70]
        c, s = tot.get(k, (0, 0.0))
        tot[k] = (c + 1, s + e.device_time_total / 1e3 if hasattr(e, "device_time_total") else s)
    gpu = sum(s for _, s in tot.values())
    print(f"== {name}: wall {wall:.1f} ms, GPU kernel time {gpu:.1f} ms, {len(evs)} kernels")
    for k, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:14]:
        print(f"  {s:8.2f} ms  {c:5d}x  {k}")
