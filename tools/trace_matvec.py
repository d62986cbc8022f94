"""Kernel-level breakdown of the C2 BLR matvec (64 RHS) and the C4
multilevel matvec (32 volumes) via torch.profiler."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import paper_2105_01170_b200 as bt
from paper_2105_01170_b200 import configs, decomp, reconstruct, multilevel


def trace(name, fn):
    fn(); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    tot = {}
    for e in evs:
        k = e.name[:90]
        c, s = tot.get(k, (0, 0.0))
        tot[k] = (c + 1, s + e.device_time_total / 1e3)
    print(f"== {name}: wall {wall:.2f} ms, GPU {sum(s for _, s in tot.values()):.2f} ms")
    for k, (c, s) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:8]:
        print(f"  {s:8.3f} ms  {c:4d}x  {k}")


which = sys.argv[1:] or ["c2", "c4"]
if "c2" in which:
    params = configs.c2_markov()
    pat2, t2 = configs.c2_build(params)
    rep = decomp.hosvd(t2, [32, 400, 32])
    blr = reconstruct.blr_from_tucker(rep, pat2)
    rhs = torch.from_numpy(np.random.default_rng(1002).standard_normal((32768, 64))).cuda()
    trace("c2_blr_matvec64", lambda: reconstruct.matvec(blr, rhs))
if "c4" in which:
    x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
    x3 = x.reshape(255, 255, 255)
    init = configs.normal_init((255, 255, 255), 16, 2)
    decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
    res = decomp.cp_als(x3, 16, 30, 0.0)
    terms = multilevel.ml_kron_sum_from_kruskal(res.rep, mlp)
    stacks = multilevel.stack_level_mats(terms)
    vols = torch.from_numpy(np.random.default_rng(1004).standard_normal((128**3, 32))).cuda()
    trace("c4_ml_matvec32", lambda: multilevel.ml_matvec(terms, vols, stacks))
