"""C1 timings: cp_als alone (50 sweeps) and the bench's full C1 pipeline,
CUDA events over several repetitions after warm-up."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_01170_b200 as bt
from paper_2105_01170_b200 import configs, decomp, reconstruct

pat, a = configs.c1_matrix()
init = configs.normal_init((32, 32, 32), 8, 0)
rhs = torch.from_numpy(np.random.default_rng(1001).standard_normal((1024, 16))).cuda()
t = bt.mat_to_tensor(a, pat)
td = t if torch.is_tensor(t) else torch.from_numpy(t).cuda()
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]


def cp():
    return decomp.cp_als(td, 8, 50, 0.0)


def c1():
    tt = bt.mat_to_tensor(a, pat)
    res = decomp.cp_als(tt, 8, 50, 0.0)
    ks = reconstruct.kron_sum_from_kruskal(res.rep, pat)
    err = reconstruct.error_fro(a, ks)
    return reconstruct.matvec(ks, rhs), err


for name, fn in (("cp_als 50 sweeps (device tensor)", cp), ("C1 pipeline", c1)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name}: min {min(ts):.2f} ms, median {sorted(ts)[5]:.2f} ms")
