"""Small-rank two-pass CP path (cp_mid.cu) against the oracle on ragged
shapes, all fit modes, tol > 0; then the C4 timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_01170_b200 as bt
from paper_2105_01170_b200 import decomp
from oracle import port, configs as oc

def run(shape, r, iters, tol, fit, seed, noise=1e-2):
    rng = np.random.default_rng(seed)
    f = [rng.standard_normal((n, r)) for n in shape]
    x = np.einsum("ir,jr,kr->ijk", *f) + noise * rng.standard_normal(shape)
    init = oc.normal_init(shape, r, seed + 1)
    saved = decomp._cp_init
    decomp._cp_init = lambda _t, _r: [v.copy() for v in init]
    try:
        res = bt.cp_als(x, r, iters, tol, fit=fit)
    finally:
        decomp._cp_init = saved
    ref = port.cp_als(x, r, iters, tol, init=lambda _t, _r: [v.copy() for v in init])
    hg, hr = np.array(res.fit_history), np.array(ref.fit_history)
    n = min(len(hg), len(hr))
    dh = np.abs(hg[:n] - hr[:n]).max()
    rel = lambda a, b: np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)
    print(f"{shape} R={r} iters={iters} tol={tol} fit={fit}: n_iters {res.n_iters}/{ref.n_iters} conv {res.converged}/{ref.converged} "
          f"|dfit| {dh:.2e} x {rel(res.rep.x, ref.x):.2e} y {rel(res.rep.y, ref.y):.2e} z {rel(res.rep.z, ref.z):.2e}", flush=True)

run((70, 60, 33), 5, 8, 0.0, "auto", 1)
run((96, 80, 64), 16, 8, 0.0, "auto", 2)
run((96, 80, 64), 16, 8, 0.0, "gram", 2)
run((96, 80, 64), 16, 8, 0.0, "explicit", 2)
run((100, 90, 300), 12, 6, 0.0, "auto", 3)
run((65, 64, 257), 9, 6, 0.0, "auto", 4)
run((128, 33, 40), 8, 40, 1e-7, "auto", 5)
run((128, 33, 40), 16, 12, 0.0, "auto", 6, noise=1e-6)
if len(sys.argv) > 1:
    import subprocess
    subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "time_c4cp.py")])
    subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "trace_c4cp.py")])
