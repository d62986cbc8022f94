"""Per-rank compute of the C5 strong-scaling run, measured on one GPU: the
mode-3 slab a rank holds at N = 1, 2, 4, 8 (K_local = 1024 / N), 10 sweeps,
library phase events.  Comms (2 x 2 MiB + small allreduces per sweep) not
included."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, _dev
from paper_2105_01170_b200.decomp import cp_als_device

I = J = 4096
K, R = 1024, 64
init = configs.normal_init((I, J, K), R, 1003)
for n in [int(a) for a in (sys.argv[1:] or ["8", "4", "2", "1"])]:
    kl = K // n
    x = configs.c5_build(I, J, K, R, k_slab=(0, kl))
    f0 = [torch.from_numpy(init[0]).cuda(), torch.from_numpy(init[1]).cuda(),
          torch.from_numpy(init[2][:kl].copy()).cuda()]
    for rep in range(3):
        f = [v.clone() for v in f0]
        lam = _dev.empty((R,))
        ph = [0.0] * 4
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cp_als_device(x, R, f, lam, 10, 0.0, "auto", 0.0, phase_ms=ph)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    tf = 2.0 * I * J * kl * R
    print(f"N={n} K_local={kl}: {ms / 10:.2f} ms/sweep (ideal 1-GPU/N {153.4 / n:.2f}); "
          f"tree {ph[0] / 10:.2f} ms ({tf / ph[0] * 10 / 1e9:.1f} TF/s), mode2 {ph[1] / 10:.2f}, "
          f"mode3 {ph[2] / 10:.2f} ms ({tf / ph[2] * 10 / 1e9:.1f} TF/s), solves+fit {ph[3] / 10:.2f}",
          flush=True)
    del x
    torch.cuda.empty_cache()
