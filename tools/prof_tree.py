"""Time (and, under ncu, profile) the two C5 full-pass kernels in isolation
on a reduced-I slab of the C5 tensor (same J, K, R, so every CTA does the
same work as at full size): mode 1 = tree_p_ws_kernel (no P store, Q tree),
mode 2 = the Q GEMM (+ mode-2 reduction).

    python tools/prof_tree.py [I] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2105_01170_b200 import configs
from paper_2105_01170_b200.parallel import NativeCpOps

I = int(sys.argv[1]) if len(sys.argv) > 1 else 512
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 5
J, K, R = 4096, 1024, 64
x = configs.c5_build(I, J, K, R)
init = configs.normal_init((I, J, K), R, 1003)
f = [torch.from_numpy(v).cuda() for v in init]
ops = NativeCpOps(x, R, f[0], f[1], f[2], 1)
buf = ops.init_local()
ops.init_finish(buf)
flops = 2.0 * I * J * K * R
for mode in (1, 2):
    ops.mttkrp(mode)
    torch.cuda.synchronize()
    ts = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.mttkrp(mode)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"mode {mode}: {ms:.3f} ms  {flops / ms / 1e9:.2f} TF/s  (all: {[round(t, 3) for t in ts]})",
          flush=True)
ops.close()
