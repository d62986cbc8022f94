"""K7 Gram (mode-1 SYRK over the C3 1024 x 524288 unfolding) and K9 TTM
(t x1 U^T, r = 64) at C3 size: CUDA-event times and TFLOP/s.  Used bare for
timing and under ncu (-k regex:bt_gemm) for the kernel profile."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import configs, _linalg as L
from paper_2105_01170_b200.tensor import ttm_dev

reps = int(os.environ.get("REPS", "3"))
pat, t = configs.c3_build()
n = t.shape[0]
N = t.numel() // n
u = L.gaussian_dev(n, 64, 7)
for name, fn, flops in (("gram_mode1", lambda: L.unfold_gram_dev(t, 1), n * (n + 1) * N),
                        ("gram_mode2", lambda: L.unfold_gram_dev(t, 2), 512 * 513 * (t.numel() // 512)),
                        ("ttm_mode1", lambda: ttm_dev(t, 1, u, 64, transpose=True), 2.0 * 64 * t.numel()),
                        ("ttm_mode2", lambda: ttm_dev(t, 2, u[:512, :32].contiguous(), 32, transpose=True), 2.0 * 32 * t.numel())):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:12s} {ms:8.3f} ms  {flops / ms / 1e9:7.2f} TFLOP/s")
