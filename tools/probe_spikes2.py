"""Single cp_als calls (C1, C4): CUDA-event time with the NVML SM / memory
clocks and the throttle mask sampled after each call; cold vs after an
HBM-streaming warm-up."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
from paper_2105_01170_b200 import configs, decomp, multilevel, _dev
from paper_2105_01170_b200.tensor import fro_norm_dev
import paper_2105_01170_b200 as bt

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255).contiguous()
init4 = [torch.from_numpy(f).cuda() for f in configs.normal_init((255, 255, 255), 16, 2)]
pat, a = configs.c1_matrix()
t1 = bt.mat_to_tensor(a, pat)
init1 = [torch.from_numpy(f).cuda() for f in configs.normal_init((32, 32, 32), 8, 0)]
buf = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
buf2 = torch.empty_like(buf)


def hbm_warm(ms=300):
    t0 = time.time()
    while (time.time() - t0) * 1e3 < ms:
        buf2.copy_(buf)
        torch.cuda.synchronize()


def run(name, xd, init, r, iters, n=12, pre=None):
    rows = []
    nt = fro_norm_dev(xd)
    for _ in range(n):
        if pre:
            pre()
        f = [g.clone() for g in init]
        lam = _dev.empty((r,))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        decomp.cp_als_device(xd, r, f, lam, iters, 0.0, "auto", nt)
        e1.record()
        torch.cuda.synchronize()
        rows.append((round(e0.elapsed_time(e1), 2),
                     pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                     pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                     hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)),
                     pynvml.nvmlDeviceGetPowerUsage(h) // 1000))
    print(name, "(ms, sm, mem, reasons, W):", rows, flush=True)


print("max clocks", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM),
      pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_MEM))
for _ in range(2):
    run("c4", x3, init4, 16, 30)
    run("c1", t1, init1, 8, 50)
    run("c4 hbm-warm", x3, init4, 16, 30, pre=hbm_warm)
    run("c1 hbm-warm", t1, init1, 8, 50, pre=hbm_warm)
