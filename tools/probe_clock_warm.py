"""Do the light secondary configs (C1, C4 CP) run at reduced SM clocks after an
idle host phase?  Per-call CUDA-event times with the NVML SM clock sampled at
each call, cold (after 2 s idle) vs after a short all-SM warm burst."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
from paper_2105_01170_b200 import configs, decomp, multilevel
import paper_2105_01170_b200 as bt

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def clk():
    return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)


def warm(ms=400):
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.float32)
    t0 = time.time()
    while (time.time() - t0) * 1e3 < ms:
        for _ in range(4):
            a @ a
        torch.cuda.synchronize()


def series(name, fn, n):
    out = []
    for _ in range(n):
        c0 = clk()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append((round(e0.elapsed_time(e1), 2), c0, clk()))
    print(name, out, flush=True)


x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init4 = configs.normal_init((255, 255, 255), 16, 2)
pat, a = configs.c1_matrix()
t1 = bt.mat_to_tensor(a, pat)
init1 = configs.normal_init((32, 32, 32), 8, 0)


def c4():
    decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init4]
    return decomp.cp_als(x3, 16, 30, 0.0)


def c1():
    decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init1]
    return decomp.cp_als(t1, 8, 50, 0.0)


c4(); c1(); torch.cuda.synchronize()
for rnd in range(2):
    time.sleep(2.0)
    print("idle clk", clk())
    series("c4 cold", c4, 8)
    warm()
    print("after warm clk", clk())
    series("c4 warm", c4, 8)
    time.sleep(2.0)
    series("c1 cold", c1, 8)
    warm()
    series("c1 warm", c1, 8)
    warm()
    series("c1 warm+hot-loop", lambda: [c1() for _ in range(5)], 4)
