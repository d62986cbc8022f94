"""DMMA throughput vs warps per SM and independent chains per warp."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_01170_b200 import _native as N
lib = N.load()
sink = torch.zeros(1 << 16, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for warps in (4, 8, 16, 32):
    for chains in (4, 8, 16, 32):
        fl = C.c_double()
        lib.bt_peak_dmma_chains(200, 148, warps * 32, chains, sink.data_ptr(), C.byref(fl), st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.bt_peak_dmma_chains(20000, 148, warps * 32, chains, sink.data_ptr(), C.byref(fl), st)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps({"warps_per_sm": warps, "chains": chains,
                          "tflops": fl.value / e0.elapsed_time(e1) / 1e9}), flush=True)
