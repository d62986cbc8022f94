"""First-contact probe on the B200 box: host facts, FP64 DMMA/DFMA peaks,
GEMM-engine fragment-layout check against torch fp64 matmul."""
import ctypes as C, json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import _native as N

lib = C.CDLL(N.LIB_PATH)
for name in ("bt_gemm_f64", "bt_gemm_f64_ws_bytes", "bt_peak_dmma", "bt_peak_dfma", "bt_last_error"):
    res, args = N._SIGS[name]; f = getattr(lib, name); f.restype = res; f.argtypes = args
out = {}
out["nproc"] = os.cpu_count()
out["mem"] = open("/proc/meminfo").read().split("\n")[:2]
out["cpu"] = [l for l in open("/proc/cpuinfo").read().split("\n") if l.startswith("model name")][:1]
print(subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout)
dev = torch.device("cuda")
st = torch.cuda.current_stream().cuda_stream
sink = torch.zeros(4096, dtype=torch.float64, device=dev)
for name, fn in (("dmma", lib.bt_peak_dmma), ("dfma", lib.bt_peak_dfma)):
    for blocks, threads in ((148 * 4, 256), (148 * 8, 256), (148 * 2, 512)):
        fl = C.c_double()
        fn(2000, blocks, threads, sink.data_ptr(), C.byref(fl), st)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        iters = 20000
        e0.record()
        fn(iters, blocks, threads, sink.data_ptr(), C.byref(fl), st)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out[f"{name}_{blocks}x{threads}_tflops"] = fl.value / ms / 1e9
print(json.dumps(out, indent=1))

def gemm(A, B, transA=False, transB=False):
    # C = op(A) @ op(B) via bt_gemm_f64 with unit-stride choices
    M = A.shape[1] if transA else A.shape[0]; K = A.shape[0] if transA else A.shape[1]
    Nn = B.shape[0] if transB else B.shape[1]
    Cm = torch.zeros(M, Nn, dtype=torch.float64, device=dev)
    d = N.GemmDesc()
    d.M, d.N, d.Kin, d.Kout, d.batch = M, Nn, K, 1, 1
    d.A = A.data_ptr(); d.B = B.data_ptr(); d.C = Cm.data_ptr()
    if transA: d.sAm, d.sAki = 1, A.shape[1]
    else: d.sAm, d.sAki = A.shape[1], 1
    if transB: d.sBn, d.sBki = B.shape[1], 1
    else: d.sBn, d.sBki = 1, B.shape[1]
    d.sCm, d.sCn = Nn, 1
    d.alpha, d.beta = 1.0, 0.0
    wsb = lib.bt_gemm_f64_ws_bytes(C.byref(d))
    ws = torch.empty(max(wsb // 8, 2), dtype=torch.float64, device=dev)
    s = lib.bt_gemm_f64(C.byref(d), ws.data_ptr(), wsb, st)
    assert s == 0, lib.bt_last_error()
    return Cm

torch.manual_seed(0)
ok = True
for (M, K, Nn) in ((37, 29, 11), (128, 64, 64), (300, 513, 70), (1000, 77, 9), (5, 4000, 64)):
    for tA in (False, True):
        for tB in (False, True):
            A = torch.randn(K, M, dtype=torch.float64, device=dev) if tA else torch.randn(M, K, dtype=torch.float64, device=dev)
            B = torch.randn(Nn, K, dtype=torch.float64, device=dev) if tB else torch.randn(K, Nn, dtype=torch.float64, device=dev)
            ref = (A.T if tA else A) @ (B.T if tB else B)
            got = gemm(A, B, tA, tB)
            err = (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-300)
            print("gemm", M, K, Nn, tA, tB, "relerr", err)
            ok &= err < 1e-13
# throughput of a big GEMM
M, K, Nn = 8192, 4096, 64
A = torch.randn(M, K, dtype=torch.float64, device=dev); B = torch.randn(K, Nn, dtype=torch.float64, device=dev)
for _ in range(3): gemm(A, B)
torch.cuda.synchronize(); t0 = time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): gemm(A, B)
e1.record(); torch.cuda.synchronize()
print("gemm 8192x4096x64 TF/s", 10 * 2 * M * K * Nn / e0.elapsed_time(e1) / 1e9)
M, K, Nn = 4096, 4096, 4096
A = torch.randn(M, K, dtype=torch.float64, device=dev); B = torch.randn(K, Nn, dtype=torch.float64, device=dev)
for _ in range(2): gemm(A, B)
e0.record()
for _ in range(3): gemm(A, B)
e1.record(); torch.cuda.synchronize()
print("gemm 4096^3 TF/s", 3 * 2 * M * K * Nn / e0.elapsed_time(e1) / 1e9)
e0.record()
for _ in range(3): torch.matmul(A, B)
e1.record(); torch.cuda.synchronize()
print("torch(cublas) 4096^3 fp64 TF/s", 3 * 2 * M * K * Nn / e0.elapsed_time(e1) / 1e9)
print("ALL_OK" if ok else "GEMM_MISMATCH")
