"""Time MTTKRP mode 1 (tree kernel) / mode 3 (generic engine) and a square
GEMM under the tuning variants (BT_TREE_CFG / BT_GEMM_CFG set by caller)."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_01170_b200 import _dev, configs, _linalg as L
from paper_2105_01170_b200 import _native as N

I, J, K, R = (int(v) for v in os.environ.get("DIMS", "2048,2048,1024,64").split(","))
x = configs.c5_build(I, J, K, R)
rng = np.random.default_rng(0)
f = [torch.from_numpy(rng.standard_normal((d, R))).cuda() for d in (I, J, K)]
pb = N.CpProblem(_dev.ptr(x), I, J, K, R, 0.0)
lib = N.load()
out = {"tree": os.environ.get("BT_TREE_CFG", "0"), "gemm": os.environ.get("BT_GEMM_CFG", "-1")}
for mode in (1, 3):
    ws = _dev.workspace(lib.bt_mttkrp_ws_bytes(C.byref(pb), mode))
    o = _dev.empty(((I, J, K)[mode - 1], R))
    def run():
        N.call("bt_mttkrp_f64", C.byref(pb), mode, _dev.ptr(f[0]), _dev.ptr(f[1]), _dev.ptr(f[2]),
               _dev.ptr(o), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[f"mode{mode}_ms"] = ms
    out[f"mode{mode}_tflops"] = 2 * I * J * K * R / ms / 1e9
a = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
b = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
L.gemm_dev(a, b); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): L.gemm_dev(a, b)
e1.record(); torch.cuda.synchronize()
out["gemm4096_tflops"] = 3 * 2 * 4096**3 / e0.elapsed_time(e1) / 1e9
print(json.dumps(out))
