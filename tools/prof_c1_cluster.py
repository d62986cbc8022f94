"""Phase clocks of one sweep of the cluster CP-ALS kernel (C1), rank 0."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_01170_b200 as bt
from paper_2105_01170_b200 import configs, decomp, _native as N
pat, a = configs.c1_matrix()
init = configs.normal_init((32, 32, 32), 8, 0)
t = bt.mat_to_tensor(a, pat)
td = t if torch.is_tensor(t) else torch.from_numpy(t).cuda()
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
for _ in range(3):
    decomp.cp_als(td, 8, 50, 0.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); res = decomp.cp_als(td, 8, 50, 0.0); e1.record(); torch.cuda.synchronize()
print(f"cp_als 50 sweeps: {e0.elapsed_time(e1):.3f} ms, fit {res.fit}")
buf = (C.c_longlong * 16)()
N.load().bt_cp_cluster_clocks(buf)
c = list(buf)
names = ["P+pinv1", "M1+rows", "sync1", "finish1", "M2part", "sync2", "finish2", "M3part", "sync3", "finish3"]
print("sweep cycles", c[10] - c[0], f"({(c[10] - c[0]) / 1.965e3:.1f} us)")
for k, n in enumerate(names):
    print(f"  {n:8s} {c[k + 1] - c[k]:7d}")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    decomp.cp_als(td, 8, 50, 0.0); torch.cuda.synchronize()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        print(f"  {e.device_time_total:8.1f} us {e.name[:70]}")
