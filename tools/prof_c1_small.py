"""Phase clocks of one sweep of the fused small CP-ALS kernel (C1)."""
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
decomp.cp_als(td, 8, 50, 0.0)
torch.cuda.synchronize()
buf = (C.c_longlong * 13)()
N.load().bt_cp_small_clocks(buf)
names = ["P", "M1", "solve1", "M2", "solve2", "M3", "solve3", "fit", ]
c = list(buf)
tot = c[8] - c[0]
print("sweep cycles", tot, f"({tot / 1.965e3:.1f} us at 1965 MHz)")
for k in range(8):
    print(f"  {names[k]:7s} {c[k + 1] - c[k]:8d} cycles")
print("pinv warp cycles (mode 1, 2, 3):", c[12], c[11], c[10])
