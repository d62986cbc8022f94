"""Host-side profile of the C1 cp_als call (where the ~0.7 ms outside the kernel goes)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_01170_b200 as bt
from paper_2105_01170_b200 import configs, decomp
pat, a = configs.c1_matrix()
init = configs.normal_init((32, 32, 32), 8, 0)
t = bt.mat_to_tensor(a, pat)
td = t if torch.is_tensor(t) else torch.from_numpy(t).cuda()
decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
for _ in range(5):
    decomp.cp_als(td, 8, 50, 0.0)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    decomp.cp_als(td, 8, 50, 0.0)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr).sort_stats("cumulative")
st.print_stats(22)
