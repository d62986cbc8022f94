import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2105_01170_b200 import configs, decomp
pat, t = configs.c2_build(configs.c2_markov())
rep = decomp.hosvd(t, [32, 400, 32])
for k, f in enumerate(rep.factors):
    f = f if torch.is_tensor(f) else torch.from_numpy(f).cuda()
    g = f.T @ f
    print(k, tuple(f.shape), "max |F^T F - I| =", float((g - torch.eye(g.shape[0], dtype=g.dtype, device=g.device)).abs().max()))
