import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2105_01170_b200 import configs, decomp
pat, t = configs.c2_build(configs.c2_markov())
decomp.hosvd(t, [32, 400, 32]); torch.cuda.synchronize()
print("=== second call", file=sys.stderr)
decomp.hosvd(t, [32, 400, 32]); torch.cuda.synchronize()
