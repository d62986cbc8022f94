import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2105_01170_b200 import configs, decomp
pat, t = configs.c2_build(configs.c2_markov())
for _ in range(3): decomp.hosvd(t, [32, 400, 32])
ts=[]
for _ in range(11):
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); r=decomp.hosvd(t, [32, 400, 32]); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("c2 hosvd ms median", sorted(ts)[5], "min", min(ts), os.environ.get("BT_HOSVD_SIDE"))
