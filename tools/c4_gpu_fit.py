"""C4 full-size CP-ALS fit history on the device vs the oracle's
(tests/golden/c4_oracle_hist.json, tools/c4_oracle_fit.py)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_01170_b200 import configs, decomp, multilevel  # noqa: E402

ref = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                  "c4_oracle_hist.json")))["fit_history"]
x, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(configs.c4_psf()).cuda(), grid=128)
x3 = x.reshape(255, 255, 255)
init = configs.normal_init((255, 255, 255), 16, 2)
for fit_mode in ("explicit", "auto"):
    saved = decomp._cp_init
    decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
    try:
        res = decomp.cp_als(x3, 16, 30, 0.0, fit=fit_mode)
    finally:
        decomp._cp_init = saved
    h = np.array(res.fit_history)
    d = np.abs(h - np.array(ref))
    print(fit_mode, "first sweep with |diff| > 1e-10:", int(np.argmax(d > 1e-10)) if np.any(d > 1e-10) else None)
    print(" ".join(f"{v:.3e}" for v in d))
