"""C4 full-size CP-ALS fit history from the oracle port (numpy pinv/SVD as
in decomp.py:344-410), for comparison with the device path.  CPU only.
    python tools/c4_oracle_fit.py > tests/golden/c4_oracle_hist.json"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402

t0 = time.time()
x = oc.c4_tensor()
x3 = x.reshape(255, 255, 255)
init = oc.normal_init((255, 255, 255), 16, 2)
res = port.cp_als(x3, 16, 30, 0.0, init=lambda t, r: init)
print(json.dumps({"fit_history": list(map(float, res.fit_history)), "secs": time.time() - t0}))
