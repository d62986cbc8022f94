"""Phase timings of detect_pattern on the 32768^2 stand-in (digest kernel,
host grouping, verify kernel) -- CUDA events + perf_counter."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_01170_b200 as bt  # noqa: E402
from paper_2105_01170_b200 import _dev, configs  # noqa: E402
from paper_2105_01170_b200 import _native as N  # noqa: E402


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def main():
    patg, blocks = configs.gather_standin()
    a = bt.struct_assemble(patg, torch.from_numpy(blocks).cuda())
    m = n = patg.m
    ell, q = patg.ell, patg.q
    cells = ell * q
    h1 = torch.empty(cells, dtype=torch.int64, device="cuda")
    h2 = torch.empty_like(h1)
    nz = torch.empty(cells, dtype=torch.int32, device="cuda")
    res = {}
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = ev()
        N.call("bt_block_digest_f64", _dev.ptr(a), int(a.shape[1]), ell, q, m, n, 0.0,
               _dev.ptr(h1), _dev.ptr(h2), _dev.ptr(nz), _dev.stream())
        e1 = ev()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        keep = np.flatnonzero(nz.cpu().numpy())
        key = np.stack([h1.cpu().numpy()[keep], h2.cpu().numpy()[keep]], axis=1)
        _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
        leader = keep[first][inv.reshape(-1)]
        cand = np.where(leader == keep, -1, leader)
        t1 = time.perf_counter()
        cd = torch.from_numpy(cand).cuda()
        eq = torch.zeros(cells, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        e2 = ev()
        N.call("bt_block_match_f64", _dev.ptr(a), int(a.shape[1]), ell, q, m, n, _dev.ptr(cd),
               0.0, 1, _dev.ptr(eq), _dev.stream())
        e3 = ev()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        bt.detect_pattern(a, m, n)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        res = {"digest_ms": e0.elapsed_time(e1), "host_group_ms": 1e3 * (t1 - t0),
               "match_ms": e2.elapsed_time(e3), "detect_total_ms": 1e3 * (t3 - t2),
               "digest_gbs": a.numel() * 8 / e0.elapsed_time(e1) / 1e6,
               "match_gbs": a.numel() * 8 / e2.elapsed_time(e3) / 1e6}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
