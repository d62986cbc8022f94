"""The mode-3-sharded CP-ALS orchestration (parallel.cp_als_sharded) with
world_size 2 over gloo on CPU, against the single-process oracle: checks that
the exchange points (sums of the mode-1/2 MTTKRP partials, of the mode-3
Gram/inner buffer, of the residual and init buffers) reproduce the unsharded
algorithm of decomp.py:344-410."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402
from paper_2105_01170_b200.parallel import cp_als_sharded, shard_bounds, torch_allreduce  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_no, dims, r, iters, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from _np_cp_ops import NumpyCpOps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        I, J, K = dims
        x = oc.c5_tensor(I, J, K, r)
        init = oc.normal_init((I, J, K), r, 1003)
        k0, k1 = shard_bounds(K, world, rank)
        ops = NumpyCpOps(np.ascontiguousarray(x[:, :, k0:k1]), r, init[0], init[1],
                         init[2][k0:k1], iters)
        hist, n, conv = cp_als_sharded(ops, iters, 0.0, torch_allreduce())
        q.put((rank, hist, ops.f[0], ops.f[1], ops.f[2], k0, k1))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover():
    for K in (1, 7, 8, 1024, 1023):
        for world in (1, 2, 3, 4, 8):
            if world > K:
                continue
            spans = [shard_bounds(K, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == K
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


@pytest.mark.parametrize("dims,r", [((12, 10, 9), 3), ((16, 8, 6), 4)])
def test_sharded_cp_matches_single_process(dims, r):
    world, iters = 2, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _port()
    procs = [ctx.Process(target=_worker, args=(k, world, port_no, dims, r, iters, q))
             for k in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = oc.c5_tensor(*dims, r)
    ref = port.cp_als(x, r, iters, 0.0, init=port.cp_init_normal(1003))
    # every rank computes the same fit history and the same replicated factors
    for rank, hist, a, b, c, k0, k1 in res:
        np.testing.assert_allclose(hist, ref.fit_history, rtol=0, atol=1e-12)
        np.testing.assert_allclose(a, ref.x, rtol=0, atol=1e-10 * np.abs(ref.x).max())
        np.testing.assert_allclose(b, ref.y, rtol=0, atol=1e-10)
        np.testing.assert_allclose(c, ref.z[k0:k1], rtol=0, atol=1e-10)
    assert np.array_equal(res[0][2], res[1][2])


def _tucker_worker(rank, world, port_no, side, lags, r13, r2, sweeps, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from _np_tucker_ops import TorchCpuTuckerOps
    from paper_2105_01170_b200.parallel import (hooi_sharded, st_hosvd_sharded,
                                                torch_allgather_mode2)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, _, t = oc.c3_tensor(side=side, lags=lags)
        p0, p1 = shard_bounds(t.shape[1], world, rank)
        xl = torch.from_numpy(np.ascontiguousarray(t[:, p0:p1, :]))
        ops = TorchCpuTuckerOps()
        red, gat = torch_allreduce(), torch_allgather_mode2()
        u, v, core = st_hosvd_sharded(ops, xl, r13, r2, red, gat)
        u2, v2, core2 = hooi_sharded(ops, xl, u, v, sweeps, p0, p1, red, gat)
        q.put((rank, u.numpy(), v.numpy(), core.numpy(), u2.numpy(), v2.numpy(), core2.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_st_hosvd_hooi_matches_single_process(world):
    """C3 recipe (reduced): the time-mode-sharded ST-HOSVD + HOOI (mode-1 Gram
    sums, mode-2 all-gather, U-step partial sums) reproduces the unsharded
    oracle (decomp.st_hosvd / hooi restated in oracle/port.py)."""
    side, lags, r13, r2, sweeps = 4, 7, 5, 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _port()
    procs = [ctx.Process(target=_tucker_worker,
                         args=(k, world, port_no, side, lags, r13, r2, sweeps, q))
             for k in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, _, t = oc.c3_tensor(side=side, lags=lags)
    core_o, (uo, vo, _) = port.st_hosvd_shared13(t, r13, r2)
    core_h, (uh, vh, _) = port.hooi_shared13(t, uo, vo, sweeps)

    def recon(core, u, v):
        return port.mode_multiply(port.mode_multiply(port.mode_multiply(core, 1, u), 2, v), 3, u)

    ref0, ref1 = recon(core_o, uo, vo), recon(core_h, uh, vh)
    for rank, u, v, core, u2, v2, core2 in res:
        assert np.linalg.norm(recon(core, u, v) - ref0) <= 1e-10 * np.linalg.norm(ref0)
        assert np.linalg.norm(recon(core2, u2, v2) - ref1) <= 1e-10 * np.linalg.norm(ref1)
        # (factors themselves are not compared: the small C3 grid has
        # degenerate singular pairs, so only the reconstructions are unique)
    for k in range(1, world):
        assert np.array_equal(res[0][1], res[k][1]) and np.array_equal(res[0][6], res[k][6])
