"""The native CP phase API under mode-3 sharding, emulated in lockstep on one
GPU: R logical ranks hold their slabs; at every exchange point the harness sums
the ranks' buffers (no kernel waits on another).  Must reproduce the one-rank
run and the oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402
from paper_2105_01170_b200 import configs  # noqa: E402
from paper_2105_01170_b200.parallel import NativeCpOps, cp_als_sharded, shard_bounds  # noqa: E402


def lockstep(ops_list, iters):
    def sum_all(bufs):
        tot = bufs[0].clone()
        for b in bufs[1:]:
            tot += b          # harness plumbing: the "allreduce"
        for b in bufs:
            b.copy_(tot)

    bufs = [o.init_local() for o in ops_list]
    sum_all(bufs)
    for o, b in zip(ops_list, bufs):
        o.init_finish(b)
    for ix in range(iters):
        for mode in (1, 2):
            ms = [o.mttkrp(mode) for o in ops_list]
            sum_all(ms)
            for o, m in zip(ops_list, ms):
                o.solve_finish(mode, ix, o.solve(mode, m).clone())
        gs = [o.solve(3, o.mttkrp(3)).clone() for o in ops_list]
        sum_all(gs)
        for o, g in zip(ops_list, gs):
            o.solve_finish(3, ix, g)
        rs = [o.residual().clone() for o in ops_list]
        sum_all(rs)
        for o, r in zip(ops_list, rs):
            o.residual_finish(ix, r)
    return [o.finish(iters) for o in ops_list]


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_native_cp(world):
    I, J, K, r, iters = 40, 36, 30, 5, 8
    x = configs.c5_build(I, J, K, r)
    init = oc.normal_init((I, J, K), r, 1003)
    ops = []
    for rank in range(world):
        k0, k1 = shard_bounds(K, world, rank)
        xs = x[:, :, k0:k1].contiguous()
        f = [torch.from_numpy(init[0]).cuda(), torch.from_numpy(init[1]).cuda(),
             torch.from_numpy(init[2][k0:k1].copy()).cuda()]
        ops.append(NativeCpOps(xs, r, f[0], f[1], f[2], iters, fit="explicit"))
    hists = lockstep(ops, iters)
    ref = port.cp_als(x.cpu().numpy(), r, iters, 0.0, init=port.cp_init_normal(1003))
    for h in hists:
        np.testing.assert_allclose(h, ref.fit_history, rtol=0, atol=1e-11)
    zc = torch.cat([o.f[2] for o in ops]).cpu().numpy()
    np.testing.assert_allclose(zc, ref.z, rtol=0, atol=1e-9)
    np.testing.assert_allclose(ops[0].f[0].cpu().numpy(), ref.x, rtol=0,
                               atol=1e-9 * np.abs(ref.x).max())
    for o in ops:
        o.close()


def test_cp_als_sharded_single_rank_matches_driver():
    I, J, K, r, iters = 33, 20, 17, 4, 6
    x = configs.c5_build(I, J, K, r)
    init = oc.normal_init((I, J, K), r, 1003)
    f = [torch.from_numpy(v).cuda() for v in init]
    ops = NativeCpOps(x, r, f[0], f[1], f[2], iters)
    hist, n, conv = cp_als_sharded(ops, iters, 0.0, lambda b: None)
    ref = port.cp_als(x.cpu().numpy(), r, iters, 0.0, init=port.cp_init_normal(1003))
    np.testing.assert_allclose(hist, ref.fit_history, rtol=0, atol=1e-11)
    ops.close()
