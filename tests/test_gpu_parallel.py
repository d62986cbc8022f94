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


def test_tucker_sharded_native_single_rank_matches_decomp():
    """parallel.st_hosvd_sharded / hooi_sharded on the native ops with
    identity collectives == decomp.st_hosvd / hooi (shared=(1, 3))."""
    import paper_2105_01170_b200 as bt
    from paper_2105_01170_b200.parallel import NativeTuckerOps, hooi_sharded, st_hosvd_sharded

    pat, t = configs.c3_build(side=6, lags=10)
    ops = NativeTuckerOps()
    ident = lambda b: None  # noqa: E731
    same = lambda y: y      # noqa: E731
    u, v, core = st_hosvd_sharded(ops, t, 8, 4, ident, same)
    rep = bt.st_hosvd(t, [8, 4, 8], shared=(1, 3))
    assert torch.equal(u, rep.factors[0]) and torch.equal(v, rep.factors[1])
    assert torch.equal(core, rep.core)
    u2, v2, core2 = hooi_sharded(ops, t, u, v, 2, 0, int(t.shape[1]), ident, same)
    rep2 = bt.hooi(t, rep, 2, shared=(1, 3))
    assert torch.equal(u2, rep2.factors[0]) and torch.equal(v2, rep2.factors[1])

    def recon(c, uu, vv):
        return port.mode_multiply(port.mode_multiply(port.mode_multiply(c, 1, uu), 2, vv), 3, uu)

    a = recon(core2.cpu().numpy(), u2.cpu().numpy(), v2.cpu().numpy())
    b = recon(rep2.core.cpu().numpy(), rep2.factors[0].cpu().numpy(), rep2.factors[1].cpu().numpy())
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)


def test_tucker_c3_distributed_single_process():
    from paper_2105_01170_b200.parallel import tucker_c3_distributed

    _, _, t = oc.c3_tensor(side=6, lags=10)
    rep = tucker_c3_distributed(t, 8, 4, hooi_sweeps=2)
    assert isinstance(rep.core, np.ndarray) and rep.factors[0] is rep.factors[2]
    core_o, fac = port.st_hosvd_shared13(t, 8, 4)
    core_h, (uh, vh, _) = port.hooi_shared13(t, fac[0], fac[1], 2)

    def recon(c, uu, vv):
        return port.mode_multiply(port.mode_multiply(port.mode_multiply(c, 1, uu), 2, vv), 3, uu)

    ref = recon(core_h, uh, vh)
    got = recon(rep.core, rep.factors[0], rep.factors[1])
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("world", [2, 3])
def test_matvec_rhs_sharded_concat_equals_full(world):
    import paper_2105_01170_b200 as bt
    from paper_2105_01170_b200.parallel import matvec_sharded

    _, a = oc.c1_inputs()
    pat = bt.build_pattern("toeplitz", 32, 32, 32, 32, block_symmetric=True)
    res = bt.cp_als(bt.mat_to_tensor(a, pat), 4, 5, 0.0)
    rep = bt.kron_sum_from_kruskal(res.rep, pat)
    x = np.random.default_rng(1001).standard_normal((1024, 16))
    full = bt.matvec(rep, x)
    parts = [matvec_sharded(rep, x, world, k) for k in range(world)]
    got = np.concatenate(parts, axis=1)
    assert np.linalg.norm(got - full) <= 1e-14 * np.linalg.norm(full)


def _variant(x, r):
    import ctypes as C

    from paper_2105_01170_b200 import _dev
    from paper_2105_01170_b200 import _native as N

    I, J, K = (int(s) for s in x.shape)
    pb = N.CpProblem(_dev.ptr(x), I, J, K, r, 0.0)
    return N.load().bt_cp_tree_variant(C.byref(pb))


@pytest.mark.parametrize("world", [1, 2, 4])
def test_sharded_native_cp_qtree(world):
    """Short mode-3 slabs (a rank's slab at 4-8 GPUs) take the Q = X x1 A
    dimension tree (mode 1 a direct GEMM, modes 2/3 from Q): same fits as the
    oracle, sharded and not."""
    I, J, K, r, iters = 160, 48, 40, 20, 6
    x = configs.c5_build(I, J, K, r)
    init = oc.normal_init((I, J, K), r, 1003)
    ops = []
    for rank in range(world):
        k0, k1 = shard_bounds(K, world, rank)
        xs = x[:, :, k0:k1].contiguous()
        assert _variant(xs, r) == 1
        f = [torch.from_numpy(init[0]).cuda(), torch.from_numpy(init[1]).cuda(),
             torch.from_numpy(init[2][k0:k1].copy()).cuda()]
        ops.append(NativeCpOps(xs, r, f[0], f[1], f[2], iters, fit="explicit"))
    hists = lockstep(ops, iters)
    ref = port.cp_als(x.cpu().numpy(), r, iters, 0.0, init=port.cp_init_normal(1003))
    for h in hists:
        np.testing.assert_allclose(h, ref.fit_history, rtol=0, atol=1e-11)
    zc = torch.cat([o.f[2] for o in ops]).cpu().numpy()
    np.testing.assert_allclose(zc, ref.z, rtol=0, atol=1e-9)
    np.testing.assert_allclose(ops[0].f[1].cpu().numpy(), ref.y, rtol=0, atol=1e-9)
    for o in ops:
        o.close()


def test_cp_als_qtree_public_api_and_variant_rule():
    import paper_2105_01170_b200 as bt
    from paper_2105_01170_b200 import decomp

    assert _variant(configs.c5_build(64, 64, 64, 4), 4) == 0        # R <= 16: P tree
    assert _variant(configs.c5_build(32, 64, 64, 32), 32) == 0      # K > I: P tree
    # K <= 256: mode 1 through the batched T = X[i]^T B GEMM; K > 256: the
    # tree kernel without its P store
    for I, J, K, r, iters in ((200, 64, 48, 24, 10), (300, 16, 272, 20, 6)):
        x = configs.c5_build(I, J, K, r)
        assert _variant(x, r) == 1
        init = oc.normal_init((I, J, K), r, 7)
        saved = decomp._cp_init
        decomp._cp_init = lambda _t, _r: [v.copy() for v in init]
        try:
            res = bt.cp_als(x.cpu().numpy(), r, iters, 0.0, fit="explicit")
        finally:
            decomp._cp_init = saved
        ref = port.cp_als(x.cpu().numpy(), r, iters, 0.0,
                          init=lambda _t, _r: [v.copy() for v in init])
        np.testing.assert_allclose(res.fit_history, ref.fit_history, rtol=0, atol=1e-11)
        np.testing.assert_allclose(res.rep.z, ref.z, rtol=0, atol=1e-9)
