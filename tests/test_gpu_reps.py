"""GPU parity for the map-back stage, the matvecs, the PSD and multilevel
paths and the K3 builders -- against the reference's golden vectors and the
CPU oracle (tolerances from BASELINE.json north_star: operators/matvecs
1e-10 relative Frobenius, subspaces 1e-8 principal angle)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_01170_b200 as bt  # noqa: E402
from paper_2105_01170_b200 import configs, decomp, multilevel, psd, reconstruct  # noqa: E402
from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402

from _helpers import (PATTERN_KINDS, pattern_from, random_blocks, random_pattern,  # noqa: E402
                      random_ranks, subspace_angle)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


# ---------------------------------------------------------------------------
# converters + matvec against golden vectors
# ---------------------------------------------------------------------------

def test_converters_and_matvec_golden(golden):
    z = golden("reps")
    for c in range(int(z["n_cases"])):
        k = f"r{c}"
        pat = pattern_from(z[k + "_cells"], z[k + "_offs"], z[k + "_dims"])
        tk = bt.TuckerRep(core=z[k + "_core"], factors=(z[k + "_u"], z[k + "_v"], z[k + "_w"]))
        ks = reconstruct.kron_sum_from_tucker(tk, pat)
        assert np.array_equal(ks.coeffs, z[k + "_kc"])
        assert rel(ks.terms, z[k + "_kt"]) < 1e-13
        blr = reconstruct.blr_from_tucker(tk, pat)
        assert rel(blr.middles, z[k + "_bm"]) < 1e-13
        x = z[k + "_x"]
        c1, c2 = reconstruct.FlopCounter(), reconstruct.FlopCounter()
        assert rel(reconstruct.matvec(ks, x, c1), z[k + "_yk"]) < 1e-12
        assert rel(reconstruct.matvec(blr, x, c2), z[k + "_yb"]) < 1e-12
        assert c1.flops == int(z[k + "_fk"]) and c2.flops == int(z[k + "_fb"])
        assert rel(reconstruct.densify(ks), z[k + "_dk"]) < 1e-13
        kr = bt.KruskalRep(x=z[k + "_cx"], y=z[k + "_cy"], z=z[k + "_cz"])
        kf = reconstruct.kron_sum_from_kruskal(kr, pat)
        assert np.array_equal(kf.coeffs, z[k + "_kfc"])
        assert np.array_equal(kf.terms, z[k + "_kft"])        # exact rank-1 outer products
        if k + "_kqc" in z:
            kq = reconstruct.kron_sum_from_kruskal(kr, pat, split="qr")
            assert rel(kq.coeffs, z[k + "_kqc"]) < 1e-12
            assert rel(kq.terms, z[k + "_kqt"]) < 1e-12
        bk = reconstruct.blr_from_kruskal(kr, pat)
        assert rel(bk.left, z[k + "_bkl"]) < 1e-12
        assert rel(bk.right, z[k + "_bkr"]) < 1e-12
        assert rel(bk.middles, z[k + "_bkm"]) < 1e-11


def test_matvec_matches_dense_all_kinds():
    """test_reconstruct.py:137-149 / acceptance criterion 9 style."""
    rng = np.random.default_rng(99)
    for trial in range(40):
        pat = random_pattern(rng, PATTERN_KINDS[trial % len(PATTERN_KINDS)])
        a = port.assemble(pat, random_blocks(rng, pat))
        t = bt.mat_to_tensor(a, pat)
        tk = bt.hosvd(t, random_ranks(rng, t.shape))
        x = rng.standard_normal(pat.shape[1])
        for rep in (reconstruct.kron_sum_from_tucker(tk, pat), reconstruct.blr_from_tucker(tk, pat)):
            dense = reconstruct.densify(rep)
            ref = dense @ x
            got = reconstruct.matvec(rep, x)
            assert np.linalg.norm(ref - got) <= 1e-12 * max(np.linalg.norm(ref), 1e-300) + 1e-300


def test_matvec_block_of_rhs_equals_columns():
    rng = np.random.default_rng(5)
    pat = bt.build_pattern("hankel", 6, 6, 5, 4)
    a = port.assemble(pat, random_blocks(rng, pat))
    t = bt.mat_to_tensor(a, pat)
    tk = bt.hosvd(t, (3, 7, 4))
    xs = rng.standard_normal((pat.shape[1], 9))
    for rep in (reconstruct.kron_sum_from_tucker(tk, pat), reconstruct.blr_from_tucker(tk, pat)):
        cnt = reconstruct.FlopCounter()
        ys = reconstruct.matvec(rep, xs, cnt)
        one = reconstruct.FlopCounter()
        for c in range(9):
            np.testing.assert_allclose(ys[:, c], reconstruct.matvec(rep, xs[:, c], one),
                                       rtol=0, atol=1e-13 * np.abs(ys).max())
        assert cnt.flops == one.flops


def test_blr_matvec_wide_ranks_and_partial_patterns():
    """The row-group BLR kernel (rl <= 32 -> 4 block rows per CTA, 33..64 ->
    2; column splits; > 64 RHS) and the per-row fallback (odd rr) against
    densify @ x, on full (Hankel) and partial (banded: uncovered cells)
    patterns.  Reference semantics: reconstruct.py:300-315."""
    rng = np.random.default_rng(17)
    cases = [("hankel", dict(), 48, 40), ("banded", dict(band=3), 24, 32),
             ("toeplitz", dict(), 64, 64), ("hankel", dict(), 30, 33)]
    for kind, kw, rl, rr in cases:
        pat = bt.build_pattern(kind, 13, 13, 70, 66, **kw)
        left = rng.standard_normal((pat.m, rl))
        right = rng.standard_normal((pat.n, rr))
        mids = rng.standard_normal((pat.p, rl, rr))
        rep = reconstruct.BlockLowRankRep(pattern=pat, left=left, right=right, middles=mids)
        xs = rng.standard_normal((pat.shape[1], 70))
        ref = port.expand(pat, np.einsum("ma,kab,nb->kmn", left, mids, right)) @ xs
        got = reconstruct.matvec(rep, xs)
        assert rel(got, ref) < 1e-12, (kind, rl, rr)


@pytest.mark.parametrize("nrhs", [1, 3, 16, 17, 32, 33, 64, 70])
def test_blr_matvec_every_rhs_tile_width(nrhs):
    """The row-group kernel's RHS tile is 16, 32 or 64 wide by the number of
    right-hand sides (reconstruct.py:300-315 semantics): every width, its
    ragged edges and the > 64 RHS grid against densify @ x."""
    rng = np.random.default_rng(100 + nrhs)
    pat = bt.build_pattern("toeplitz", 11, 11, 40, 40, block_symmetric=True)
    rl = rr = 24
    left = rng.standard_normal((pat.m, rl))
    right = rng.standard_normal((pat.n, rr))
    mids = rng.standard_normal((pat.p, rl, rr))
    rep = reconstruct.BlockLowRankRep(pattern=pat, left=left, right=right, middles=mids)
    xs = rng.standard_normal((pat.shape[1], nrhs))
    ref = port.expand(pat, np.einsum("ma,kab,nb->kmn", left, mids, right)) @ xs
    got = reconstruct.matvec(rep, xs)
    assert rel(got, ref) < 1e-12


@pytest.mark.parametrize("nin,nout", [((8, 6, 10), (8, 6, 10)), ((12, 10, 8), (6, 14, 16)),
                                      ((7, 6, 10), (8, 6, 10)), ((4, 4, 4), (4, 4, 5))])
def test_ml_matvec_tma_route_equals_engine_route(nin, nout):
    """The multilevel matvec's TMA route (three rotated mode products on the
    transposed-A kernel; even extents) and the cp.async engine route (the
    fallback for odd extents) against each other and against the dense
    Kronecker sum, on cubic, non-cubic and odd level sizes."""
    import os

    rng = np.random.default_rng(sum(nin) + sum(nout))

    class T:
        def __init__(self, mats):
            self.level_mats = mats
            self.block = np.ones((1, 1))

    terms = [T([rng.standard_normal((nout[l], nin[l])) for l in range(3)]) for _ in range(5)]
    vols = rng.standard_normal((int(np.prod(nin)), 6))
    dense = sum(np.kron(np.kron(t.level_mats[0], t.level_mats[1]), t.level_mats[2]) for t in terms)
    ref = dense @ vols
    got = multilevel.ml_matvec(terms, vols)
    assert rel(got, ref) < 1e-12
    saved = os.environ.get("BT_ML_TMA")
    os.environ["BT_ML_TMA"] = "0"
    try:
        eng = multilevel.ml_matvec(terms, vols)
    finally:
        if saved is None:
            os.environ.pop("BT_ML_TMA", None)
        else:
            os.environ["BT_ML_TMA"] = saved
    assert rel(eng, ref) < 1e-12
    assert rel(got, eng) < 1e-13


def test_flop_count_linear_in_terms():
    """test_reconstruct.py:152-165 / acceptance 9: r * (2mnq + 2m nnz)."""
    rng = np.random.default_rng(8)
    pat = bt.build_pattern("toeplitz", 6, 6, 8, 8)
    a = port.assemble(pat, random_blocks(rng, pat))
    t = bt.mat_to_tensor(a, pat)
    x = rng.standard_normal(pat.shape[1])
    nnz = sum(pat.counts)
    per = 2 * pat.m * pat.n * pat.q + 2 * pat.m * nnz
    for r in range(1, 7):
        rep = reconstruct.kron_sum_from_tucker(bt.tucker_partial(t, [None, r, None]), pat)
        cnt = reconstruct.FlopCounter()
        reconstruct.matvec(rep, x, cnt)
        assert cnt.flops == r * per


def test_error_fro_equals_tensor_error_and_c1(golden):
    z = golden("cp")
    pat_o, a = oc.c1_inputs()
    pat = bt.build_pattern("toeplitz", 32, 32, 32, 32, block_symmetric=True)
    kr = bt.KruskalRep(x=z["c1_x"], y=z["c1_y"], z=z["c1_z"])
    ks = reconstruct.kron_sum_from_kruskal(kr, pat)
    err = reconstruct.error_fro(a, ks)
    assert abs(err - float(z["c1_relerr"])) < 1e-12
    ys = reconstruct.matvec(ks, z["c1_rhs"])
    assert rel(ys, z["c1_mv"]) < 1e-12


def test_densify_guard_and_shapes():
    big = bt.build_pattern("diagonal", 11000, 11000, 1, 1)
    rep = reconstruct.KronSumRep(pattern=big, coeffs=np.ones((big.p, 1)), terms=np.ones((1, 1, 1)))
    with pytest.raises(bt.ShapeError):
        reconstruct.densify(rep)
    pat = bt.build_pattern("diagonal", 2, 2, 2, 2)
    with pytest.raises(bt.ShapeError):
        reconstruct.matvec(reconstruct.KronSumRep(pattern=pat, coeffs=np.ones((2, 1)),
                                                  terms=np.ones((1, 2, 2))), np.zeros(5))


# ---------------------------------------------------------------------------
# Tucker / PSD (C2, C3 at reduced size)
# ---------------------------------------------------------------------------

def test_c2_small_hosvd_blr_matvec(golden):
    z = golden("tucker")
    pat, t = configs.c2_build(z["c2s_params"])
    assert np.array_equal(t.cpu().numpy(), z["c2s_t"])   # K3 Hankel builder is bit-exact
    rep = bt.hosvd(z["c2s_t"], [8, 40, 8])
    # leading, well-separated part of the mode-2 basis agrees; the operator agrees
    sv = np.linalg.svd(port.unfold(z["c2s_t"], 2), compute_uv=False)
    lead = int(np.sum(sv > 1e-3 * sv[0]))
    assert subspace_angle(rep.factors[1][:, :lead], z["c2s_v"][:, :lead]) < 1e-8
    blr = reconstruct.blr_from_tucker(rep, pat)
    ys = reconstruct.matvec(blr, z["c2s_rhs"])
    assert rel(ys, z["c2s_mv"]) < 1e-10
    cnt = reconstruct.FlopCounter()
    reconstruct.matvec(blr, z["c2s_rhs"][:, 0], cnt)
    assert cnt.flops == int(z["c2s_flops"])


def test_c3_small_partial_tucker_and_spsd(golden):
    z = golden("tucker")
    rep = bt.tucker_partial(z["c3s_t"], [8, 4, 8], shared=(1, 3))
    assert rep.factors[0] is rep.factors[2]
    assert subspace_angle(rep.factors[0], z["c3s_u"]) < 1e-8
    # the core depends on the basis inside degenerate singular pairs (the
    # symmetric tensor has them); the projected tensor does not
    recon = lambda c, u: port.mode_multiply(port.mode_multiply(c, 1, u), 3, u)  # noqa: E731
    assert rel(recon(rep.core, rep.factors[0]), recon(z["c3s_core"], z["c3s_u"])) < 1e-10
    pat = bt.build_pattern("toeplitz", 10, 10, 36, 36, block_symmetric=True)
    sp = psd.spsd_compress_blocks(pat, z["c3s_blocks"], 8)
    assert subspace_angle(sp.basis, z["c3s_spsd_u"]) < 1e-8
    proj = lambda u, b: np.einsum("ia,kab,jb->kij", u, b, u)  # noqa: E731
    assert rel(proj(sp.basis, sp.blocks), proj(z["c3s_spsd_u"], z["c3s_spsd_blocks"])) < 1e-10
    assert abs(sp.trace() - float(z["c3s_trace"])) < 1e-9 * abs(float(z["c3s_trace"]))
    d1 = sp.densify()
    d2 = reconstruct.densify(sp.as_blr())
    assert np.max(np.abs(d1 - d2)) < 1e-12


def test_c3_builder_and_st_hosvd_hooi_vs_oracle():
    pat, t = configs.c3_build(side=6, lags=10)
    _, _, to = oc.c3_tensor(side=6, lags=10)
    assert rel(t.cpu().numpy(), to) < 1e-14
    rep = decomp.st_hosvd(to, [8, 4, 8], shared=(1, 3))
    core_o, fac_o = port.st_hosvd_shared13(to, 8, 4)
    assert subspace_angle(rep.factors[0], fac_o[0]) < 1e-8
    assert subspace_angle(rep.factors[1], fac_o[1]) < 1e-8
    rep2 = decomp.hooi(to, rep, 3, shared=(1, 3))
    core2, fac2 = port.hooi_shared13(to, fac_o[0], fac_o[1], 3)
    assert subspace_angle(rep2.factors[0], fac2[0]) < 1e-8
    recon = lambda c, f: port.mode_multiply(port.mode_multiply(port.mode_multiply(c, 1, f[0]), 2, f[1]), 3, f[2])  # noqa: E731
    assert rel(recon(rep2.core, rep2.factors), recon(core2, fac2)) < 1e-10


def test_transpose_closure_rejection():
    pat = bt.build_pattern("toeplitz", 3, 3, 2, 2)
    blocks = np.arange(5 * 4, dtype=float).reshape(5, 2, 2)
    with pytest.raises(bt.PatternMismatchError, match="block transpose differs"):
        psd.check_transpose_closed(pat, blocks)
    cells = np.array([[0, 1], [1, 2]])
    pat_up = bt.BlockPattern(ell=3, q=3, m=2, n=2, placements=(cells,))
    with pytest.raises(bt.PatternMismatchError, match="transposed support"):
        psd.check_transpose_closed(pat_up, blocks[:1])
    with pytest.raises(bt.ShapeError):
        psd.spsd_compress_blocks(bt.build_pattern("toeplitz", 3, 3, 2, 3), np.zeros((5, 2, 3)), 1)


# ---------------------------------------------------------------------------
# multilevel + builders
# ---------------------------------------------------------------------------

def test_psf_tensor_bit_exact_and_ml_matvec(golden):
    z = golden("psf")
    for k in (3, 5, 7):
        x, mlp = multilevel.psf_weighted_tensor(z[f"psf{k}"])
        assert np.array_equal(x, z[f"x{k}"])
        assert mlp.dims == (1, k, k, k, 1)
    # generalised grid against the oracle
    psf = oc.c4_psf(7)
    x, mlp = multilevel.psf_weighted_tensor(psf, grid=9)
    assert np.array_equal(x[0, :, :, :, 0], port.psf_weighted(psf, 9))
    # CP route -> multilevel terms -> batched matvec vs the reference's dense operator
    kr = bt.KruskalRep(x=z["c4s_cx"], y=z["c4s_cy"], z=z["c4s_cz"])
    x7, mlp7 = multilevel.psf_weighted_tensor(z["c4s_psf"])
    terms = multilevel.ml_kron_sum_from_kruskal(kr, mlp7)
    y = multilevel.ml_matvec(terms, z["c4s_vols"])
    assert rel(y, z["c4s_mv"]) < 1e-12


def test_c4_small_cp_matches_reference(golden):
    z = golden("psf")
    t = z["c4s_x"][0, :, :, :, 0]
    saved = decomp._cp_init
    decomp._cp_init = lambda _t, _r: [f.copy() for f in oc.normal_init(t.shape, 3, 2)]
    try:
        res = bt.cp_als(t, 3, 30, 0.0)
    finally:
        decomp._cp_init = saved
    np.testing.assert_allclose(np.array(res.fit_history), z["c4s_hist"], rtol=0, atol=1e-9)


def test_c5_builder_vs_oracle(golden):
    z = golden("cp")
    i, j, k, r = (int(v) for v in z["c5s_dims"])
    x = configs.c5_build(i, j, k, r).cpu().numpy()
    assert rel(x, z["c5s_t"]) < 1e-14
    xs = configs.c5_build(i, j, k, r, k_slab=(8, 20)).cpu().numpy()
    assert rel(xs, z["c5s_t"][:, :, 8:20]) < 1e-14


def test_mttkrp_modes_vs_oracle():
    import ctypes as C

    from paper_2105_01170_b200 import _dev
    from paper_2105_01170_b200 import _native as N
    from scipy.linalg import khatri_rao

    rng = np.random.default_rng(3)
    for dims, r in (((9, 13, 7), 5), ((40, 33, 70), 16), ((64, 130, 48), 64), ((20, 21, 22), 70)):
        x = rng.standard_normal(dims)
        f = [rng.standard_normal((d, r)) for d in dims]
        xd = torch.from_numpy(x).cuda()
        fd = [torch.from_numpy(v).cuda() for v in f]
        pb = N.CpProblem(_dev.ptr(xd), *dims, r, 0.0)
        for mode in (1, 2, 3):
            ws = _dev.workspace(N.load().bt_mttkrp_ws_bytes(C.byref(pb), mode))
            out = _dev.empty((dims[mode - 1], r))
            N.call("bt_mttkrp_f64", C.byref(pb), mode, _dev.ptr(fd[0]), _dev.ptr(fd[1]),
                   _dev.ptr(fd[2]), _dev.ptr(out), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
            o = [j for j in range(3) if j != mode - 1]
            ref = port.unfold(x, mode) @ khatri_rao(f[o[1]], f[o[0]])
            assert rel(out.cpu().numpy(), ref) < 1e-13, (dims, r, mode)
