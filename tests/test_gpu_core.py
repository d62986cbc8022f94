"""GPU parity: GEMM engine, K1/K2 maps, CP-ALS, eigensolver, Tucker against
the reference's golden vectors and the CPU oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_01170_b200 as bt  # noqa: E402
from paper_2105_01170_b200 import _linalg as L  # noqa: E402
from paper_2105_01170_b200 import decomp  # noqa: E402
from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402

from _helpers import pattern_from, subspace_angle  # noqa: E402


def with_init(init):
    saved = decomp._cp_init
    decomp._cp_init = lambda t, r: [np.array(f, copy=True) for f in init]
    return saved


# ---------------------------------------------------------------------------
# GEMM engine
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(37, 29, 11), (300, 513, 70), (1000, 77, 9), (5, 4000, 64),
                                   (130, 17, 130)])
@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
def test_gemm_layouts(shape, ta, tb):
    M, K, Nn = shape
    g = torch.Generator(device="cuda").manual_seed(M + K + Nn)
    a = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn((Nn, K) if tb else (K, Nn), dtype=torch.float64, device="cuda", generator=g)
    ref = (a.T if ta else a) @ (b.T if tb else b)
    got = L.gemm_dev(a, b, ta, tb)
    assert torch.allclose(got, ref, rtol=0, atol=1e-12 * ref.abs().max().item())


@pytest.mark.parametrize("dims,mode", [((7, 9, 5), 1), ((7, 9, 5), 2), ((7, 9, 5), 3),
                                       ((40, 300, 33), 2), ((300, 4, 6), 1), ((3, 5, 260), 3)])
def test_unfold_gram(dims, mode):
    x = np.random.default_rng(1).standard_normal(dims)
    g = L.unfold_gram_dev(torch.from_numpy(x).cuda(), mode).cpu().numpy()
    u = port.unfold(x, mode)
    np.testing.assert_allclose(g, u @ u.T, rtol=0, atol=1e-12 * np.abs(g).max())
    assert np.array_equal(g, g.T)


@pytest.mark.parametrize("dims,mode,rows", [((7, 9, 5), 1, 3), ((7, 9, 5), 2, 4), ((7, 9, 5), 3, 6),
                                            ((64, 40, 130), 1, 8), ((64, 40, 130), 3, 70)])
def test_mode_multiply(dims, mode, rows):
    rng = np.random.default_rng(2)
    x = rng.standard_normal(dims)
    u = rng.standard_normal((rows, dims[mode - 1]))
    got = bt.mode_multiply(x, mode, u)
    np.testing.assert_allclose(got, port.mode_multiply(x, mode, u), rtol=0,
                               atol=1e-12 * np.abs(got).max())


@pytest.mark.parametrize("dims,rows", [((9, 31, 64), 34), ((5, 130, 48), 64), ((3, 77, 250), 70),
                                       ((2, 300, 18), 96), ((4, 50, 33), 64), ((1, 1, 16), 40)])
def test_last_mode_product_on_tree_kernel_matches_oracle_and_engine(dims, rows, monkeypatch):
    """x x_3 u^T with u given as (K, rows), rows > 32 (tensor.py:75-90): the
    TMA tree kernel without its reduction epilogue for even K and rows, the
    cp.async engine otherwise (odd K: (4, 50, 33)) -- both against the
    oracle, ragged row counts and a K below one k-tile included."""
    from paper_2105_01170_b200.tensor import ttm_dev

    rng = np.random.default_rng(sum(dims) + rows)
    x = rng.standard_normal(dims)
    u = rng.standard_normal((dims[2], rows))
    want = port.mode_multiply(x, 3, u.T)
    xd, ud = torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda()
    got = ttm_dev(xd, 3, ud, rows, transpose=True).cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 * np.abs(want).max())
    # a (rows, K) factor (no transpose flag) and a view at an odd offset take the engine
    got2 = ttm_dev(xd, 3, ud.t().contiguous(), rows).cpu().numpy()
    np.testing.assert_allclose(got2, want, rtol=0, atol=1e-12 * np.abs(want).max())
    pad = torch.zeros(x.size + 1, dtype=torch.float64, device="cuda")
    pad[1:] = xd.reshape(-1)
    got3 = ttm_dev(pad[1:].view(*dims), 3, ud, rows, transpose=True).cpu().numpy()
    np.testing.assert_allclose(got3, want, rtol=0, atol=1e-12 * np.abs(want).max())


# ---------------------------------------------------------------------------
# K1 / K2 maps: bit-exact against the reference's golden vectors
# ---------------------------------------------------------------------------

def test_gather_scatter_bit_exact(golden):
    z = golden("maps")
    for c in range(int(z["n_cases"])):
        k = f"c{c}"
        pat = pattern_from(z[k + "_cells"], z[k + "_offs"], z[k + "_dims"])
        a = z[k + "_a"]
        assert np.array_equal(bt.mat_to_tensor(a, pat), z[k + "_t"])
        assert np.array_equal(bt.mat_to_tensor(a, pat, weighted=False), z[k + "_tu"])
        assert np.array_equal(bt.tensor_to_mat(z[k + "_t"], pat), z[k + "_back"])
        assert np.array_equal(bt.struct_scalars(pat, z[k + "_coeffs"]), z[k + "_scalars"])
        blocks = bt.extract_blocks(a, pat)
        assert np.array_equal(bt.struct_assemble(pat, blocks), a)


def test_gather_rejects_like_the_reference():
    rng = np.random.default_rng(4)
    pat = bt.build_pattern("toeplitz", 3, 3, 2, 2)
    a = bt.struct_assemble(pat, [rng.standard_normal((2, 2)) for _ in range(pat.p)])
    bad = a.copy()
    bad[-1, -1] += 1.0
    with pytest.raises(bt.PatternMismatchError, match=r"class 1: block at grid cell \(3, 3\)"):
        bt.mat_to_tensor(bad, pat)
    diag = bt.build_pattern("diagonal", 2, 2, 2, 2)
    b = bt.struct_assemble(diag, [rng.standard_normal((2, 2)) for _ in range(diag.p)])
    b[0, -1] = 1.0
    with pytest.raises(bt.PatternMismatchError, match=r"grid cell \(1, 2\) is outside"):
        bt.extract_blocks(b, diag)
    # numpy NaN semantics: a NaN difference masks the cell (np.max -> NaN > tol is False)
    c = a.copy()
    c[-1, -1] = np.nan
    c[-2, -2] += 5.0
    t = bt.mat_to_tensor(c, pat)
    assert t.shape == (2, pat.p, 2)
    # tolerance
    d = a.copy()
    d[-1, -1] += 1e-9
    bt.mat_to_tensor(d, pat, tol=1e-8)


# ---------------------------------------------------------------------------
# CP-ALS
# ---------------------------------------------------------------------------

def test_cp_c1_matches_reference(golden):
    z = golden("cp")
    pat, a = oc.c1_inputs()
    t = bt.mat_to_tensor(a, bt.build_pattern("toeplitz", 32, 32, 32, 32, block_symmetric=True))
    assert np.array_equal(t, z["c1_t"])
    saved = with_init(oc.normal_init(t.shape, 8, 0))
    try:
        res = bt.cp_als(t, 8, 50, 0.0)
    finally:
        decomp._cp_init = saved
    np.testing.assert_allclose(np.array(res.fit_history), z["c1_hist"], rtol=0, atol=1e-10)
    assert abs(res.fit - float(z["c1_fit"])) < 1e-10
    recon = port.mode_multiply  # noqa: F841
    got = np.einsum("ir,jr,kr->ijk", res.rep.x, res.rep.y, res.rep.z)
    ref = np.einsum("ir,jr,kr->ijk", z["c1_x"], z["c1_y"], z["c1_z"])
    assert np.linalg.norm(got - ref) <= 1e-8 * np.linalg.norm(ref)


@pytest.mark.parametrize("fit", ["auto", "explicit", "gram"])
def test_cp_mid_and_odd(golden, fit):
    z = golden("cp")
    for name in ("mid", "odd"):
        t = z[f"{name}_t"]
        r = int(z[f"{name}_r"])
        saved = with_init(oc.normal_init(t.shape, r, 5))
        try:
            res = bt.cp_als(t, r, int(z[f"{name}_iters"]), 0.0, fit=fit)
        finally:
            decomp._cp_init = saved
        np.testing.assert_allclose(np.array(res.fit_history), z[f"{name}_hist"], rtol=0,
                                   atol=1e-9)
        np.testing.assert_allclose(res.rep.x, z[f"{name}_x"], rtol=0, atol=1e-7)


def test_cp_rank1_exact_and_padded_init(golden):
    z = golden("cp")
    res = bt.cp_als(z["rank1_t"], 1)
    assert res.fit > 1 - 1e-13
    np.testing.assert_allclose(np.einsum("ir,jr,kr->ijk", res.rep.x, res.rep.y, res.rep.z),
                               z["rank1_t"], atol=1e-12)
    res = bt.cp_als(z["pad_t"], 4, max_iters=200)
    assert res.rep.x.shape == (2, 4)
    assert 0 < res.fit <= 1 + 1e-12
    assert abs(res.fit - float(z["pad_fit"])) < 1e-8


def test_cp_c5_small(golden):
    z = golden("cp")
    i, j, k, r = (int(v) for v in z["c5s_dims"])
    x = z["c5s_t"]
    saved = with_init(oc.normal_init((i, j, k), r, 1003))
    try:
        res = bt.cp_als(x, r, 10, 0.0)
    finally:
        decomp._cp_init = saved
    np.testing.assert_allclose(np.array(res.fit_history), z["c5s_hist"], rtol=0, atol=1e-9)


def test_cp_rejects_bad_args():
    with pytest.raises(ValueError):
        bt.cp_als(np.zeros((2, 2, 2)), 1)
    with pytest.raises(bt.ShapeError):
        bt.cp_als(np.zeros((2, 2)), 1)
    with pytest.raises(bt.ShapeError):
        bt.cp_als(np.ones((2, 2, 2)), 0)


# ---------------------------------------------------------------------------
# eigensolver / SVD / Tucker
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 7, 64, 96, 97, 200, 513])
def test_eigh(n):
    rng = np.random.default_rng(n)
    g = rng.standard_normal((n, n + 3))
    a = g @ g.T
    w, v = L.eigh_dev(torch.from_numpy(a).cuda())
    w, v = w.cpu().numpy(), v.cpu().numpy()
    ref = np.linalg.eigvalsh(a)[::-1]
    np.testing.assert_allclose(w, ref, rtol=0, atol=1e-11 * ref[0])
    np.testing.assert_allclose(v.T @ v, np.eye(n), atol=1e-12)
    np.testing.assert_allclose(a @ v, v * w, atol=1e-11 * ref[0])
    lead = np.argmax(np.abs(v), axis=0)
    assert np.all(v[lead, np.arange(n)] > 0)


def test_svd_truncated_sign_rule(golden):
    z = golden("tucker")
    u, s, v = bt.svd_truncated(z["svd_a"], 3)
    np.testing.assert_allclose(u, z["svd_u"], atol=1e-12)
    np.testing.assert_allclose(s, z["svd_s"], atol=1e-12)
    np.testing.assert_allclose(v, z["svd_v"], atol=1e-12)


@pytest.mark.parametrize("shape", [(40, 300), (300, 40), (64, 64)])
def test_svd_truncated_both_sides_vs_oracle(shape):
    """Gram of the short side either way; the sign rule lands on u and is
    compensated in v (decomp.py:176-179), as in the oracle's LAPACK SVD."""
    rng = np.random.default_rng(sum(shape))
    m, n = shape
    a = rng.standard_normal((m, 6)) @ np.diag(10.0 ** -np.arange(6)) @ rng.standard_normal((6, n))
    a += 1e-7 * rng.standard_normal((m, n))
    u, s, v = bt.svd_truncated(a, 4)
    uo, so, vo = port.svd_trunc(a, 4)
    np.testing.assert_allclose(s, so, rtol=1e-10)
    np.testing.assert_allclose(u, uo, atol=1e-9)
    np.testing.assert_allclose(v, vo, atol=1e-9)


def test_hosvd_golden(golden):
    z = golden("tucker")
    for n in range(int(z["n_hosvd"])):
        rep = bt.hosvd(z[f"h{n}_t"], [int(v) for v in z[f"h{n}_ranks"]])
        np.testing.assert_allclose(rep.core, z[f"h{n}_core"], atol=1e-12)
        for k in range(3):
            np.testing.assert_allclose(rep.factors[k], z[f"h{n}_u{k}"], atol=1e-12)


@pytest.mark.parametrize("shape,ranks", [((20, 130, 12), (20, 40, 12)), ((8, 12, 200), (5, 12, 30)),
                                         ((120, 9, 110), (30, 9, 25))])
def test_hosvd_side_stream_modes_match_serial_and_oracle(shape, ranks, monkeypatch):
    """hosvd (decomp.py:237-259) with short and long modes mixed: the short
    modes' first pass runs on a side stream beside the long modes; factors and
    core are bit-identical to the serial order (BT_HOSVD_SIDE=0 path) and
    match the oracle's HOSVD (numpy and device input)."""
    from paper_2105_01170_b200 import decomp

    rng = np.random.default_rng(sum(shape))
    g = rng.standard_normal(ranks)
    us = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in zip(shape, ranks)]
    t = np.einsum("abc,ia,jb,kc->ijk", g, *us) + 1e-3 * rng.standard_normal(shape)
    rep = bt.hosvd(t, list(ranks))
    monkeypatch.setattr(decomp, "_SIDE_MODES", False)
    ser = bt.hosvd(t, list(ranks))
    monkeypatch.setattr(decomp, "_SIDE_MODES", True)
    dev = bt.hosvd(torch.from_numpy(t).cuda(), list(ranks))
    assert np.array_equal(rep.core, ser.core)
    assert np.array_equal(dev.core.cpu().numpy(), ser.core)
    for a, b in zip(rep.factors, ser.factors):
        assert np.array_equal(a, b)
    core_o, fac_o = port.hosvd(t, list(ranks))
    np.testing.assert_allclose(rep.core, core_o, atol=1e-8)
    for a, b in zip(rep.factors, fac_o):
        np.testing.assert_allclose(a, b, atol=1e-8)


@pytest.mark.parametrize("n", [1, 2, 5, 17, 31, 32])
def test_svd_small_vs_numpy(n):
    """bt_svd_small_f64 (the np.linalg.svd of decomp.py:172 on the projected
    factor of a basis refinement): graded and random matrices -- singular
    values against LAPACK's (absolute accuracy eps sigma_1), m = u diag(s) v^T,
    orthonormal factors, the sign rule of decomp.py:176-179, bit-reproducible."""
    rng = np.random.default_rng(n)
    q1, _ = np.linalg.qr(rng.standard_normal((n, n)))
    q2, _ = np.linalg.qr(rng.standard_normal((n, n)))
    graded = (q1 * 10.0 ** (-np.linspace(0, 11, n))) @ q2.T
    for m in (rng.standard_normal((n, n)), graded, np.diag(np.arange(n, 0, -1.0)), np.zeros((n, n))):
        md = torch.from_numpy(np.ascontiguousarray(m)).cuda()
        u, sv, v = L.svd_small_dev(md)
        u2, sv2, v2 = L.svd_small_dev(md)
        assert torch.equal(u, u2) and torch.equal(sv, sv2) and torch.equal(v, v2)
        u, sv, v = u.cpu().numpy(), sv.cpu().numpy(), v.cpu().numpy()
        ref = np.linalg.svd(m, compute_uv=False)
        assert np.all(np.diff(sv) <= 0)
        scale = max(ref[0], 1e-300)
        np.testing.assert_allclose(sv, ref, rtol=0, atol=1e-14 * scale)
        np.testing.assert_allclose((u * sv) @ v.T, m, rtol=0, atol=1e-14 * scale)
        np.testing.assert_allclose(v.T @ v, np.eye(n), atol=1e-13)
        live = sv > 1e-13 * scale
        uu = u[:, live]
        np.testing.assert_allclose(uu.T @ uu, np.eye(uu.shape[1]), atol=1e-12)
        for c in range(uu.shape[1]):
            assert uu[np.argmax(np.abs(uu[:, c])), c] > 0


@pytest.mark.parametrize("R", [3, 8, 16, 33, 64, 96])
def test_pinv_sym_vs_numpy(R):
    """bt_pinv_sym_f64 (decomp.py:387 np.linalg.pinv of the Hadamard Gram):
    well-conditioned SPD (Cholesky path), rank-deficient PSD (eigen path with
    numpy's 1e-15 cutoff) across the NP size classes."""
    from paper_2105_01170_b200 import _dev
    from paper_2105_01170_b200 import _native as N

    rng = np.random.default_rng(R)
    g = rng.standard_normal((R, 2 * R))
    cases = [g @ g.T]
    h = rng.standard_normal((R, max(1, R // 2)))
    cases.append(h @ h.T)                       # rank R/2: pinv != inverse
    for v in cases:
        vd = torch.from_numpy(v).cuda()
        out = torch.empty_like(vd)
        N.call("bt_pinv_sym_f64", _dev.ptr(vd), R, _dev.ptr(out), _dev.stream())
        ref = np.linalg.pinv(v)
        err = np.abs(out.cpu().numpy() - ref).max() / np.abs(ref).max()
        assert err < 1e-9, (R, err)


@pytest.mark.parametrize("shape,cond", [((4096, 64), 1e2), ((2047, 96), 1e4), ((300, 40), 1e9),
                                        ((50, 5), 1e1)])
def test_qr_thin_vs_numpy(shape, cond):
    """decomp.py:182-193 thin QR (diag R >= 0): CholeskyQR2 for moderate
    conditioning, Householder fallback beyond (cond 1e9 case)."""
    rng = np.random.default_rng(int(cond))
    m, n = shape
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (u * np.logspace(0, -np.log10(cond), n)) @ v.T
    q, r = bt.qr_thin(a)
    qo, ro = np.linalg.qr(a)
    sg = np.sign(np.diag(ro))
    sg[sg == 0] = 1
    qo, ro = qo * sg, ro * sg[:, None]
    assert np.all(np.diag(r) >= 0)
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-12
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.abs(r - ro).max() <= 1e-12 * cond * np.abs(ro).max()


# ---------------------------------------------------------------------------
# fused one-CTA CP-ALS (SM-sized tensors) vs the phase kernels
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dims,r,fit", [((32, 32, 32), 8, "auto"), ((7, 19, 11), 5, "explicit"),
                                        ((40, 9, 33), 13, "gram"), ((16, 16, 64), 16, "auto"),
                                        ((5, 6, 7), 1, "auto")])
def test_cp_fused_small_matches_phase_kernels(dims, r, fit):
    """cp_als on a tensor that fits one SM runs cp_small_kernel (one launch
    for all sweeps); the phase C-ABI (bt_cp_*) runs the multi-kernel sweep.
    Same fit histories, factors and weights (different summation orders)."""
    from paper_2105_01170_b200 import _dev
    from paper_2105_01170_b200.parallel import NativeCpOps, cp_als_sharded

    rng = np.random.default_rng(sum(dims) + r)
    x = rng.standard_normal(dims)
    init = oc.normal_init(dims, r, 7)
    iters = 12
    saved = with_init(init)
    try:
        res = bt.cp_als(x, r, iters, 0.0, fit=fit)
    finally:
        decomp._cp_init = saved
    xd = torch.from_numpy(x).cuda()
    f = [torch.from_numpy(v.copy()).cuda() for v in init]
    ops = NativeCpOps(xd, r, f[0], f[1], f[2], iters, fit=fit)
    hist, n, conv = cp_als_sharded(ops, iters, 0.0, lambda b: None)
    ops.close()
    np.testing.assert_allclose(res.fit_history, hist, rtol=0, atol=1e-11)
    ref = port.cp_als(x, r, iters, 0.0, init=lambda _t, _r: [v.copy() for v in init])
    np.testing.assert_allclose(res.fit_history, ref.fit_history, rtol=0, atol=1e-10)
    assert res.n_iters == iters and not res.converged
    assert _dev.is_device(res.rep.x) is False


def test_cp_fused_small_tol_stops_like_reference():
    """tol > 0: the in-kernel |fit - prev| < tol test stops at the same sweep
    as decomp.py:398-401 (oracle restatement)."""
    rng = np.random.default_rng(3)
    a, b, c = (rng.standard_normal((n, 3)) for n in (12, 10, 9))
    x = np.einsum("ir,jr,kr->ijk", a, b, c) + 1e-3 * rng.standard_normal((12, 10, 9))
    init = oc.normal_init(x.shape, 3, 11)
    saved = with_init(init)
    try:
        res = bt.cp_als(x, 3, 200, 1e-9)
    finally:
        decomp._cp_init = saved
    ref = port.cp_als(x, 3, 200, 1e-9, init=lambda _t, _r: [v.copy() for v in init])
    assert res.converged == ref.converged and res.n_iters == ref.n_iters
    np.testing.assert_allclose(res.fit_history, ref.fit_history, rtol=0, atol=1e-10)


# ---------------------------------------------------------------------------
# leading eigenpairs of a deflation pass (bt_leading_subspace_f64)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n,need,decay", [(300, 20, 8.0), (600, 64, 3.0), (257, 5, 14.0)])
def test_leading_subspace_vs_numpy(n, need, decay):
    rng = np.random.default_rng(n + need)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-decay * np.linspace(0, 1, n) ** 0.5)
    g = (q * lam) @ q.T
    g = (g + g.T) / 2
    gd = torch.from_numpy(g).cuda()
    out = L._leading_subspace(gd, need, 1e-6)
    if out is None:          # predicted too slow: the caller's tridiagonal fallback
        w, v = L.eigh_dev(gd, nvec=need, tau=1e-6)
        k = need
    else:
        w, v, k = out
    w, v = w.cpu().numpy(), v.cpu().numpy()
    assert k >= 1
    ref_w, ref_v = np.linalg.eigh(g)
    ref_w, ref_v = ref_w[::-1], ref_v[:, ::-1]
    np.testing.assert_allclose(w[:k], ref_w[:k], rtol=0, atol=64 * 2.2e-16 * ref_w[0])
    # accepted vectors: residual-certified, orthonormal, sign rule applied
    vk = v[:, :k]
    assert np.abs(vk.T @ vk - np.eye(k)).max() < 1e-12
    res = np.linalg.norm(g @ vk - vk * w[:k], axis=0)
    assert res.max() <= 40 * 2.2e-16 * ref_w[0]
    idx = np.argmax(np.abs(vk), axis=0)
    assert np.all(vk[idx, np.arange(k)] > 0)


def test_leading_subspace_warm_start_and_shape_guard():
    rng = np.random.default_rng(5)
    n = 400
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-40 * np.linspace(0, 1, n))   # 10^-0.1 per index: a fast block edge
    g = (q * lam) @ q.T
    g = (g + g.T) / 2
    gd = torch.from_numpy(g).cuda()
    w0, v0, k0 = L._leading_subspace(gd, 30, 1e-6)
    # warm start with the answer: converges to the same pairs
    w1, v1, k1 = L._leading_subspace(gd, 30, 1e-6, start=v0[:, :k0].contiguous())
    kk = min(k0, k1)
    assert subspace_angle(v0[:, :kk].cpu().numpy(), v1[:, :kk].cpu().numpy()) < 1e-10
    # a block wider than n / 2 is not applicable (status 2 -> None)
    small = torch.from_numpy(g[:40, :40].copy()).cuda()
    assert L._leading_subspace(small, 30, 1e-6) is None


@pytest.mark.parametrize("shape", [(37, 1000), (1, 5), (1025, 33), (4096, 32), (64, 64)])
def test_transpose_kernel(shape):
    """bt_transpose_f64 (the matvec RHS layout flip) is an exact transpose,
    ragged tile edges included."""
    from paper_2105_01170_b200 import _dev

    x = torch.from_numpy(np.random.default_rng(shape[0]).standard_normal(shape)).cuda()
    y = _dev.transpose(x)
    assert tuple(y.shape) == shape[::-1]
    assert torch.equal(y.cpu(), x.cpu().T)
