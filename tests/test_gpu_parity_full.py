"""Config-size parity against the UNMODIFIED reference (north_star tolerances).

Fixtures: ``tests/golden/make_golden_big.py`` ran the reference in the build
container at the configs' own sizes and ranks (big_c3, big_c4, big_c5,
mltucker .npz).  Here the product runs the same seeded inputs on the B200
and is compared with them; where a fixture keeps only samples, the full
output is also compared with the CPU oracle (oracle/port.py, pinned to the
reference by tests/test_oracle_golden.py) on the box's host.

Tolerances (BASELINE.json north_star): Tucker subspaces <= 1e-8 principal
angle (on the leading block that a spectral gap makes well defined, SURVEY
H4), reconstructed operators and matvec outputs <= 1e-10 relative Frobenius,
relative approximation errors (1 - fit) <= 1e-8 absolute.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_01170_b200 as bt  # noqa: E402
from paper_2105_01170_b200 import configs, decomp, multilevel, psd, reconstruct  # noqa: E402
from paper_2105_01170_b200.blocks import build_pattern, kernel_level_pattern  # noqa: E402
from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402

from _helpers import subspace_angle  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def host(v):
    return v.cpu().numpy() if torch.is_tensor(v) else np.asarray(v)


def gapped_lead(sv, r, gap=1e-6):
    """Largest k <= r whose leading k-dimensional singular subspace is defined
    to ~1e-10 in double precision: sigma_k - sigma_{k+1} >= gap * sigma_1
    (a computed basis resolves it to ~eps * sigma_1 / gap)."""
    best = 0
    for k in range(1, r + 1):
        nxt = sv[k] if k < len(sv) else 0.0
        if sv[k - 1] - nxt >= gap * sv[0]:
            best = k
    return best


# ---------------------------------------------------------------------------
# ml_kron_sum_from_tucker (multilevel.py:197-225): the Tucker route
# ---------------------------------------------------------------------------


def _ref_level(k, bm, bn, grid):
    return kernel_level_pattern(k, bm, bn, grid)


def _mlt_patterns():
    inner = build_pattern("banded", 3, 3, 2, 2, band=1)
    outer = build_pattern("hankel", 2, 2, inner.shape[0], inner.shape[1])
    t_in = build_pattern("toeplitz", 3, 3, 2, 3)
    t_out = build_pattern("toeplitz", 2, 2, t_in.shape[0], t_in.shape[1], block_symmetric=True)
    return {"hb": multilevel.MultilevelPattern(levels=(outer, inner)),
            "psf": multilevel.MultilevelPattern(levels=(_ref_level(5, 16, 16, 4),
                                                        _ref_level(5, 4, 4, 4),
                                                        _ref_level(5, 1, 1, 4))),
            "tt": multilevel.MultilevelPattern(levels=(t_out, t_in))}


@pytest.mark.parametrize("case", ["hb", "psf", "tt"])
@pytest.mark.parametrize("variant", ["full", "ident"])
def test_ml_kron_sum_from_tucker_golden(golden, case, variant):
    z = golden("mltucker")
    key = f"{case}_{variant}"
    mlp = _mlt_patterns()[case]
    core = z[key + "_core"]
    facs = []
    for i in range(len(mlp.dims)):
        f = z[key + f"_f{i}"]
        facs.append(None if f.size == 0 else torch.from_numpy(f).cuda())
    tk = bt.TuckerRep(core=torch.from_numpy(core).cuda(), factors=tuple(facs))
    terms = multilevel.ml_kron_sum_from_tucker(tk, mlp)
    assert len(terms) == int(z[key + "_nterms"])
    dense = 0.0
    for j, tm in enumerate(terms):
        for lvl, m in enumerate(tm.level_mats):
            # struct_scalars: c_k / sqrt(eta_k) on the cells -- bit-exact
            assert np.array_equal(host(m), z[key + f"_t{j}_l{lvl}"]), (j, lvl)
        b_ref = z[key + f"_t{j}_b"]
        assert rel(host(tm.block), b_ref) <= 1e-13 or np.abs(host(tm.block) - b_ref).max() < 1e-14
        dense = dense + host(tm.densify())
    if key + "_dense" in z:
        assert rel(dense, z[key + "_dense"]) < 1e-13
    if case == "psf" and variant == "full":
        # 1 x 1 innermost blocks: the Tucker-route terms drive the multilevel
        # matvec, which must equal the reference's densified operator
        xs = np.random.default_rng(5).standard_normal((dense.shape[1], 3))
        y = multilevel.ml_matvec(terms, torch.from_numpy(xs).cuda())
        assert rel(host(y), z[key + "_dense"] @ xs) < 1e-12


# ---------------------------------------------------------------------------
# C4 at full size: the 128^3 multilevel matvec of the reference's factors
# ---------------------------------------------------------------------------


def test_c4_full_ml_matvec_vs_reference(golden):
    z = golden("big_c4")
    k, grid, r = 255, 128, 16
    _, mlp = multilevel.psf_weighted_tensor(torch.from_numpy(oc.c4_psf(k)).cuda(), grid=grid)
    kr = bt.KruskalRep(x=torch.from_numpy(z["x"]).cuda(), y=torch.from_numpy(z["y"]).cuda(),
                       z=torch.from_numpy(z["z"]).cuda())
    terms = multilevel.ml_kron_sum_from_kruskal(kr, mlp)
    # the reference's struct_scalars level matrices (Toeplitz: first column + row)
    for t, tm in enumerate(terms):
        for lvl in range(3):
            m = host(tm.level_mats[lvl])
            assert np.array_equal(m[:, 0], z["col"][t, lvl]) and np.array_equal(m[0, :], z["row"][t, lvl])
    vols = np.random.default_rng(1004).standard_normal((grid**3, 32))
    y = host(multilevel.ml_matvec(terms, torch.from_numpy(vols).cuda()))
    assert rel(y[::61, :4], z["y_sampled"]) < 1e-10
    np.testing.assert_allclose(np.linalg.norm(y[:, :4], axis=0), z["y_norms"], rtol=1e-12)
    # every entry of the 4 volumes against the oracle's restated matvec
    levels = [port.kernel_level_pattern(k, grid * grid, grid * grid, grid),
              port.kernel_level_pattern(k, grid, grid, grid), port.kernel_level_pattern(k, 1, 1, grid)]
    to = port.ml_kron_from_kruskal(levels, z["x"], z["y"], z["z"])
    yo = port.ml_matvec(to, vols[:, :4].T.reshape(4, grid, grid, grid)).reshape(4, -1).T
    assert rel(y[:, :4], yo) < 1e-10


# ---------------------------------------------------------------------------
# C5 recipe at 1024 x 1024 x 512, R = 64 (the headline rank)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("fit", ["auto", "explicit"])
def test_c5_r64_vs_reference(golden, fit):
    z = golden("big_c5")
    i, j, k, r, sweeps = (int(v) for v in z["dims"])
    x = configs.c5_build(i, j, k, r)
    assert abs(float(torch.linalg.norm(x)) / float(z["norm"]) - 1.0) < 1e-14
    init = oc.normal_init((i, j, k), r, 1003)
    saved = decomp._cp_init
    decomp._cp_init = lambda _t, _r: [torch.from_numpy(f).cuda() for f in init]
    try:
        res = bt.cp_als(x, r, sweeps, 0.0, fit=fit)
    finally:
        decomp._cp_init = saved
    del x
    torch.cuda.empty_cache()
    # north_star: relative errors agree within 1e-8 absolute (measured ~1e-13)
    np.testing.assert_allclose(res.fit_history, z["hist"], rtol=0, atol=1e-8)
    for got, ref in ((res.rep.x, z["x"]), (res.rep.y, z["y"]), (res.rep.z, z["z"])):
        assert rel(host(got), ref) < 1e-8


# ---------------------------------------------------------------------------
# C3 at full size (1024 x 512 x 1024): tucker_partial, SPSD, ST-HOSVD + HOOI,
# and the BLR operator of the (64, 32, 64) Tucker
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def c3_full():
    pat, t = configs.c3_build()
    yield pat, t
    del t
    torch.cuda.empty_cache()


def test_c3_full_tucker_partial_and_spsd_vs_reference(golden, c3_full):
    z = golden("big_c3")
    pat, t = c3_full
    sv = z["sv1"]
    lead = gapped_lead(sv, 64)
    assert lead >= 20, (lead, sv[:70] / sv[0])
    rep = bt.tucker_partial(t, [64, None, 64], shared=(1, 3))
    u = host(rep.factors[0])
    assert rep.factors[2] is rep.factors[0]
    assert subspace_angle(u[:, :lead], z["tp_u"][:, :lead]) < 1e-8
    # the compressed operator on the sampled lags: U core_k U^T (basis-free)
    sl = z["slices"]
    core = host(rep.core)
    for n, kk in enumerate(sl):
        got = u @ core[:, kk, :] @ u.T
        ref = z["tp_u"] @ z["tp_core_slices"][:, n, :] @ z["tp_u"].T
        assert rel(got, ref) < 1e-10, kk
    assert abs(np.linalg.norm(core) / float(z["tp_core_norm"]) - 1.0) < 1e-12
    del rep, core
    eta = torch.tensor(pat.counts, dtype=torch.float64, device="cuda")
    blocks = (t.permute(1, 0, 2) / eta.sqrt()[:, None, None]).contiguous()
    sp = psd.spsd_compress_blocks(pat, blocks, 64)
    del blocks
    ub = host(sp.basis)
    assert subspace_angle(ub[:, :lead], z["spsd_u"][:, :lead]) < 1e-8
    sb = host(sp.blocks)
    for n, kk in enumerate(sl):
        got = ub @ sb[kk] @ ub.T
        ref = z["spsd_u"] @ z["spsd_blocks_slices"][n] @ z["spsd_u"].T
        assert rel(got, ref) < 1e-10, kk
    assert abs(float(sp.trace()) / float(z["spsd_trace"]) - 1.0) < 1e-10


def test_c3_full_st_hosvd_hooi_and_blr_vs_reference(golden, c3_full):
    z = golden("big_c3")
    pat, t = c3_full
    lead = gapped_lead(z["sv1"], 64)
    st = decomp.st_hosvd(t, [64, 32, 64], shared=(1, 3))
    assert subspace_angle(host(st.factors[0])[:, :lead], z["st_u"][:, :lead]) < 1e-8
    h = decomp.hooi(t, st, 5, shared=(1, 3))
    u, v, core = host(h.factors[0]), host(h.factors[1]), host(h.core)
    assert subspace_angle(u[:, :lead], z["hooi_u"][:, :lead]) < 1e-8

    def recon(c, uu, vv):
        return port.mode_multiply(port.mode_multiply(port.mode_multiply(c, 1, uu), 2, vv), 3, uu)

    # the Tucker approximation itself, every entry (oracle arithmetic on the host)
    got = recon(core, u, v)
    ref = recon(z["hooi_core"], z["hooi_u"], z["hooi_v"])
    assert rel(got, ref) < 1e-10
    del got, ref
    # C3's second output: blr_from_tucker (reconstruct.py:229-240)
    # of the (64, 32, 64) Tucker, and its matvec on the seeded RHS
    blr = reconstruct.blr_from_tucker(h, pat)
    sl = z["slices"]
    mids = host(blr.middles)
    for n, kk in enumerate(sl):
        got = u @ mids[kk] @ u.T
        ref = z["hooi_u"] @ z["blr_mid_slices"][n] @ z["hooi_u"].T
        assert rel(got, ref) < 1e-10, kk
    rhs = np.random.default_rng(1003).standard_normal(pat.shape[1])
    y = host(reconstruct.matvec(blr, torch.from_numpy(rhs).cuda()))
    assert rel(y, z["blr_y"]) < 1e-10


# ---------------------------------------------------------------------------
# C2 at full size: the config's 64 right-hand sides
# ---------------------------------------------------------------------------


def test_c2_full_size_64_rhs():
    params = configs.c2_markov()
    pat, t = configs.c2_build(params)
    _, to = oc.c2_tensor(params)
    rep = bt.hosvd(t, [32, 400, 32])
    core_o, fac_o = port.hosvd(to, [32, 400, 32])
    blr = reconstruct.blr_from_tucker(rep, pat)
    left, right, mids = port.blr_from_tucker(core_o, fac_o, pat.m, pat.n)
    rhs = np.random.default_rng(1002).standard_normal((32768, 64))
    y = host(reconstruct.matvec(blr, torch.from_numpy(rhs).cuda()))
    yo = port.matvec_blr_fast(pat, left, right, mids, rhs)
    assert rel(y, yo) < 1e-10
    for c in range(64):
        assert rel(y[:, c], yo[:, c]) < 1e-10, c
