"""Pin the CPU oracle (oracle/port.py) to golden vectors produced by the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import configs as oc
from oracle import port

from conftest import GOLDEN


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _flat(pat):
    cells = np.vstack(pat.placements) if pat.p else np.zeros((0, 2), np.int64)
    return cells.astype(np.int64), np.cumsum([0] + list(pat.counts)).astype(np.int64)


def _pattern_from(cells, offs, dims):
    ell, q, m, n = (int(v) for v in dims)
    pl = tuple(cells[offs[k]:offs[k + 1]] for k in range(len(offs) - 1))
    return port.Pattern(ell, q, m, n, pl)


def test_small_patterns_bit_exact(golden):
    meta = json.load(open(os.path.join(GOLDEN, "patterns.json")))
    z = golden("patterns")
    for idx, spec in enumerate(meta["small"]):
        pat = port.make_pattern(spec["kind"], spec["ell"], spec["ell"], 2, 3,
                                band=spec["band"], block_symmetric=spec["sym"])
        cells, offs = _flat(pat)
        assert np.array_equal(cells, z[f"cells_{idx}"]), spec
        assert np.array_equal(offs, z[f"offs_{idx}"]), spec
        assert pat.structure_class == spec["tag"]


def test_config_patterns_bit_exact():
    meta = json.load(open(os.path.join(GOLDEN, "patterns.json")))
    for spec in meta["big"]:
        if spec["kind"] == "kernel_level":
            pat = port.kernel_level_pattern(spec["ell"], 1, 1)
        else:
            pat = port.make_pattern(spec["kind"], spec["ell"], spec["ell"], spec["m"], spec["n"],
                                    block_symmetric=spec["sym"])
        cells, offs = _flat(pat)
        assert pat.p == spec["p"]
        assert _sha(cells) == spec["cells_sha"] and _sha(offs) == spec["offs_sha"], spec


def test_gather_scatter_golden(golden):
    z = golden("maps")
    for c in range(int(z["n_cases"])):
        k = f"c{c}"
        pat = _pattern_from(z[k + "_cells"], z[k + "_offs"], z[k + "_dims"])
        a = z[k + "_a"]
        assert np.array_equal(port.gather(a, pat), z[k + "_t"])
        assert np.array_equal(port.gather(a, pat, weighted=False), z[k + "_tu"])
        assert np.array_equal(port.scatter(z[k + "_t"], pat), z[k + "_back"])
        assert np.array_equal(port.scalars(pat, z[k + "_coeffs"]), z[k + "_scalars"])


def test_cp_als_golden(golden):
    z = golden("cp")
    res = port.cp_als(z["rank1_t"], 1)
    assert res.fit == z["rank1_fit"] and res.n_iters == z["rank1_iters"]
    res = port.cp_als(z["pad_t"], 4, max_iters=200)
    np.testing.assert_array_equal(np.array(res.fit_history), z["pad_hist"])
    init = port.cp_init_hosvd(z["pad_t"], 4)
    for k in range(3):
        np.testing.assert_array_equal(init[k], z[f"pad_init{k}"])
    pat, a = oc.c1_inputs()
    assert _sha(a) == str(z["c1_a_sha"])
    t = port.gather(a, pat)
    np.testing.assert_array_equal(t, z["c1_t"])
    res = port.cp_als(t, 8, 50, 0.0, init=port.cp_init_normal(0))
    np.testing.assert_array_equal(np.array(res.fit_history), z["c1_hist"])
    for name in ("mid", "odd"):
        r = int(z[f"{name}_r"])
        res = port.cp_als(z[f"{name}_t"], r, int(z[f"{name}_iters"]), 0.0,
                          init=port.cp_init_normal(5))
        np.testing.assert_array_equal(np.array(res.fit_history), z[f"{name}_hist"])
        np.testing.assert_array_equal(res.x, z[f"{name}_x"])


def test_c5_generator_and_slabs(golden):
    z = golden("cp")
    i, j, k, r = (int(v) for v in z["c5s_dims"])
    x = oc.c5_tensor(i, j, k, r)
    np.testing.assert_array_equal(x, z["c5s_t"])
    slab = oc.c5_tensor(i, j, k, r, k_slab=(8, 20))
    np.testing.assert_array_equal(slab, x[:, :, 8:20])
    res = port.cp_als(x, r, 10, 0.0, init=port.cp_init_normal(1003))
    np.testing.assert_allclose(np.array(res.fit_history), z["c5s_hist"], rtol=0, atol=1e-13)


def test_tucker_golden(golden):
    z = golden("tucker")
    for n in range(int(z["n_hosvd"])):
        core, fac = port.hosvd(z[f"h{n}_t"], [int(v) for v in z[f"h{n}_ranks"]])
        np.testing.assert_array_equal(core, z[f"h{n}_core"])
        for k in range(3):
            np.testing.assert_array_equal(fac[k], z[f"h{n}_u{k}"])
    u, s, v = port.svd_trunc(z["svd_a"], 3)
    np.testing.assert_array_equal(u, z["svd_u"])
    np.testing.assert_array_equal(port.mode_basis(z["mb_a"], 5), z["mb_u"])
    pat, t = oc.c2_tensor(z["c2s_params"])
    np.testing.assert_array_equal(t, z["c2s_t"])
    core, fac = port.hosvd(t, [8, 40, 8])
    np.testing.assert_array_equal(core, z["c2s_core"])
    left, right, mids = port.blr_from_tucker(core, fac, pat.m, pat.n)
    np.testing.assert_array_equal(mids, z["c2s_mid"])
    for c in range(z["c2s_rhs"].shape[1]):
        y = port.matvec_blr(pat, left, right, mids, z["c2s_rhs"][:, c])
        np.testing.assert_allclose(y, z["c2s_mv"][:, c], rtol=0, atol=1e-14)
    yf = port.matvec_blr_fast(pat, left, right, mids, z["c2s_rhs"])
    np.testing.assert_allclose(yf, z["c2s_mv"], rtol=0, atol=1e-13)
    pat3, blocks3, t3 = oc.c3_tensor(side=6, lags=10)
    np.testing.assert_array_equal(t3, z["c3s_t"])
    core, fac = port.tucker_partial(t3, [8, 4, 8], shared=(1, 3))
    np.testing.assert_array_equal(core, z["c3s_core"])
    u, proj = port.spsd_blocks(pat3, blocks3, 8)
    np.testing.assert_array_equal(u, z["c3s_spsd_u"])
    np.testing.assert_array_equal(proj, z["c3s_spsd_blocks"])


def test_st_hosvd_reduces_to_partial_tucker(golden):
    """SURVEY 8c anchor: ST-HOSVD's shared mode-1 step == tucker_partial(shared=(1,3))."""
    z = golden("tucker")
    core, fac = port.st_hosvd_shared13(z["c3s_t"], 8, 4)
    np.testing.assert_array_equal(fac[0], z["c3s_u"])
    # HOOI with zero sweeps is the ST-HOSVD result; sweeps never increase the error
    t = z["c3s_t"]
    err0 = np.linalg.norm(t - port.mode_multiply(port.mode_multiply(port.mode_multiply(
        core, 1, fac[0]), 2, fac[1]), 3, fac[2]))
    core2, fac2 = port.hooi_shared13(t, fac[0], fac[1], 3)
    err1 = np.linalg.norm(t - port.mode_multiply(port.mode_multiply(port.mode_multiply(
        core2, 1, fac2[0]), 2, fac2[1]), 3, fac2[2]))
    assert err1 <= err0 * (1 + 1e-12)


def test_reps_and_matvec_golden(golden):
    z = golden("reps")
    for c in range(int(z["n_cases"])):
        k = f"r{c}"
        pat = _pattern_from(z[k + "_cells"], z[k + "_offs"], z[k + "_dims"])
        fac = [z[k + "_u"], z[k + "_v"], z[k + "_w"]]
        coeffs, terms = port.kron_from_tucker(z[k + "_core"], fac, pat.p)
        np.testing.assert_array_equal(coeffs, z[k + "_kc"])
        np.testing.assert_array_equal(terms, z[k + "_kt"])
        left, right, mids = port.blr_from_tucker(z[k + "_core"], fac, pat.m, pat.n)
        np.testing.assert_array_equal(mids, z[k + "_bm"])
        # the reference sums C_j through scipy CSR; the oracle through a dense
        # C_j -- same products, different summation order
        yk = z[k + "_yk"]
        np.testing.assert_allclose(port.matvec_kron(pat, coeffs, terms, z[k + "_x"]), yk,
                                   rtol=0, atol=1e-14 * max(1.0, np.abs(yk).max()))
        np.testing.assert_array_equal(port.matvec_blr(pat, left, right, mids, z[k + "_x"]), z[k + "_yb"])
        np.testing.assert_array_equal(port.densify_kron(pat, coeffs, terms), z[k + "_dk"])
        fc, ft = port.kron_from_kruskal(z[k + "_cx"], z[k + "_cy"], z[k + "_cz"])
        np.testing.assert_array_equal(fc, z[k + "_kfc"])
        np.testing.assert_array_equal(ft, z[k + "_kft"])
        if k + "_kqc" in z:
            qc, qt = port.kron_from_kruskal(z[k + "_cx"], z[k + "_cy"], z[k + "_cz"], split="qr")
            np.testing.assert_array_equal(qc, z[k + "_kqc"])
            np.testing.assert_array_equal(qt, z[k + "_kqt"])


def test_psf_and_multilevel_golden(golden):
    z = golden("psf")
    for k in (3, 5, 7):
        x = port.psf_weighted(z[f"psf{k}"])
        np.testing.assert_array_equal(x, z[f"x{k}"][0, :, :, :, 0])
    np.testing.assert_array_equal(oc.c4_psf(7), z["c4s_psf"])
    t = z["c4s_x"][0, :, :, :, 0]
    res = port.cp_als(t, 3, 30, 0.0, init=port.cp_init_normal(2))
    np.testing.assert_array_equal(np.array(res.fit_history), z["c4s_hist"])
    levels = [port.kernel_level_pattern(7, 49, 49), port.kernel_level_pattern(7, 7, 7),
              port.kernel_level_pattern(7, 1, 1)]
    terms = port.ml_kron_from_kruskal(levels, z["c4s_cx"], z["c4s_cy"], z["c4s_cz"])
    vols = z["c4s_vols"].T.reshape(3, 7, 7, 7)
    y = port.ml_matvec(terms, vols).reshape(3, -1).T
    np.testing.assert_allclose(y, z["c4s_mv"], rtol=0, atol=1e-13 * np.abs(z["c4s_mv"]).max())
    # generalised grid == K reduces to the reference weighting
    np.testing.assert_array_equal(port.psf_weighted(z["psf5"], 5), z["x5"][0, :, :, :, 0])


def test_spd_compress_golden(golden):
    """oracle spd_compress / cholesky vs the reference (psd.py:205-271)."""
    z = golden("spd")
    for case, (seed, ell, nb) in enumerate(((21, 4, 5), (22, 3, 8), (23, 6, 3))):
        pat, a = oc.spd_toeplitz(seed, ell, nb)
        assert np.array_equal(a, z[f"s{case}_a"])
        for r in range(1, nb + 1):
            low, cells, u, proj = port.spd_compress(a, pat, r)
            dense = port.densify_spd(pat, low, cells, u, proj)
            ref = z[f"s{case}_r{r}_dense"]
            assert np.linalg.norm(dense - ref) <= 1e-12 * np.linalg.norm(ref)
            if r == 1:
                assert np.array_equal(low, z[f"s{case}_chol"])
                assert np.array_equal(np.concatenate(cells), z[f"s{case}_rem_cells"])
                assert [len(c) for c in cells] == list(z[f"s{case}_rem_counts"])
                assert port.classify_placements(tuple(cells), ell, ell) == str(
                    z[f"s{case}_rem_class"])
    assert np.array_equal(port.cholesky(z["chol_in"]), z["chol_out"])
    pat = port.Pattern(3, 3, 4, 4, (np.column_stack([np.arange(3)] * 2),))
    low, cells, u, proj = port.spd_compress(z["bd_a"], pat, 2)
    assert cells == []
    assert np.abs(port.densify_spd(pat, low, cells, u, proj) - z["bd_dense"]).max() < 1e-12


def test_detect_pattern_golden(golden):
    """oracle detect_pattern vs the reference (blocks.py:266-329), bit-exact."""
    z = golden("detect")
    meta = {d["name"]: d for d in json.load(open(os.path.join(GOLDEN, "detect.json")))}
    for name, a, m, n, tol in oc.detect_cases():
        pl, reps, cls = port.detect_pattern(a, m, n, tol)
        cells = np.vstack(pl).astype(np.int64)
        offs = np.cumsum([0] + [len(c) for c in pl]).astype(np.int64)
        assert np.array_equal(cells, z[f"{name}_cells"]), name
        assert np.array_equal(offs, z[f"{name}_offs"]), name
        assert np.array_equal(np.stack(reps).view(np.int64), z[f"{name}_reps"].view(np.int64)), name
        assert cls == meta[name]["structure_class"], name


def test_era_golden(golden):
    """oracle ERA vs the reference (apps.py:153-237): invariant quantities."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    z = golden("era")
    cases = (("full", 71, 6, 2, 2, 20, (2, 39, 2), 6, False),
             ("cut", 72, 5, 3, 2, 16, (3, 12, 2), 5, False),
             ("tera", 73, 4, 3, 3, 12, (2, 0, 2), 4, True),
             ("siso", 74, 2, 1, 1, 10, (1, 19, 1), 2, False))
    for name, seed, d, no, ni, s, ranks, order, tera in cases:
        a, b, c = oc.era_system(seed, d, no, ni)
        params = port.markov_from_lti(a, b, c, 2 * s - 1)
        assert np.allclose(params, z[f"{name}_params"], rtol=0, atol=1e-14)
        at, bt_, ct, sv, red, u, w = port.era_identify(params, ranks, order, tera)
        assert np.abs(sv - z[f"{name}_sv"]).max() <= 1e-12 * sv[0], name
        assert np.abs(red - z[f"{name}_reduced"]).max() <= 1e-12 * np.abs(red).max(), name
        mk = port.markov_from_lti(at, bt_, ct, 2 * s - 1)
        assert np.abs(mk - z[f"{name}_markov"]).max() <= 1e-10 * np.abs(mk).max(), name
