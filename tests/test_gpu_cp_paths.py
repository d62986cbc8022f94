"""GPU parity of the three single-GPU CP-ALS paths behind ``cp_als``
(decomp.py:344-410) against the CPU oracle and against each other:

* the cluster kernel (cp_cluster.cuh: SM-sized tensors, X resident in the
  distributed shared memory of 8 CTAs) and its one-CTA fallback;
* the small-rank two-pass path (cp_mid.cu: R <= 16 beyond one SM -- C4's
  shape class);
* the general phase kernels (cp.cu), reached with the switches off.

The switches (BT_CP_CLUSTER / BT_CP_SMALL / BT_CP_MID = 0) are read per call."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_01170_b200 as bt  # noqa: E402
from paper_2105_01170_b200 import decomp  # noqa: E402
from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402


def _low_rank(shape, r, seed, noise):
    rng = np.random.default_rng(seed)
    f = [rng.standard_normal((n, r)) for n in shape]
    return np.einsum("ir,jr,kr->ijk", *f) + noise * rng.standard_normal(shape)


def _run(x, r, iters, tol, fit, init, **env):
    saved_env = {k: os.environ.get(k) for k in env}
    saved = decomp._cp_init
    decomp._cp_init = lambda _t, _r: [v.copy() for v in init]
    os.environ.update(env)
    try:
        return bt.cp_als(x, r, iters, tol, fit=fit)
    finally:
        decomp._cp_init = saved
        for k, v in saved_env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def _check(res, ref, tol_hist=1e-10, tol_fac=1e-9):
    assert res.n_iters == ref.n_iters and res.converged == ref.converged
    np.testing.assert_allclose(res.fit_history, ref.fit_history, rtol=0, atol=tol_hist)
    assert _rel(res.rep.x, ref.x) < tol_fac
    assert _rel(res.rep.y, ref.y) < tol_fac
    assert _rel(res.rep.z, ref.z) < tol_fac


# ---------------------------------------------------------------------------
# cluster kernel and its one-CTA fallback (SM-sized tensors)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("shape,r,fit,noise", [
    ((32, 32, 32), 8, "auto", 1e-2),      # C1's shape
    ((5, 17, 9), 3, "auto", 1e-2),        # fewer mode-1 rows than CTAs: empty slabs
    ((13, 10, 11), 4, "explicit", 1e-2),  # ragged slabs, K not a multiple of 4
    ((20, 12, 30), 16, "gram", 1e-2),     # R = 16 (two column tiles)
    ((24, 16, 18), 6, "auto", 1e-6),      # near-exact: the explicit residual takes over
    ((9, 130, 7), 2, "auto", 1e-2),       # long mode 2
    ((1, 60, 50), 3, "auto", 1e-2),       # a single mode-1 row: seven empty slabs
    ((40, 1, 33), 2, "explicit", 1e-2),   # J = 1
    ((30, 44, 2), 2, "auto", 1e-2),       # K = 2 (one padded k-step)
    ((6, 7, 5), 1, "auto", 1e-2),         # R = 1
])
def test_cluster_and_one_cta_paths_match_oracle(shape, r, fit, noise):
    x = _low_rank(shape, r, sum(shape) + r, noise)
    init = oc.normal_init(shape, r, 5)
    ref = port.cp_als(x, r, 10, 0.0, init=lambda _t, _r: [v.copy() for v in init])
    tol_hist = 1e-10 if fit != "gram" else 1e-9
    res_cl = _run(x, r, 10, 0.0, fit, init)
    _check(res_cl, ref, tol_hist)
    res_1 = _run(x, r, 10, 0.0, fit, init, BT_CP_CLUSTER="0")
    _check(res_1, ref, tol_hist)
    np.testing.assert_allclose(res_cl.fit_history, res_1.fit_history, rtol=0, atol=1e-11)


def test_cluster_tol_stops_like_reference_and_is_deterministic():
    x = _low_rank((16, 14, 12), 3, 21, 1e-3)
    init = oc.normal_init(x.shape, 3, 11)
    ref = port.cp_als(x, 3, 300, 1e-9, init=lambda _t, _r: [v.copy() for v in init])
    r1 = _run(x, 3, 300, 1e-9, "auto", init)
    r2 = _run(x, 3, 300, 1e-9, "auto", init)
    _check(r1, ref)
    assert r1.fit_history == r2.fit_history            # bit-reproducible
    assert np.array_equal(np.asarray(r1.rep.x), np.asarray(r2.rep.x))


# ---------------------------------------------------------------------------
# small-rank two-pass path (R <= 16 beyond one SM)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("shape,r,fit,noise", [
    ((70, 60, 33), 5, "auto", 1e-2),       # R < 8: one column tile live
    ((96, 80, 64), 16, "auto", 1e-2),
    ((96, 80, 64), 16, "gram", 1e-2),
    ((96, 80, 64), 16, "explicit", 1e-2),
    ((100, 90, 300), 12, "auto", 1e-2),    # K > 256: two k spans in pass 2
    ((65, 64, 257), 9, "auto", 1e-2),      # K = 257: ragged 8-blocks
    ((128, 33, 40), 16, "auto", 1e-6),     # near-exact fit
    ((520, 300, 1), 2, "auto", 1e-2),      # K = 1: one padded 8-block per row
    ((400, 400, 3), 1, "explicit", 1e-2),  # R = 1, K = 3
    ((576, 70, 5), 3, "auto", 1e-2),       # the largest mode-1 extent the one-CTA update holds
    ((600, 70, 5), 3, "auto", 1e-2),       # one past it: the general path
    ((9, 470, 33), 4, "auto", 1e-2),       # short mode 1, long mode 2
])
def test_small_rank_path_matches_oracle(shape, r, fit, noise):
    x = _low_rank(shape, r, sum(shape) + r, noise)
    init = oc.normal_init(shape, r, 9)
    ref = port.cp_als(x, r, 8, 0.0, init=lambda _t, _r: [v.copy() for v in init])
    res = _run(x, r, 8, 0.0, fit, init)
    # the oracle's fit is the explicit residual; the Gram identity loses
    # ~eps ||X||^2 / (2 res) in the fit, far below 1e-9 at these fits
    _check(res, ref, 1e-10 if fit != "gram" else 1e-9, 1e-8)


def test_small_rank_path_vs_general_path_and_tol():
    shape, r = (128, 33, 40), 8
    x = _low_rank(shape, r, 77, 1e-3)
    init = oc.normal_init(shape, r, 6)
    ref = port.cp_als(x, r, 60, 1e-7, init=lambda _t, _r: [v.copy() for v in init])
    mid = _run(x, r, 60, 1e-7, "auto", init)
    gen = _run(x, r, 60, 1e-7, "auto", init, BT_CP_MID="0")
    _check(mid, ref)
    _check(gen, ref)
    again = _run(x, r, 60, 1e-7, "auto", init)
    assert mid.fit_history == again.fit_history        # ticket scheduling, fixed-order sums


@pytest.mark.parametrize("R", [8, 16])
def test_pinv_singular_matches_numpy_rank_and_projector(R):
    """The R <= 16 fallback (pivoted Cholesky + one-sided Jacobi on its factor)
    on numerically singular V: same kept rank as numpy's pinv (1e-15 cutoff)
    and the same range projector V pinv(V)."""
    from paper_2105_01170_b200 import _dev
    from paper_2105_01170_b200 import _native as N

    rng = np.random.default_rng(R)
    q, _ = np.linalg.qr(rng.standard_normal((R, R)))
    for lo in (-6.0, -12.0, -17.0, -20.0):
        lam = np.logspace(0, lo, R)
        v = (q * lam) @ q.T
        v = (v + v.T) / 2
        vd = torch.from_numpy(v).cuda()
        out = torch.empty_like(vd)
        N.call("bt_pinv_sym_f64", _dev.ptr(vd), R, _dev.ptr(out), _dev.stream())
        got = out.cpu().numpy()
        ref = np.linalg.pinv(v)
        rank_ref = np.linalg.matrix_rank(ref @ v, tol=0.5)
        rank_got = np.linalg.matrix_rank(got @ v, tol=0.5)
        assert rank_got == rank_ref, (lo, rank_got, rank_ref)
        # full numerical rank: the inverse, to the kappa * eps both sides can claim
        if lo > -14.0:
            assert np.abs(got - ref).max() <= 50 * 10.0 ** (-lo) * 2.2e-16 * np.abs(ref).max(), lo
