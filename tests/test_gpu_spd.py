"""GPU parity for the SPD-preserving compression (psd.py:205-271,
decomp.py:196-212) against the reference's golden vectors
(tests/golden/spd.npz).  Tolerances: operators 1e-10 relative Frobenius
(BASELINE.json north_star); the Cholesky factor 1e-13 relative."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_01170_b200 as bt  # noqa: E402
from oracle import configs as oc  # noqa: E402

CASES = ((21, 4, 5), (22, 3, 8), (23, 6, 3))


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def test_cholesky_golden_and_errors(golden):
    z = golden("spd")
    low = bt.cholesky(z["chol_in"])
    assert isinstance(low, np.ndarray)
    assert rel(low, z["chol_out"]) < 1e-13
    assert np.all(np.triu(low, 1) == 0)
    with pytest.raises(bt.NotPositiveDefiniteError):
        bt.cholesky(np.diag([1.0, -1.0]))
    with pytest.raises(bt.ShapeError):
        bt.cholesky(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(bt.ShapeError):
        bt.cholesky(np.zeros((2, 3)))
    # larger SPD matrix: L L^T reproduces the input
    g = np.random.default_rng(3).standard_normal((300, 300))
    a = g @ g.T + 300 * np.eye(300)
    low = bt.cholesky(a)
    assert rel(low @ low.T, a) < 1e-14
    assert rel(low, np.linalg.cholesky(a)) < 1e-13


@pytest.mark.parametrize("case", range(len(CASES)))
def test_spd_compress_every_rank_golden(golden, case):
    z = golden("spd")
    seed, ell, nb = CASES[case]
    _, a = oc.spd_toeplitz(seed, ell, nb)
    pat = bt.build_pattern("toeplitz", ell, ell, nb, nb)
    for r in range(1, nb + 1):
        rep = bt.spd_compress(a, pat, r)
        assert rep.rank == r and rep.shape == a.shape
        dense = rep.densify()
        ref = z[f"s{case}_r{r}_dense"]
        assert rel(dense, ref) < 1e-10, (case, r)
        np.linalg.cholesky((dense + dense.T) / 2)  # SPD at every rank
        if r == 1:
            assert rel(rep.chol, z[f"s{case}_chol"]) < 1e-13
            cells = np.concatenate(rep.remainder.pattern.placements)
            assert np.array_equal(cells, z[f"s{case}_rem_cells"])
            assert list(rep.remainder.pattern.counts) == list(z[f"s{case}_rem_counts"])
            assert rep.remainder.pattern.structure_class == str(z[f"s{case}_rem_class"])
        if r == nb:
            assert rel(dense, a) < 1e-10
    # quadratic-form identity x'Tx = x1'(I + M)x1, x1 = (I (x) L^T) x
    rep = bt.spd_compress(a, pat, 2)
    lfull = np.kron(np.eye(ell), rep.chol)
    inner = np.eye(ell * nb) + rep.remainder.densify()
    x = np.random.default_rng(15).standard_normal(ell * nb)
    x1 = lfull.T @ x
    assert np.isclose(x @ rep.densify() @ x, x1 @ inner @ x1, rtol=1e-12)


def test_spd_device_inputs_stay_on_device():
    _, a = oc.spd_toeplitz(21, 4, 5)
    pat = bt.build_pattern("toeplitz", 4, 4, 5, 5)
    ad = torch.from_numpy(a).cuda()
    rep = bt.spd_compress(ad, pat, 3)
    assert rep.chol.is_cuda and rep.remainder.basis.is_cuda
    dense = rep.densify()
    assert dense.is_cuda
    assert rel(dense.cpu().numpy(), bt.spd_compress(a, pat, 3).densify()) < 1e-14


def test_spd_block_diagonal_and_errors(golden):
    z = golden("spd")
    cells = np.column_stack([np.arange(3), np.arange(3)])
    pat = bt.BlockPattern(ell=3, q=3, m=4, n=4, placements=(cells,), structure_class="diagonal")
    rep = bt.spd_compress(z["bd_a"], pat, 2)
    assert rep.remainder.pattern.p == 0
    assert np.abs(rep.densify() - z["bd_dense"]).max() < 1e-12
    with pytest.raises(bt.NotPositiveDefiniteError):
        bt.spd_compress(-np.eye(6), bt.build_pattern("diagonal", 3, 3, 2, 2), 1)
    corner = bt.BlockPattern(ell=3, q=3, m=2, n=2, placements=(np.array([[1, 1], [2, 2]]),))
    with pytest.raises(bt.PatternMismatchError):
        bt.spd_compress(bt.struct_assemble(corner, np.stack([np.eye(2)])), corner, 1)
    with pytest.raises(bt.ShapeError):
        bt.spd_compress(np.zeros((6, 7)), bt.build_pattern("diagonal", 3, 3, 2, 2), 1)


def test_spd_larger_anchor():
    """n = 96 blocks on an 8 x 8 Toeplitz grid: full rank reproduces A."""
    rng = np.random.default_rng(31)
    nb, ell = 96, 8
    pat = bt.build_pattern("toeplitz", ell, ell, nb, nb)
    g = rng.standard_normal((nb, nb))
    anchor = g @ g.T + nb * np.eye(nb)
    up = [0.05 * rng.standard_normal((nb, nb)) for _ in range(ell - 1)]
    blocks = np.stack([anchor] + up + [u.T for u in up])
    a = bt.struct_assemble(pat, blocks)
    rep = bt.spd_compress(a, pat, nb)
    assert rel(rep.densify(), a) < 1e-10
    rep = bt.spd_compress(a, pat, 10)
    np.linalg.cholesky(rep.densify())
