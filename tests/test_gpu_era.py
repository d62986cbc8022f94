"""GPU parity for the compressed-coordinate ERA (apps.py:153-237; SURVEY
§8f #3) against the reference's golden output (tests/golden/era.npz).
Singular vectors have LAPACK's sign freedom, so the realized (A, B, C) are
compared through similarity invariants: eigenvalues and the realized Markov
parameters.  Tolerances: reduced Hankel and leading singular values 1e-10
relative (north_star operators), realized Markov parameters 1e-9."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_01170_b200 as bt  # noqa: E402
from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402

CASES = (("full", 71, 6, 2, 2, 20, (2, 39, 2), 6, False),
         ("cut", 72, 5, 3, 2, 16, (3, 12, 2), 5, False),
         ("tera", 73, 4, 3, 3, 12, (2, 0, 2), 4, True),
         ("siso", 74, 2, 1, 1, 10, (1, 19, 1), 2, False))


def _hausdorff(x, y):
    d = np.abs(np.asarray(x)[:, None] - np.asarray(y)[None, :])
    return max(d.min(axis=1).max(), d.min(axis=0).max())


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_era_matches_reference(golden, case):
    z = golden("era")
    name, seed, d, no, ni, s, ranks, order, tera = case
    a, b, c = oc.era_system(seed, d, no, ni)
    seq = bt.markov_from_lti(bt.LtiSystem(a=a, b=b, c=c), 2 * s - 1)
    assert np.allclose(seq.params, z[f"{name}_params"], rtol=1e-13, atol=1e-14)
    res = bt.era_identify_compressed(seq, ranks, order, tera=tera)
    sv = res.sing_vals
    ref_sv = z[f"{name}_sv"]
    assert np.abs(sv[:order] - ref_sv[:order]).max() <= 1e-10 * ref_sv[0]
    assert np.abs(sv - ref_sv).max() <= 1e-12 * ref_sv[0]        # tail at rounding level
    red = z[f"{name}_reduced"]
    assert np.abs(res.reduced_hankel - red).max() <= 1e-10 * np.abs(red).max()
    assert _hausdorff(res.system.eigenvalues(), z[f"{name}_eig"]) <= 1e-8
    mk = bt.markov_from_lti(res.system, 2 * s - 1).params
    ref_mk = z[f"{name}_markov"]
    assert np.abs(mk - ref_mk).max() <= 1e-9 * np.abs(ref_mk).max()
    approx = res.hankel_approx()
    assert np.abs(approx - z[f"{name}_approx"]).max() <= 1e-10 * np.abs(approx).max()


def test_era_full_rank_reproduces_hankel_and_true_eigs():
    a, b, c = oc.era_system(75, 6, 2, 2)
    s = 50
    seq = bt.markov_from_lti(bt.LtiSystem(a=a, b=b, c=c), 2 * s - 1)
    res = bt.era_identify_compressed(seq, (2, 2 * s - 1, 2), order=6)
    assert _hausdorff(res.system.eigenvalues(), np.linalg.eigvals(a)) <= 1e-6
    pat, params = bt.hankel_pattern_from_markov(seq)
    h = bt.struct_assemble(pat, params)
    assert np.abs(res.hankel_approx() - h).max() <= 1e-11 * np.abs(h).max()
    # device-resident inputs stay on the device
    seq_d = bt.MarkovSequence(params=torch.from_numpy(np.asarray(seq.params)).cuda())
    res_d = bt.era_identify_compressed(seq_d, (2, 2 * s - 1, 2), order=6)
    assert res_d.system.a.is_cuda and res_d.reduced_hankel.is_cuda


def test_era_errors():
    with pytest.raises(bt.ConvergenceError):
        bt.era_identify_compressed(bt.MarkovSequence(params=np.zeros((9, 2, 2))), (2, 9, 2), 1)
    a, b, c = oc.era_system(76, 2, 1, 1)
    seq = bt.markov_from_lti(bt.LtiSystem(a=a, b=b, c=c), 9)
    with pytest.raises(bt.ShapeError):
        bt.era_identify_compressed(seq, (1, 9, 1), order=0)
    with pytest.raises(bt.ConvergenceError):
        bt.era_identify_compressed(seq, (1, 9, 1), order=4)
    with pytest.raises(bt.ShapeError):
        bt.era_identify_compressed(bt.MarkovSequence(params=np.ones((1, 1, 1))), (1, 1, 1), 1)
