"""GPU parity for detect_pattern (blocks.py:266-329): device
digest + verify passes against the reference's golden output, bit-exact
(placements, class order, representatives, structure tag)."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2105_01170_b200 as bt  # noqa: E402
from oracle import configs as oc  # noqa: E402
from oracle import port  # noqa: E402

from conftest import GOLDEN  # noqa: E402


def _flat(pat):
    cells = np.vstack(pat.placements).astype(np.int64)
    return cells, np.cumsum([0] + list(pat.counts)).astype(np.int64)


def test_detect_golden_bit_exact(golden):
    z = golden("detect")
    meta = {d["name"]: d for d in json.load(open(os.path.join(GOLDEN, "detect.json")))}
    for name, a, m, n, tol in oc.detect_cases():
        pat, reps = bt.detect_pattern(a, m, n, tol=tol)
        cells, offs = _flat(pat)
        assert np.array_equal(cells, z[f"{name}_cells"]), name
        assert np.array_equal(offs, z[f"{name}_offs"]), name
        assert np.array_equal(np.stack(reps).view(np.int64), z[f"{name}_reps"].view(np.int64)), name
        assert pat.structure_class == meta[name]["structure_class"], name
        # device input: same pattern, device representatives
        pd, rd = bt.detect_pattern(torch.from_numpy(a).cuda(), m, n, tol=tol)
        assert pd == pat and rd[0].is_cuda
        assert np.array_equal(np.stack([r.cpu().numpy() for r in rd]).view(np.int64),
                              np.stack(reps).view(np.int64))


def test_detect_errors_and_roundtrip():
    with pytest.raises(bt.PatternMismatchError):
        bt.detect_pattern(np.zeros((4, 4)), 2, 2)
    with pytest.raises(bt.PatternMismatchError):
        bt.detect_pattern(np.full((4, 4), -0.0), 2, 2)
    with pytest.raises(bt.ShapeError):
        bt.detect_pattern(np.zeros((5, 4)), 2, 2)
    with pytest.raises(bt.ShapeError):
        bt.detect_pattern(np.zeros(4), 2, 2)
    pat, blocks = bt.detect_pattern(np.eye(4), 2, 2)
    assert pat.p == 1 and pat.counts == (2,) and pat.structure_class == "diagonal"
    rng = np.random.default_rng(1)
    for kind in ("toeplitz", "hankel", "diagonal"):
        p0 = bt.build_pattern(kind, 7, 7, 3, 4)
        blocks = [rng.standard_normal((3, 4)) for _ in range(p0.p)]
        a = bt.struct_assemble(p0, np.stack(blocks))
        p1, b1 = bt.detect_pattern(a, 3, 4)
        assert np.array_equal(bt.struct_assemble(p1, np.stack(b1)), a)


def test_detect_large_matches_oracle():
    """256 x 256 grid of 32 x 32 blocks (64 MiB): symmetric block Toeplitz
    with a few zeroed cells -- the digest path at scale, vs the oracle."""
    rng = np.random.default_rng(7)
    ell, nb = 256, 32
    pat = port.make_pattern("toeplitz", ell, ell, nb, nb)
    blocks = [rng.standard_normal((nb, nb)) for _ in range(pat.p)]
    a = port.assemble(pat, blocks)
    a[:nb, 5 * nb:6 * nb] = 0.0
    got, reps = bt.detect_pattern(a, nb, nb)
    pl, reps_o, cls = port.detect_pattern(a, nb, nb)
    assert got.p == len(pl) and got.structure_class == cls
    for x, y in zip(got.placements, pl):
        assert np.array_equal(x, y)
    for x, y in zip(reps, reps_o):
        assert np.array_equal(x, y)
