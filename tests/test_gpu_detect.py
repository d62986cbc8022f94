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


def _group_dev(h1, h2, nz):
    from paper_2105_01170_b200 import _dev
    from paper_2105_01170_b200 import _native as N

    cells = len(h1)
    d1 = torch.from_numpy(h1.view(np.int64)).cuda()
    d2 = torch.from_numpy(h2.view(np.int64)).cuda()
    dz = torch.from_numpy(nz.astype(np.int32)).cuda()
    lead = torch.empty(cells, dtype=torch.int64, device="cuda")
    cand = torch.empty(cells, dtype=torch.int64, device="cuda")
    ws = _dev.workspace(int(N.load().bt_block_group_ws_bytes(cells)))
    N.call("bt_block_group", _dev.ptr(d1), _dev.ptr(d2), _dev.ptr(dz), cells, _dev.ptr(lead),
           _dev.ptr(cand), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    return lead.cpu().numpy(), cand.cpu().numpy()


@pytest.mark.parametrize("cells,distinct", [(1, 1), (7, 1), (1000, 3), (5000, 5000), (40000, 257)])
def test_block_group_first_occurrence(cells, distinct):
    """bt_block_group against a host dictionary: the leader of a kept cell is
    the first kept cell with the same 128-bit key (keys that share h1 or h2
    alone stay apart), skipped cells get -1, cand is -1 for leaders."""
    rng = np.random.default_rng(cells + distinct)
    pool1 = rng.integers(0, 2**63, size=distinct, dtype=np.int64).astype(np.uint64)
    pool2 = rng.integers(0, 2**63, size=distinct, dtype=np.int64).astype(np.uint64)
    if distinct >= 3:            # same h1 / different h2 and the other way round
        pool1[1] = pool1[0]
        pool2[2] = pool2[0]
    pick = rng.integers(0, distinct, size=cells)
    h1, h2 = pool1[pick].copy(), pool2[pick].copy()
    nz = (rng.random(cells) > 0.2).astype(np.int32)
    if cells == 1:
        nz[:] = 1
    lead, cand = _group_dev(h1, h2, nz)
    seen, want = {}, np.full(cells, -1, dtype=np.int64)
    for c in range(cells):
        if nz[c]:
            want[c] = seen.setdefault((int(h1[c]), int(h2[c])), c)
    assert np.array_equal(lead, want)
    assert np.array_equal(cand, np.where(want == np.arange(cells), -1, want))


@pytest.mark.parametrize("m,n,ell,q", [(5, 3, 7, 9), (33, 6, 4, 5), (70, 34, 3, 3), (2, 2, 40, 40),
                                       (64, 1030, 2, 2)])
def test_detect_ragged_block_shapes_match_oracle(m, n, ell, q):
    """Block shapes off the digest kernel's fast walk: odd widths (8-byte
    accesses), rows that do not divide the CTA, ragged tails, a row wider
    than the CTA -- placements and representatives against the oracle."""
    rng = np.random.default_rng(m * 131 + n)
    pool = [rng.standard_normal((m, n)) for _ in range(5)]
    pool.append(np.zeros((m, n)))
    pool.append(-pool[0])                       # sign flips only
    swapped = pool[1].copy()
    swapped[0, 0], swapped[-1, -1] = swapped[-1, -1], swapped[0, 0]
    pool.append(swapped)                        # same multiset of entries
    pick = rng.integers(0, len(pool), size=(ell, q))
    a = np.block([[pool[pick[i, j]] for j in range(q)] for i in range(ell)])
    got, reps = bt.detect_pattern(a, m, n)
    pl, reps_o, cls = port.detect_pattern(a, m, n)
    assert got.p == len(pl) and got.structure_class == cls
    for x, y in zip(got.placements, pl):
        assert np.array_equal(x, y)
    for x, y in zip(reps, reps_o):
        assert np.array_equal(x, y)
    gd, rd = bt.detect_pattern(torch.from_numpy(a).cuda()[:, :], m, n)
    assert all(np.array_equal(x, y) for x, y in zip(gd.placements, pl))
