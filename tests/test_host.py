"""Host logic (CPU only): pattern builders bit-exact against the reference's
golden vectors, validation semantics, device-map construction, and the
C-ABI library loading with every symbol include/bt200.h declares."""

import ctypes
import hashlib
import json
import os
import re

import numpy as np
import pytest

from paper_2105_01170_b200 import _native
from paper_2105_01170_b200.blocks import BlockPattern, build_pattern, kernel_level_pattern
from paper_2105_01170_b200.errors import ShapeError

from conftest import GOLDEN, ROOT


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _flat(pat):
    cells = np.vstack(pat.placements) if pat.p else np.zeros((0, 2), np.int64)
    return cells.astype(np.int64), np.cumsum([0] + list(pat.counts)).astype(np.int64)


def test_builders_bit_exact_small(golden):
    meta = json.load(open(os.path.join(GOLDEN, "patterns.json")))
    z = golden("patterns")
    for idx, spec in enumerate(meta["small"]):
        pat = build_pattern(spec["kind"], spec["ell"], spec["ell"], 2, 3, band=spec["band"],
                            block_symmetric=spec["sym"])
        cells, offs = _flat(pat)
        assert np.array_equal(cells, z[f"cells_{idx}"]), spec
        assert np.array_equal(offs, z[f"offs_{idx}"]), spec
        assert pat.structure_class == spec["tag"]
        for c in pat.placements:
            assert c.dtype == np.int64


def test_builders_bit_exact_config_sizes():
    meta = json.load(open(os.path.join(GOLDEN, "patterns.json")))
    for spec in meta["big"]:
        if spec["kind"] == "kernel_level":
            pat = kernel_level_pattern(spec["ell"], 1, 1)
        else:
            pat = build_pattern(spec["kind"], spec["ell"], spec["ell"], spec["m"], spec["n"],
                                block_symmetric=spec["sym"])
        cells, offs = _flat(pat)
        assert pat.p == spec["p"] and pat.structure_class == spec["tag"]
        assert _sha(cells) == spec["cells_sha"] and _sha(offs) == spec["offs_sha"], spec


def test_pattern_validation_matches_reference():
    with pytest.raises(ShapeError, match=r"grid cell \(1, 1\) claimed by two classes"):
        BlockPattern(ell=2, q=2, m=1, n=1, placements=(np.array([[0, 0]]), np.array([[0, 0]])))
    with pytest.raises(ShapeError, match="class 1: placement outside"):
        BlockPattern(ell=2, q=2, m=1, n=1, placements=(np.array([[2, 0]]),))
    with pytest.raises(ShapeError, match="nonempty"):
        BlockPattern(ell=2, q=2, m=1, n=1, placements=(np.zeros((0, 2)),))
    # first failing class wins: overlap in class 2 before a range error in class 3
    with pytest.raises(ShapeError, match="claimed by two"):
        BlockPattern(ell=3, q=3, m=1, n=1, placements=(np.array([[0, 0]]), np.array([[1, 1], [0, 0]]),
                                                       np.array([[5, 5]])))
    with pytest.raises(ShapeError):
        build_pattern("toeplitz", 3, 4, 2, 2)
    with pytest.raises(ShapeError):
        build_pattern("banded", 4, 4, 2, 2)
    with pytest.raises(ValueError):
        build_pattern("circulant", 4, 4, 2, 2)


def test_host_maps_brute_force():
    rng = np.random.default_rng(3)
    for kind, band, sym in (("toeplitz", None, True), ("hankel", None, False),
                            ("banded", 1, True), ("diagonal", None, False)):
        pat = build_pattern(kind, 5, 5, 2, 3, band=band, block_symmetric=sym)
        h = pat.host_maps()
        rank = 0
        for k, cells in enumerate(pat.placements):
            assert h["rep_cell"][k] == cells[0, 0] * 5 + cells[0, 1]
            assert h["eta"][k] == len(cells)
            for i, j in cells:
                assert h["cell_class"][i * 5 + j] == k
                assert h["cell_order"][i * 5 + j] == rank
                rank += 1
        unc = np.argwhere(h["cell_class"].reshape(5, 5) < 0)
        for i, j in unc:
            assert h["cell_order"][i * 5 + j] == h["nnz"] + i * 5 + j
        # row CSR: every cell once, rows ascending, columns ascending
        for i in range(5):
            ents = h["row_cells"][h["row_ptr"][i]:h["row_ptr"][i + 1]]
            cols = ents // pat.p
            assert np.all(np.diff(cols) > 0)
            for e in ents:
                j, k = divmod(int(e), pat.p)
                assert h["cell_class"][i * 5 + j] == k
    del rng


def test_library_exports_every_header_symbol():
    lib_path = _native.LIB_PATH
    if not os.path.exists(lib_path):
        from paper_2105_01170_b200.build import build
        build()
    header = open(os.path.join(ROOT, "include", "bt200.h")).read()
    names = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(bt_\w+)\s*\(", header, re.M))
    assert len(names) >= 25
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_native.exported_symbols()) <= names | {"bt_version", "bt_last_error"}
    assert names <= set(_native.exported_symbols())
    _native.load()
    assert _native.load().bt_version() == 1


def test_classify_placements_matches_oracle():
    """blocks.py:228-263 host tag on every builder kind and on random splits."""
    from oracle import port as _port
    from paper_2105_01170_b200.blocks import build_pattern, classify_placements

    rng = np.random.default_rng(5)
    for kind in ("toeplitz", "hankel", "diagonal", "banded", "circulant", "general"):
        for ell in (1, 2, 4, 7):
            try:
                pat = build_pattern(kind, ell, ell, 2, 2, **({"band": 1} if kind == "banded" else {}))
            except Exception:
                continue
            pl = pat.placements
            assert classify_placements(pl, ell, ell) == _port.classify_placements(pl, ell, ell)
            # split every class by the diagonal as spd_compress does
            split = []
            for c in pl:
                on = c[:, 0] == c[:, 1]
                split += [x for x in (c[on], c[~on]) if len(x)]
            split = [split[i] for i in rng.permutation(len(split))]
            assert (classify_placements(tuple(split), ell, ell)
                    == _port.classify_placements(tuple(split), ell, ell))
    assert classify_placements((), 3, 3) == "general"


def test_classify_placements_random_families():
    """Vectorised classify vs the per-class restatement on random families,
    including exact diagonals, +-d pairs, anti-diagonals and partial ones."""
    from oracle import port as _port
    from paper_2105_01170_b200.blocks import classify_placements

    rng = np.random.default_rng(11)
    for trial in range(400):
        ell = int(rng.integers(1, 7))
        q = ell if rng.random() < 0.8 else int(rng.integers(1, 7))
        cells = np.array([(i, j) for i in range(ell) for j in range(q)], dtype=np.int64)
        mode = trial % 4
        if mode == 0:      # by diagonal offset, some merged +-d, maybe dropped cells
            key = cells[:, 1] - cells[:, 0]
            if rng.random() < 0.5:
                key = np.abs(key)
        elif mode == 1:    # by anti-diagonal
            key = cells[:, 0] + cells[:, 1]
        elif mode == 2:    # diagonal only
            key = np.where(cells[:, 0] == cells[:, 1], 0, -1)
        else:              # random
            key = rng.integers(0, 4, len(cells))
        keep = rng.random(len(cells)) > (0.15 if trial % 3 == 0 else 0.0)
        fam = [cells[(key == k) & keep] for k in np.unique(key[key >= 0])]
        fam = tuple(f for f in fam if len(f))
        assert classify_placements(fam, ell, q) == _port.classify_placements(fam, ell, q), (ell, q, fam)
