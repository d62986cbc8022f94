"""Multilevel (nested) block structure (drop-in for multilevel.py).

C4 path: ``psf_weighted_tensor`` builds the weighted 3-level tensor on the
GPU (K3), generalised to an image grid larger than the kernel (the
reference fixes image == kernel size, multilevel.py:268-298); ``cp_als`` on
its squeezed (K, K, K) core; ``ml_kron_sum_from_kruskal`` maps the CP factors
to one 3-level Kronecker term per component (level matrices are the
``struct_scalars`` assemblies of the factor columns, multilevel.py:214-218);
``ml_matvec`` applies the sum of terms to a batch of volumes with DMMA mode
products -- the reference has no structured multilevel matvec (it densifies,
cli.py:247-248).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from functools import reduce
from itertools import product

import numpy as np

from . import _dev
from . import _native as N
from .blocks import BlockPattern, kernel_level_pattern, struct_scalars
from .decomp import KruskalRep, TuckerRep
from .errors import ShapeError
from .tensor import ttm_dev

__all__ = ["MultilevelPattern", "MlKronTerm", "ml_kron_sum_from_tucker",
           "ml_kron_sum_from_kruskal", "ml_matvec", "psf_weighted_tensor", "MAX_LEVELS",
           "MultilevelTuckerRep"]

MAX_LEVELS = 3  # multilevel.py:40


@dataclass(frozen=True)
class MultilevelPattern:
    """multilevel.py:43-88: chain of block patterns, outermost first."""

    levels: tuple

    def __post_init__(self) -> None:
        if not 1 <= len(self.levels) <= MAX_LEVELS:
            raise ShapeError(f"between 1 and {MAX_LEVELS} levels supported")
        for t in range(len(self.levels) - 1):
            outer, inner = self.levels[t], self.levels[t + 1]
            if (outer.m, outer.n) != inner.shape:
                raise ShapeError(f"level {t + 1} block extents {(outer.m, outer.n)} != "
                                 f"level {t + 2} assembled shape {inner.shape}")

    @property
    def depth(self) -> int:
        return len(self.levels)

    @property
    def m(self) -> int:
        return self.levels[-1].m

    @property
    def n(self) -> int:
        return self.levels[-1].n

    @property
    def class_counts(self) -> tuple:
        return tuple(lv.p for lv in self.levels)

    @property
    def dims(self) -> tuple:
        return (self.m, *self.class_counts, self.n)

    @property
    def shape(self) -> tuple:
        return self.levels[0].shape


@dataclass(frozen=True)
class MultilevelTuckerRep:
    """multilevel.py:156-183: a level chain with the Tucker factorization of
    its weighted order-(L+2) tensor."""

    pattern: MultilevelPattern
    tucker: object

    def __post_init__(self) -> None:
        if self.tucker.dims != self.pattern.dims:
            raise ShapeError(f"tucker dims {self.tucker.dims} != pattern dims {self.pattern.dims}")

    @property
    def shape(self) -> tuple:
        return self.pattern.shape

    def terms(self):
        return ml_kron_sum_from_tucker(self.tucker, self.pattern)

    def densify(self):
        """multilevel.py:177-183: ml_tensor_to_mat of the reconstructed
        tensor, as K2 scatters from the innermost level outwards (each level's
        assembled matrices are the next level's class items)."""
        from .blocks import _scatter_dev
        from .reconstruct import DENSIFY_LIMIT

        rows, cols = self.pattern.shape
        if rows * cols > DENSIFY_LIMIT:
            raise ShapeError(f"dense result would hold {rows * cols} entries (limit {DENSIFY_LIMIT})")
        t = _dev.torch()
        x = _dev.to_device(self.tucker.reconstruct())          # (m, p1, ..., pL, n)
        levels = self.pattern.levels
        depth = len(levels)
        # items[prefix] = (M, p_t, N) tensor of level t, prefix over outer classes
        outer = [range(lv.p) for lv in levels[:-1]]
        mats = {}
        for prefix in product(*outer):
            idx = (slice(None),) + tuple(prefix) + (slice(None), slice(None))
            items = x[idx]                                       # (m, pL, n) view
            sm, sp, sn = (int(v) for v in items.stride())
            pat = levels[-1]
            mats[prefix] = _scatter_dev(items, sm, sp, sn, pat)
        for lvl in range(depth - 2, -1, -1):
            pat = levels[lvl]
            nxt = {}
            for prefix in product(*outer[:lvl]):
                items = t.stack([mats[prefix + (k,)] for k in range(pat.p)], dim=1).contiguous()
                sm, sp, sn = (int(v) for v in items.stride())
                nxt[prefix] = _scatter_dev(items, sm, sp, sn, pat)
            mats = nxt
        return _dev.like_input(self.tucker.core, mats[()])


@dataclass(frozen=True)
class MlKronTerm:
    """multilevel.py:186-194: level_mats[0] (x) ... (x) block."""

    level_mats: tuple
    block: object

    def densify(self):
        """multilevel.py:193-194: level_mats[0] (x) ... (x) block, folded
        left to right like the reference's reduce(np.kron, ...)."""
        mats = (*self.level_mats, self.block)
        if _dev.is_device(self.block):
            kron = _dev.torch().kron
            mats = tuple(_dev.to_device(m) for m in mats)
        else:
            kron = np.kron
            mats = tuple(np.asarray(m) for m in mats)
        return reduce(kron, mats)


def psf_weighted_tensor(psf, grid: int | None = None):
    """multilevel.py:268-298 on the GPU, with an optional image grid (per
    side) larger than the kernel: ``eta_i = grid - |i - h|``.  Returns
    ``(tensor (1, K, K, K, 1), MultilevelPattern)``."""
    if _dev.is_device(psf):
        pd = psf.to(dtype=_dev.torch().float64).contiguous()
    else:
        pd = _dev.to_device(np.asarray(psf, dtype=np.float64))
    if pd.ndim != 3 or len(set(pd.shape)) != 1:
        raise ShapeError("psf must be a K x K x K cube")
    k = int(pd.shape[0])
    if k % 2 == 0:
        raise ShapeError("psf extent K must be odd")
    grid = k if grid is None else int(grid)
    x = _dev.empty((k, k, k))
    N.call("bt_build_psf_f64", _dev.ptr(pd), k, grid, _dev.ptr(x), _dev.stream())
    lv3 = kernel_level_pattern(k, 1, 1, grid)
    lv2 = kernel_level_pattern(k, grid, grid, grid)
    lv1 = kernel_level_pattern(k, grid * grid, grid * grid, grid)
    mlp = MultilevelPattern(levels=(lv1, lv2, lv3))
    return _dev.like_input(psf, x.reshape(1, k, k, k, 1)), mlp


def ml_kron_sum_from_tucker(t: TuckerRep, mlp: MultilevelPattern):
    """multilevel.py:197-225: one term per mode-2..L+1 core multi-index."""
    if t.core.ndim != mlp.depth + 2:
        raise ShapeError(f"Tucker order {t.core.ndim} != pattern order {mlp.depth + 2}")
    if t.dims != mlp.dims:
        raise ShapeError(f"Tucker dims {t.dims} != pattern dims {mlp.dims}")
    u, w = t.factors[0], t.factors[-1]
    tt = _dev.torch()
    facs = [tt.eye(lv.p, dtype=tt.float64, device="cuda") if f is None else _dev.to_device(f)
            for lv, f in zip(mlp.levels, t.factors[1:-1])]
    core = _dev.to_device(t.core)
    if u is not None:
        core = ttm_dev(core, 1, _dev.to_device(u), int(u.shape[0]))
    if w is not None:
        core = ttm_dev(core, core.ndim, _dev.to_device(w), int(w.shape[0]))
    terms = []
    for multi in product(*(range(int(f.shape[1])) for f in facs)):
        mats = tuple(_dev.like_input(t.core, struct_scalars(lv, facs[k][:, multi[k]].contiguous()))
                     for k, lv in enumerate(mlp.levels))
        blk = core[(slice(None), *multi, slice(None))].contiguous()
        terms.append(MlKronTerm(level_mats=mats, block=_dev.like_input(t.core, blk)))
    return terms


def ml_kron_sum_from_kruskal(k: KruskalRep, mlp: MultilevelPattern):
    """CP route (new): term r = (S1(x_r), S2(y_r), S3(z_r)) with
    a 1 x 1 innermost block -- the Tucker route of multilevel.py:197-225
    applied to the superdiagonal core, keeping only its nonzero terms."""
    if mlp.depth != 3 or (mlp.m, mlp.n) != (1, 1):
        raise ShapeError("CP route needs a 3-level pattern with 1 x 1 innermost blocks")
    if k.dims != mlp.class_counts:
        raise ShapeError(f"CP dims {k.dims} != class counts {mlp.class_counts}")
    fac = [_dev.to_device(f) for f in (k.x, k.y, k.z)]
    one = np.ones((1, 1)) if not _dev.is_device(k.x) else _dev.torch().ones((1, 1), dtype=_dev.torch().float64, device="cuda")
    terms = []
    for r in range(k.rank):
        mats = tuple(_dev.like_input(k.x, struct_scalars(lv, fac[t][:, r].contiguous()))
                     for t, lv in enumerate(mlp.levels))
        terms.append(MlKronTerm(level_mats=mats, block=one))
    return terms


def stack_level_mats(terms):
    """Device stacks S_t (nterms, rows, cols) for t = 1..3."""
    tt = _dev.torch()
    return [tt.stack([_dev.to_device(term.level_mats[t]) for term in terms]).contiguous()
            for t in range(3)]


def ml_matvec(terms, x, stacks=None):
    """y = sum_r (S1_r (x) S2_r (x) S3_r) x for 3-level terms with 1 x 1
    blocks (block values fold into S3).  x: (N,) or (N, nrhs) with the first
    image axis fastest (multilevel.py:312-318 vectorisation)."""
    if not terms:
        raise ShapeError("no terms")
    for term in terms:
        if len(term.level_mats) != 3 or tuple(term.block.shape) != (1, 1):
            raise ShapeError("ml_matvec supports 3-level terms with 1 x 1 blocks")
    s1, s2, s3 = stacks if stacks is not None else stack_level_mats(terms)
    blocks = np.array([float(t.block[0, 0]) for t in terms])
    if not np.all(blocks == 1.0):
        bscale = _dev.to_device(blocks).reshape(-1, 1, 1)
        s3 = (s3 * bscale).contiguous()
    nterms = int(s1.shape[0])
    nin = (int(s1.shape[2]), int(s2.shape[2]), int(s3.shape[2]))
    nout = (int(s1.shape[1]), int(s2.shape[1]), int(s3.shape[1]))
    ntot = nin[0] * nin[1] * nin[2]
    if x.ndim == 1:
        if x.shape[0] != ntot:
            raise ShapeError(f"vector length {x.shape[0]} != {ntot}")
        xd = _dev.to_device(x).reshape(1, ntot)
        nrhs = 1
    else:
        if x.shape[0] != ntot:
            raise ShapeError(f"right-hand sides of shape {tuple(x.shape)} != ({ntot}, nrhs)")
        xd = _dev.transpose(_dev.to_device(x))
        nrhs = int(x.shape[1])
    y = _dev.empty((nrhs, nout[0] * nout[1] * nout[2]))
    cin = (C.c_int64 * 3)(*nin)
    cout = (C.c_int64 * 3)(*nout)
    ws = _dev.workspace(N.load().bt_ml_matvec_ws_bytes(nterms, cin, cout, nrhs))
    N.call("bt_ml_matvec_f64", nterms, cin, cout, _dev.ptr(s1), _dev.ptr(s2), _dev.ptr(s3),
           _dev.ptr(xd), nrhs, _dev.ptr(y), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    out = y[0] if x.ndim == 1 else _dev.transpose(y)
    return _dev.like_input(x, out)
