"""Structured representations and their matvecs (drop-in for reconstruct.py).

Converters out of CP / Tucker (reconstruct.py:170-263) are DMMA products on
device; ``matvec`` (reconstruct.py:271-315) runs the K11 kernels and accepts
either one vector (reference signature) or a (q*n, nrhs) block of
right-hand sides (extension: all columns in one launch sequence).  The
``counter`` argument receives exactly the reference's FlopCounter counts
(reconstruct.py:295, 302, 309, 312), times the number of columns.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _dev
from . import _linalg as L
from . import _native as N
from .blocks import BlockPattern, struct_expand, struct_scalars
from .decomp import KruskalRep, TuckerRep, qr_thin
from .errors import ShapeError
from .tensor import fro_norm_dev, ttm_dev

__all__ = [
    "KronSumRep", "BlockLowRankRep", "TuckerBlockRep", "FlopCounter", "kron_sum_from_tucker",
    "kron_sum_from_kruskal", "blr_from_tucker", "blr_from_kruskal", "matvec", "densify",
    "error_fro", "DENSIFY_LIMIT", "c_term_dense",
]

DENSIFY_LIMIT = 10**8  # reconstruct.py:45


class FlopCounter:
    """reconstruct.py:48-55."""

    def __init__(self) -> None:
        self.flops = 0

    def add(self, n) -> None:
        self.flops += int(n)


@dataclass(frozen=True)
class KronSumRep:
    """reconstruct.py:58-99: sum_j C_j (x) terms[j], C_j = sum_k coeffs[k,j] E_k."""

    pattern: BlockPattern
    coeffs: object
    terms: object

    def __post_init__(self) -> None:
        p, r = self.coeffs.shape
        if p != self.pattern.p:
            raise ShapeError(f"coeffs rows {p} != number of classes {self.pattern.p}")
        if tuple(self.terms.shape) != (r, self.pattern.m, self.pattern.n):
            raise ShapeError(f"terms shape {tuple(self.terms.shape)} != "
                             f"({r}, {self.pattern.m}, {self.pattern.n})")

    @property
    def n_terms(self) -> int:
        return int(self.coeffs.shape[1])

    @property
    def shape(self) -> tuple:
        return self.pattern.shape

    def c_matrix(self, j: int):
        """Sparse C_j as scipy CSR (host helper, reconstruct.py:91-99)."""
        import scipy.sparse as sp

        pat = self.pattern
        coeffs = self.coeffs if not _dev.is_device(self.coeffs) else _dev.to_host(self.coeffs)
        rows, cols, data = [], [], []
        for k, cells in enumerate(pat.placements):
            rows.extend(cells[:, 0])
            cols.extend(cells[:, 1])
            data.extend([coeffs[k, j] / np.sqrt(len(cells))] * len(cells))
        return sp.csr_matrix((data, (rows, cols)), shape=(pat.ell, pat.q))


@dataclass(frozen=True)
class BlockLowRankRep:
    """reconstruct.py:102-128: (I (x) left) S (I (x) right^T)."""

    pattern: BlockPattern
    left: object
    right: object
    middles: object

    def __post_init__(self) -> None:
        rl, rr = self.left.shape[1], self.right.shape[1]
        if self.left.shape[0] != self.pattern.m or self.right.shape[0] != self.pattern.n:
            raise ShapeError("side bases do not match the pattern's block extents")
        if tuple(self.middles.shape) != (self.pattern.p, rl, rr):
            raise ShapeError(f"middles shape {tuple(self.middles.shape)} != "
                             f"({self.pattern.p}, {rl}, {rr})")

    @property
    def shape(self) -> tuple:
        return self.pattern.shape


@dataclass(frozen=True)
class TuckerBlockRep:
    """reconstruct.py:131-152."""

    pattern: BlockPattern
    tucker: TuckerRep

    def __post_init__(self) -> None:
        pat = self.pattern
        if self.tucker.dims != (pat.m, pat.p, pat.n):
            raise ShapeError(f"tucker dims {self.tucker.dims} != pattern dims "
                             f"{(pat.m, pat.p, pat.n)}")

    @property
    def shape(self) -> tuple:
        return self.pattern.shape

    def to_kron_sum(self) -> KronSumRep:
        return kron_sum_from_tucker(self.tucker, self.pattern)


# ---------------------------------------------------------------------------
# converters
# ---------------------------------------------------------------------------


def _tucker_side(t: TuckerRep, pattern: BlockPattern):
    if t.core.ndim != 3:
        raise ShapeError("expected an order-3 Tucker representation")
    if t.dims != (pattern.m, pattern.p, pattern.n):
        raise ShapeError(f"Tucker dims {t.dims} do not match pattern "
                         f"({pattern.m}, {pattern.p}, {pattern.n})")
    return t.factors


def kron_sum_from_tucker(t: TuckerRep, pattern: BlockPattern) -> KronSumRep:
    """reconstruct.py:170-189: coeffs = V (or I), D_j = U core[:, j, :] W^T."""
    u, v, w = _tucker_side(t, pattern)
    ref = t.core
    cd = _dev.to_device(t.core)
    if u is not None:
        cd = ttm_dev(cd, 1, _dev.to_device(u), int(u.shape[0]))
    if w is not None:
        cd = ttm_dev(cd, 3, _dev.to_device(w), int(w.shape[0]))
    terms = cd.permute(1, 0, 2).contiguous()
    if v is None:
        coeffs = _dev.torch().eye(pattern.p, dtype=_dev.torch().float64, device="cuda")
    else:
        coeffs = _dev.to_device(v).clone()
    return KronSumRep(pattern=pattern, coeffs=_dev.like_input(ref, coeffs),
                      terms=_dev.like_input(ref, terms))


def _outer_terms(xd, zd, gcols=None):
    """terms[j] = (x * g[:, j]) @ z^T on DMMA; gcols=None means g = I."""
    m, r = int(xd.shape[0]), int(xd.shape[1])
    n = int(zd.shape[0])
    out = _dev.empty((r, m, n))
    d = N.GemmDesc()
    if gcols is None:
        # rank-1 outer products: batch j, reduction of length 1
        d.M, d.N, d.Kin, d.Kout, d.batch = m, n, 1, 1, r
        d.A, d.sAm, d.sAki, d.sAb = _dev.ptr(xd), r, 1, 1
        d.B, d.sBn, d.sBki, d.sBb = _dev.ptr(zd), r, 1, 1
    else:
        # D_j = X diag(g[:, j]) Z^T: the diagonal rides on the A-scale along r
        # (gcols is g^T, row j = g[:, j])
        d.M, d.N, d.Kin, d.Kout, d.batch = m, n, r, 1, r
        d.A, d.sAm, d.sAki, d.sAb = _dev.ptr(xd), r, 1, 0
        d.B, d.sBn, d.sBki, d.sBb = _dev.ptr(zd), r, 1, 0
        d.ascale, d.s_ascale_ko, d.s_ascale_b = _dev.ptr(gcols), 0, r
    d.C, d.sCm, d.sCn, d.sCb = _dev.ptr(out), n, 1, m * n
    d.alpha, d.beta = 1.0, 0.0
    ws = _dev.workspace(N.load().bt_gemm_f64_ws_bytes(C.byref(d)))
    N.call("bt_gemm_f64", C.byref(d), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    return out


def kron_sum_from_kruskal(k: KruskalRep, pattern: BlockPattern, split: str = "factor"):
    """reconstruct.py:192-226."""
    if k.dims != (pattern.m, pattern.p, pattern.n):
        raise ShapeError(f"CP dims {k.dims} do not match pattern "
                         f"({pattern.m}, {pattern.p}, {pattern.n})")
    r = k.rank
    xd, zd = _dev.to_device(k.x), _dev.to_device(k.z)
    if split == "factor":
        f = _dev.to_device(k.y).clone()
        terms = _outer_terms(xd, zd)
    elif split == "qr":
        if k.y.shape[0] < r:
            raise ShapeError("qr split needs p >= r")
        fq, ry = qr_thin(_dev.to_device(k.y))
        f = fq
        terms = _outer_terms(xd, zd, gcols=ry.contiguous())  # row j of ry = g[:, j]
    else:
        raise ValueError(f"unknown split {split!r}")
    return KronSumRep(pattern=pattern, coeffs=_dev.like_input(k.x, f),
                      terms=_dev.like_input(k.x, terms))


def blr_from_tucker(t: TuckerRep, pattern: BlockPattern) -> BlockLowRankRep:
    """reconstruct.py:229-240: middles[k] = sum_j V[k, j] core[:, j, :]."""
    u, v, w = _tucker_side(t, pattern)
    tt = _dev.torch()
    left = tt.eye(pattern.m, dtype=tt.float64, device="cuda") if u is None else _dev.to_device(u)
    right = tt.eye(pattern.n, dtype=tt.float64, device="cuda") if w is None else _dev.to_device(w)
    cd = _dev.to_device(t.core)
    if v is not None:
        cd = ttm_dev(cd, 2, _dev.to_device(v), int(v.shape[0]))
    mids = cd.permute(1, 0, 2).contiguous()
    ref = t.core
    return BlockLowRankRep(pattern=pattern, left=_dev.like_input(ref, left.clone()),
                           right=_dev.like_input(ref, right.clone()),
                           middles=_dev.like_input(ref, mids))


def blr_from_kruskal(k: KruskalRep, pattern: BlockPattern) -> BlockLowRankRep:
    """reconstruct.py:243-263: thin QR of the outer factors, middles
    R_x diag(Y[k, :]) R_z^T."""
    if k.dims != (pattern.m, pattern.p, pattern.n):
        raise ShapeError(f"CP dims {k.dims} do not match pattern "
                         f"({pattern.m}, {pattern.p}, {pattern.n})")
    r = k.rank
    if pattern.m < r or pattern.n < r:
        raise ShapeError(f"CP rank {r} exceeds a block extent ({pattern.m} x {pattern.n})")
    qx, rx = qr_thin(_dev.to_device(k.x))
    qz, rz = qr_thin(_dev.to_device(k.z))
    yd = _dev.to_device(k.y)
    # middles[kk] = (rx * y[kk, :]) @ rz^T : rx scaled along r by y[kk] (A-scale)
    p = pattern.p
    out = _dev.empty((p, r, r))
    d = N.GemmDesc()
    d.M, d.N, d.Kin, d.Kout, d.batch = r, r, r, 1, p
    d.A, d.sAm, d.sAki, d.sAb = _dev.ptr(rx), r, 1, 0
    d.ascale, d.s_ascale_ko, d.s_ascale_b = _dev.ptr(yd), 0, r
    d.B, d.sBn, d.sBki, d.sBb = _dev.ptr(rz), r, 1, 0
    d.C, d.sCm, d.sCn, d.sCb = _dev.ptr(out), r, 1, r * r
    d.alpha, d.beta = 1.0, 0.0
    ws = _dev.workspace(N.load().bt_gemm_f64_ws_bytes(C.byref(d)))
    N.call("bt_gemm_f64", C.byref(d), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    ref = k.x
    return BlockLowRankRep(pattern=pattern, left=_dev.like_input(ref, qx),
                           right=_dev.like_input(ref, qz), middles=_dev.like_input(ref, out))


# ---------------------------------------------------------------------------
# actions
# ---------------------------------------------------------------------------


def _rhs_block(x, qn):
    """(nrhs, q*n) contiguous device block from a vector or (q*n, nrhs) array."""
    if x.ndim == 1:
        if tuple(x.shape) != (qn,):
            raise ShapeError(f"vector length {tuple(x.shape)} != {(qn,)}")
        return _dev.to_device(x).reshape(1, qn), 1
    if x.ndim != 2 or x.shape[0] != qn:
        raise ShapeError(f"right-hand sides of shape {tuple(x.shape)} != ({qn}, nrhs)")
    xd = _dev.to_device(x)
    return _dev.transpose(xd), int(x.shape[1])


def flops_kron(pat: BlockPattern, r: int) -> int:
    nnz = sum(pat.counts)
    return r * (2 * pat.m * pat.n * pat.q + 2 * pat.m * nnz)


def flops_blr(pat: BlockPattern, rl: int, rr: int) -> int:
    return 2 * pat.n * rr * pat.q + sum(pat.counts) * 2 * rl * rr + 2 * pat.m * rl * pat.ell


def matvec(rep, x, counter: FlopCounter | None = None):
    """reconstruct.py:271-315 without densifying; x is (q*n,) or (q*n, nrhs)."""
    pat = rep.pattern
    qn = pat.q * pat.n
    xd, nrhs = _rhs_block(x, qn)
    d, s, h = pat.device()
    y = _dev.empty((nrhs, pat.ell * pat.m))
    lib = N.load()
    if isinstance(rep, KronSumRep):
        r = rep.n_terms
        coeffs = _dev.to_device(rep.coeffs)
        terms = _dev.to_device(rep.terms)
        ws = _dev.workspace(lib.bt_matvec_kron_ws_bytes(C.byref(s), r, nrhs))
        N.call("bt_matvec_kron_f64", C.byref(s), _dev.ptr(d["row_ptr"]), _dev.ptr(d["row_cells"]),
               _dev.ptr(coeffs), _dev.ptr(terms), r, _dev.ptr(xd), nrhs, _dev.ptr(y),
               _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
        if counter is not None:
            counter.add(nrhs * flops_kron(pat, r))
    elif isinstance(rep, BlockLowRankRep):
        left = _dev.to_device(rep.left)
        right = _dev.to_device(rep.right)
        mids = _dev.to_device(rep.middles)
        rl, rr = int(left.shape[1]), int(right.shape[1])
        ws = _dev.workspace(lib.bt_matvec_blr_ws_bytes(C.byref(s), rl, rr, nrhs))
        N.call("bt_matvec_blr_f64", C.byref(s), _dev.ptr(d["row_ptr"]), _dev.ptr(d["row_cells"]),
               _dev.ptr(left), rl, _dev.ptr(right), rr, _dev.ptr(mids), _dev.ptr(xd), nrhs,
               _dev.ptr(y), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
        if counter is not None:
            counter.add(nrhs * flops_blr(pat, rl, rr))
    else:
        raise TypeError(f"unsupported representation {type(rep).__name__}")
    out = y[0] if x.ndim == 1 else _dev.transpose(y)
    return _dev.like_input(x, out)


def _dense_items(rep):
    pat = rep.pattern
    if isinstance(rep, KronSumRep):
        coeffs = _dev.to_device(rep.coeffs)
        terms = _dev.to_device(rep.terms).reshape(rep.n_terms, -1)
        items = L.gemm_dev(coeffs, terms)            # (p, m*n)
        return items.reshape(pat.p, pat.m, pat.n)
    if isinstance(rep, BlockLowRankRep):
        left = _dev.to_device(rep.left)
        right = _dev.to_device(rep.right)
        mids = _dev.to_device(rep.middles)
        p, rl, rr = (int(s) for s in mids.shape)
        # t1[k] = mids[k] @ right^T  (p, rl, n) ; items[k] = left @ t1[k]
        t1 = ttm_dev(mids, 3, right, int(right.shape[0]))
        t2 = ttm_dev(t1, 2, left, int(left.shape[0]))
        return t2
    raise TypeError(f"unsupported representation {type(rep).__name__}")


def densify(rep):
    """reconstruct.py:318-335 (guarded by DENSIFY_LIMIT)."""
    pat = rep.pattern
    total = pat.ell * pat.m * pat.q * pat.n
    if total > DENSIFY_LIMIT:
        raise ShapeError(f"dense result would hold {total} entries (limit {DENSIFY_LIMIT})")
    items = _dense_items(rep)
    ref = rep.coeffs if isinstance(rep, KronSumRep) else rep.middles
    return _dev.like_input(ref, struct_expand(pat, items))


def error_fro(a, rep) -> float:
    """reconstruct.py:338-345: ||a - densify(rep)|| / ||a||."""
    if tuple(a.shape) != rep.shape:
        raise ShapeError(f"matrix shape {tuple(a.shape)} != representation shape {rep.shape}")
    ad = _dev.to_device(a)
    base = fro_norm_dev(ad)
    if base == 0.0:
        raise ShapeError("relative error undefined for a zero matrix")
    dense = densify(rep)
    diff = _dev.empty(tuple(ad.shape))
    N.call("bt_axpby_f64", int(ad.numel()), 1.0, _dev.ptr(ad), -1.0,
           _dev.ptr(_dev.to_device(dense)), _dev.ptr(diff), _dev.stream())
    return fro_norm_dev(diff) / base


def c_term_dense(rep: KronSumRep, j: int):
    """Dense C_j (reconstruct.py:348-350)."""
    coeffs = rep.coeffs
    col = coeffs[:, j]
    return struct_scalars(rep.pattern, col if _dev.is_device(col) else np.ascontiguousarray(col))
