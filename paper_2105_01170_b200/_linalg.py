"""Device linear-algebra helpers shared by decomp / psd / reconstruct:
unfolding Grams (DMMA SYRK), the symmetric eigensolver with the reference's
sign rule, truncated SVD / mode bases built on them, thin QR."""

from __future__ import annotations

import ctypes as C

from . import _dev
from . import _native as N
from .errors import ShapeError


def _dims(xd):
    dims = tuple(int(s) for s in xd.shape)
    return dims, (C.c_int64 * len(dims))(*dims)


def unfold_gram_dev(xd, mode: int):
    """G = X_(mode) X_(mode)^T (n x n) without forming the unfolding."""
    dims, cd = _dims(xd)
    n = dims[mode - 1]
    g = _dev.empty((n, n))
    ws = _dev.workspace(N.load().bt_unfold_gram_ws_bytes(cd, len(dims), mode))
    N.call("bt_unfold_gram_f64", _dev.ptr(xd), cd, len(dims), mode, _dev.ptr(g), _dev.ptr(ws),
           int(ws.numel()) * 8, _dev.stream())
    return g


def eigh_dev(gd):
    """(w, V): eigenvalues descending, eigenvectors as columns of V, each
    sign-normalised (largest-|.| entry positive, first on ties)."""
    n = int(gd.shape[0])
    if tuple(gd.shape) != (n, n):
        raise ShapeError("eigh expects a square matrix")
    w = _dev.empty((n,))
    v = _dev.empty((n, n))
    ws = _dev.workspace(N.load().bt_syevd_ws_bytes(n))
    N.call("bt_syevd_f64", _dev.ptr(gd.contiguous()), n, _dev.ptr(w), _dev.ptr(v), _dev.ptr(ws),
           int(ws.numel()) * 8, _dev.stream())
    return w, v


def mode_basis_dev(xd, mode: int, r: int, extra_mode: int | None = None):
    """Leading r left singular vectors of unfold(x, mode) (decomp.py:220-234),
    complete to r columns when r exceeds the unfolding's column count (the
    Gram's eigenbasis is complete).  extra_mode: basis of the column
    concatenation [unfold(x, mode), unfold(x, extra_mode)] (tucker_partial
    shared_from="concat"), whose Gram is the sum of the two Grams."""
    g = unfold_gram_dev(xd, mode)
    if extra_mode is not None:
        g = g + unfold_gram_dev(xd, extra_mode)
    _, v = eigh_dev(g)
    return v[:, :r].contiguous()


def svd_truncated_dev(ad, r: int):
    """(u, s, v) of a matrix on device via the Gram of its short side."""
    m, n = int(ad.shape[0]), int(ad.shape[1])
    t = _dev.torch()
    if m <= n:
        w, uu = eigh_dev(unfold_gram_dev(ad, 1))
        u = uu[:, :r].contiguous()
        s = t.sqrt(t.clamp(w[:r], min=0.0))
        v = _gemm_tn(ad, u)                       # a^T u   (n x r)
        v = v / t.where(s > 0, s, t.ones_like(s))
        return u, s, v
    w, vv = eigh_dev(unfold_gram_dev(ad, 2))
    v = vv[:, :r].contiguous()
    s = t.sqrt(t.clamp(w[:r], min=0.0))
    u = _gemm_nn(ad, v) / t.where(s > 0, s, t.ones_like(s))
    # sign rule on u, compensated in v (decomp.py:176-179)
    lead = t.argmax(t.abs(u), dim=0)
    sg = t.sign(u[lead, t.arange(r, device=u.device)])
    sg = t.where(sg == 0, t.ones_like(sg), sg)
    return (u * sg).contiguous(), s, (v * sg).contiguous()


def _gemm(a_ptr, M, N_, K, sAm, sAk, b_ptr, sBk, sBn, out):
    d = N.GemmDesc()
    d.M, d.N, d.Kin, d.Kout, d.batch = M, N_, K, 1, 1
    d.A, d.sAm, d.sAki = a_ptr, sAm, sAk
    d.B, d.sBn, d.sBki = b_ptr, sBn, sBk
    d.C, d.sCm, d.sCn = _dev.ptr(out), N_, 1
    d.alpha, d.beta = 1.0, 0.0
    ws = _dev.workspace(N.load().bt_gemm_f64_ws_bytes(C.byref(d)))
    N.call("bt_gemm_f64", C.byref(d), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    return out


def gemm_dev(a, b, ta=False, tb=False):
    """op(a) @ op(b) on the DMMA engine (contiguous inputs)."""
    a = a.contiguous()
    b = b.contiguous()
    M = a.shape[1] if ta else a.shape[0]
    K = a.shape[0] if ta else a.shape[1]
    Nn = b.shape[0] if tb else b.shape[1]
    out = _dev.empty((M, Nn))
    sAm, sAk = (1, a.shape[1]) if ta else (a.shape[1], 1)
    sBk, sBn = (1, b.shape[1]) if tb else (b.shape[1], 1)
    return _gemm(_dev.ptr(a), int(M), int(Nn), int(K), int(sAm), int(sAk), _dev.ptr(b), int(sBk),
                 int(sBn), out)


def _gemm_tn(a, b):
    return gemm_dev(a, b, ta=True)


def _gemm_nn(a, b):
    return gemm_dev(a, b)


def qr_thin_dev(ad):
    """Thin QR with nonnegative diag(R) on device (single-CTA Householder)."""
    m, n = int(ad.shape[0]), int(ad.shape[1])
    q = _dev.empty((m, n))
    r = _dev.empty((n, n))
    ws = _dev.workspace(N.load().bt_qr_thin_ws_bytes(m, n))
    N.call("bt_qr_thin_f64", _dev.ptr(ad.contiguous()), m, n, _dev.ptr(q), _dev.ptr(r),
           _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    return q, r
