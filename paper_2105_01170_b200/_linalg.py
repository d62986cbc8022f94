"""Device linear-algebra helpers shared by decomp / psd / reconstruct:
unfolding Grams (DMMA SYRK), the symmetric eigensolver with the reference's
sign rule, truncated SVD / mode bases built on them, thin QR."""

from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

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


SMALL_EIG = 96      # one-CTA Jacobi up to this size


def eigh_dev(gd, nvec: int | None = None, tau: float = -1.0):
    """(w, V): eigenvalues descending, eigenvectors as columns of V, each
    sign-normalised (largest-|.| entry positive, first on ties).  With nvec
    (< n, n > 96) only the leading nvec pairs are computed (tridiagonal
    path; vectors only for eigenvalues above tau * |w[0]| when tau >= 0, the
    rest zero); otherwise the full spectrum (Jacobi)."""
    n = int(gd.shape[0])
    if tuple(gd.shape) != (n, n):
        raise ShapeError("eigh expects a square matrix")
    if nvec is not None and SMALL_EIG < n <= 3200 and int(nvec) < n:
        nv = max(1, int(nvec))
        w = _dev.empty((nv,))
        v = _dev.empty((n, nv))
        ws = _dev.workspace(N.load().bt_syevx_ws_bytes(n, nv))
        N.call("bt_syevx_f64", _dev.ptr(gd.contiguous()), n, nv, float(tau), _dev.ptr(w),
               _dev.ptr(v), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
        return w, v
    w = _dev.empty((n,))
    v = _dev.empty((n, n))
    ws = _dev.workspace(N.load().bt_syevd_ws_bytes(n))
    N.call("bt_syevd_f64", _dev.ptr(gd.contiguous()), n, _dev.ptr(w), _dev.ptr(v), _dev.ptr(ws),
           int(ws.numel()) * 8, _dev.stream())
    return w, v


_DEBUG = bool(os.environ.get("BT_BASIS_DEBUG"))
SUBSPACE = os.environ.get("BT_SUBSPACE", "1") != "0"
# BT_SUB_DIRECT=1: a cold block of >= 48 wanted pairs at n <= 1536 goes to the
# tridiagonal solver instead of the oversampled subspace iteration (C3 mode 1:
# 8.1 ms subspace vs 15.9 ms tridiagonal)
_SUB_DIRECT = os.environ.get("BT_SUB_DIRECT", "0") == "1"
# BT_REFINE=0: warm-started bases (HOOI) take the Gram deflation passes too
REFINE = os.environ.get("BT_REFINE", "1") != "0"
SUB_OVERSAMPLE = 16
SUB_MAX_BLOCK = 96     # Rayleigh-Ritz matrices stay on the one-CTA Jacobi path


def _leading_subspace(gd, need: int, tau: float, start=None, hint=None):
    """Leading eigenpairs of a symmetric n x n Gram by block subspace
    iteration with Rayleigh-Ritz (bt_leading_subspace_f64: GEMMs, column-
    scaled SVQB and the one-CTA Jacobi on the b x b projection, driven from
    the library's host side), b = min(need, hint, 80) + 16 columns (a cold
    block of >= 48 wanted pairs: + up to need / 2, at most 96).

    Returns (w, v, k): the b Ritz values (descending, device), Ritz vectors
    (n x b, sign-normalised) and the count k of leading pairs that are
    (i) above tau * w[0] and (ii) converged to a residual
    ||G v - theta v|| <= 32 eps theta_1 -- at most b - 16, so every
    eigenvalue above the cut is known to be captured.  None when the
    iteration did not converge or was predicted too slow (the caller falls
    back to bt_syevx_f64).  Accuracy per accepted pair is the Gram
    eigensolver's (residual / gap); the deflation passes of mode_basis_dev
    handle the rest."""
    n = int(gd.shape[0])
    h = 0 if hint is None else int(hint)
    wsb = N.load().bt_leading_subspace_ws_bytes(n, int(need), h)
    if wsb <= 0:
        return None
    # the library's block is at most SUB_MAX_BLOCK columns (a cold block of
    # many wanted pairs oversamples by up to half; the call reports its size)
    b = min(n, SUB_MAX_BLOCK)
    ws = _dev.workspace(wsb)
    w = _dev.empty((b,))
    vbuf = _dev.empty((n * b,))
    bq, k, st = C.c_int64(0), C.c_int64(0), C.c_int(0)
    sp, sc = (0, 0) if start is None else (_dev.ptr(start), int(start.shape[1]))
    N.call("bt_leading_subspace_f64", _dev.ptr(gd), n, int(need), float(tau), sp or None, sc, h,
           _dev.ptr(w), _dev.ptr(vbuf), C.byref(bq), C.byref(k), C.byref(st), _dev.ptr(ws),
           int(ws.numel()) * 8, _dev.stream())
    if st.value != 0:
        return None
    nb = int(bq.value)
    return w[:nb], vbuf[:n * nb].view(n, nb), int(k.value)


NOISE_REL = 1e-22    # remainder eigenvalue below this * lambda_1 (sigma < 1e-11 sigma_1)
RESOLVE_TAU = 1e-6   # per pass: eigenvectors with lambda > tau * lambda_max are kept (cut accuracy ~eps/tau)


def _gram_modes(xd, modes, reduce=None):
    g = None
    for m in modes:
        gm = unfold_gram_dev(xd, m)
        g = gm if g is None else _axpby(1.0, g, 1.0, gm)
    if reduce is not None:
        reduce(g)
    return g


def _axpby(alpha, x, beta, y):
    z = _dev.empty(tuple(x.shape))
    N.call("bt_axpby_f64", int(x.numel()), float(alpha), _dev.ptr(x), float(beta), _dev.ptr(y),
           _dev.ptr(z), _dev.stream())
    return z


def _residual(xd, mode, basis):
    """x - (x x_mode B^T) x_mode B : the part of unfold(x, mode) orthogonal to B."""
    from .tensor import ttm_dev

    k = int(basis.shape[1])
    y = ttm_dev(xd, mode, basis, k, transpose=True)
    p = ttm_dev(y, mode, basis, int(basis.shape[0]))
    return _axpby(1.0, xd, -1.0, p)


def _orth_normalize(basis, new):
    """new - B (B^T new), columns renormalised (device)."""
    out = _axpby(1.0, new, -1.0, gemm_dev(basis, gemm_dev(basis, new, ta=True)))
    N.call("bt_col_normalize_f64", _dev.ptr(out), int(out.shape[0]), int(out.shape[1]),
           _dev.stream())
    return out


def _orthonormalize_block(y):
    """Symmetric (Loewdin) orthonormalisation Y (Y^T Y)^{-1/2} of a thin
    block on device -- GEMMs plus the one-CTA eigensolver; applied twice by
    the caller (like CholeskyQR2) for orthogonality to working precision."""
    w, v = eigh_dev(gemm_dev(y, y, ta=True))
    if float(_dev.to_host(w).min()) <= 0.0:
        raise RuntimeError("orthonormalisation of a rank-deficient block")
    s = _dev.empty(tuple(w.shape))
    N.call("bt_inv_sqrt_f64", _dev.ptr(w), int(w.numel()), _dev.ptr(s), _dev.stream())
    # Y V diag(lambda^-1/2): the diagonal rides on the engine's B-scale
    k = int(v.shape[0])
    m = int(y.shape[0])
    out = _dev.empty((m, k))
    d = N.GemmDesc()
    d.M, d.N, d.Kin, d.Kout, d.batch = m, k, k, 1, 1
    d.A, d.sAm, d.sAki = _dev.ptr(y), k, 1
    d.B, d.sBn, d.sBki = _dev.ptr(v), 1, k
    d.bscale, d.s_scale_ko = _dev.ptr(s), 0
    d.C, d.sCm, d.sCn = _dev.ptr(out), k, 1
    d.alpha, d.beta = 1.0, 0.0
    ws = _dev.workspace(N.load().bt_gemm_f64_ws_bytes(C.byref(d)))
    N.call("bt_gemm_f64", C.byref(d), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    return out


def gaussian_dev(rows: int, cols: int, key: int):
    """Deterministic N(0,1) block on the device (Philox, index-addressable)."""
    out = _dev.empty((rows, cols))
    N.call("bt_fill_normal_f64", _dev.ptr(out), rows * cols, int(key), _dev.stream())
    return out


def _complete(basis, g, need: int, block: int = 32):
    """``need`` orthonormal columns orthogonal to ``basis`` from a
    deterministic Gaussian block: project out the accepted columns, then
    thin QR (CholeskyQR2 on the engine), twice for reorthogonalisation, and
    sign-normalise.  Used once the remainder is at rounding level (or
    exhausted), where any orthonormal completion is as good as LAPACK's.
    Falls back to blockwise Loewdin orthonormalisation for thin blocks."""
    t = _dev.torch()
    n = int(g.shape[0])
    k = 0 if basis is None else int(basis.shape[1])
    if need <= 1024 and k + need <= n:
        out = _dev.empty((n, need))
        st = C.c_int(1)
        ws = _dev.workspace(N.load().bt_complete_basis_ws_bytes(n, k, need))
        N.call("bt_complete_basis_f64", None if basis is None else _dev.ptr(basis.contiguous()), n, k,
               need, 12345, _dev.ptr(out), C.byref(st), _dev.ptr(ws), int(ws.numel()) * 8,
               _dev.stream())
        if st.value == 0:
            return out
    y = gaussian_dev(n, need, 12345)
    # blocks of <= 32 Gaussian columns: project out everything accepted so
    # far (twice), then column-scaled CholeskyQR2 with the one-warp Cholesky
    # (a Gaussian block is well conditioned); the larger paths below only run
    # if a block is rejected
    cur = basis
    outs = []
    ok = True
    for j0 in range(0, need, 32):
        blk = y[:, j0:j0 + 32].contiguous()
        for _ in range(2):
            if cur is not None:
                blk = _axpby(1.0, blk, -1.0, gemm_dev(cur, gemm_dev(cur, blk, ta=True)))
        qr = _qr_colscaled(blk) if int(blk.shape[1]) <= n else None
        if qr is None:
            ok = False
            break
        blk = qr[0]
        if cur is not None:     # re-orthogonalise against the accepted basis once more
            blk = _axpby(1.0, blk, -1.0, gemm_dev(cur, gemm_dev(cur, blk, ta=True)))
            qr = _qr_colscaled(blk)
            if qr is None:
                ok = False
                break
            blk = qr[0]
        outs.append(blk)
        cur = blk if cur is None else t.cat([cur, blk], dim=1).contiguous()
    if ok and outs:
        out = t.cat(outs, dim=1).contiguous()
        N.call("bt_sign_fix_f64", _dev.ptr(out), n, int(need), _dev.stream())
        return out
    if need >= 8:
        for _ in range(2):
            if basis is not None:
                y = _axpby(1.0, y, -1.0, gemm_dev(basis, gemm_dev(basis, y, ta=True)))
            y, _ = qr_thin_dev(y)
        out = y.contiguous()
        N.call("bt_sign_fix_f64", _dev.ptr(out), n, int(need), _dev.stream())
        return out
    cur = basis
    outs = []
    for j0 in range(0, need, block):
        blk = y[:, j0:j0 + block].contiguous()
        for _ in range(2):
            if cur is not None:
                blk = _axpby(1.0, blk, -1.0, gemm_dev(cur, gemm_dev(cur, blk, ta=True)))
            blk = _orthonormalize_block(blk)
        outs.append(blk)
        cur = blk if cur is None else t.cat([cur, blk], dim=1).contiguous()
    out = t.cat(outs, dim=1).contiguous()
    N.call("bt_sign_fix_f64", _dev.ptr(out), n, int(need), _dev.stream())
    return out


def _next_pass_hint(wh, k: int):
    """Predicted number of directions the next deflation pass resolves: the
    eigen/Ritz values below this pass's cut approximate the remainder's
    spectrum, so the next pass keeps about those above RESOLVE_TAU times the
    first of them.  Sizes the next subspace block only (acceptance is always
    by residual)."""
    tail = np.asarray(wh[k:], dtype=np.float64)
    if tail.size >= 6 and tail[0] > 0.0:
        cnt = int(np.sum(tail > RESOLVE_TAU * tail[0]))
        if cnt < tail.size - 4:
            return cnt + 2
    # unconverged Ritz values above the cut (or too short a tail): passes of
    # a steadily decaying spectrum resolve about as many as this one did
    return k + 4


def tsqr_dev(ad):
    """Householder-quality thin QR of a tall block with <= 32 columns (TSQR on
    the GPU; falls back to the one-CTA Householder kernel past its row cap)."""
    m, n = int(ad.shape[0]), int(ad.shape[1])
    if n > 32 or m < n or m > 6656:
        return _householder_qr(ad)
    q, r = _dev.empty((m, n)), _dev.empty((n, n))
    ws = _dev.workspace(N.load().bt_tsqr_ws_bytes(m, n))
    N.call("bt_tsqr_f64", _dev.ptr(ad.contiguous()), m, n, _dev.ptr(q), _dev.ptr(r), _dev.ptr(ws),
           int(ws.numel()) * 8, _dev.stream())
    return q, r


def _qr_colscaled_lazy(z):
    """(q, r, chk) of a tall block with <= 32 columns by column-scaled
    CholeskyQR2: Y = Z D (unit columns), two CholeskyQR passes,
    R = L2^T L1^T D^-1.  Accurate whenever Z's columns are already nearly
    orthogonal up to their scales (a refinement step near convergence:
    Z = A^T V ~ W Sigma).  No host read: chk is a device vector [pivot flag
    of pass 1, of pass 2, smallest column norm] and the factors are valid iff
    it reads [0, 0, > 0] (_colscaled_ok).  None when the shape is not
    eligible."""
    m, n = int(z.shape[0]), int(z.shape[1])
    if n > 32 or m < n:
        return None
    t = _dev.torch()
    nrm = _dev.empty((n,))
    N.call("bt_col_norms_f64", _dev.ptr(z), m, n, _dev.ptr(nrm), _dev.stream())
    dinv = 1.0 / nrm
    y = _dev.empty((m, n))
    N.call("bt_diag_scale_f64", _dev.ptr(z), m, n, None, _dev.ptr(dinv), _dev.ptr(y), _dev.stream())
    flags = t.zeros(2, dtype=t.int32, device="cuda")
    r = None
    for it in range(2):
        g = gemm_dev(y, y, ta=True)
        lt, linvt = _dev.empty((n, n)), _dev.empty((n, n))
        N.call("bt_chol_small_f64", _dev.ptr(g), n, _dev.ptr(lt), _dev.ptr(linvt),
               flags.data_ptr() + 4 * it, _dev.stream())
        y = gemm_dev(y, linvt)
        r = lt if r is None else gemm_dev(lt, r)
    rr = _dev.empty((n, n))
    N.call("bt_diag_scale_f64", _dev.ptr(r), n, n, None, _dev.ptr(nrm), _dev.ptr(rr), _dev.stream())
    chk = t.cat([flags.to(t.float64), nrm.min().reshape(1)])
    return y, rr, chk


def _colscaled_ok(chk3) -> bool:
    return chk3[0] == 0.0 and chk3[1] == 0.0 and chk3[2] > 0.0


def _qr_colscaled(z):
    """_qr_colscaled_lazy with its check read here: (q, r), or None when a
    pivot or a zero column rejects the block (the caller takes TSQR)."""
    out = _qr_colscaled_lazy(z)
    if out is None or not _colscaled_ok(_dev.to_host(out[2])):
        return None
    return out[0], out[1]


def _qr_refine(z):
    out = _qr_colscaled(z)
    return out if out is not None else tsqr_dev(z)


def _qr_refine_lazy(z):
    """(q, r, chk): the column-scaled CholeskyQR2 with its check left on the
    device, or TSQR (chk None) for shapes it does not take."""
    out = _qr_colscaled_lazy(z)
    if out is not None:
        return out
    q, r = tsqr_dev(z)
    return q, r, None


def svd_small_dev(m):
    """(u, s, v) of a small square matrix (n <= 32) by one-warp one-sided
    Jacobi (bt_svd_small_f64): s descending, sign rule on u."""
    n = int(m.shape[0])
    u, v, s = _dev.empty((n, n)), _dev.empty((n, n)), _dev.empty((n,))
    N.call("bt_svd_small_f64", _dev.ptr(m.contiguous()), n, _dev.ptr(u), _dev.ptr(s), _dev.ptr(v),
           _dev.stream())
    return u, s, v


REFINE_MAX_STEPS = 4
REFINE_TOL = 1e-12     # max change of a resolved vector between two refinement steps
REFINE_NUMEL = 1 << 26


def _refine_basis_qr(xd, mode: int, r: int, start):
    """Leading r <= 32 left singular vectors of A = unfold(x, mode) from a
    close warm start V (HOOI's previous sweep) without a Gram: subspace
    iteration  Z = A^T V -> Q_Z (Householder) -> W = A Q_Z -> Q_W R_W
    (Householder) -> R_W = U_R S V_R^T (one-sided Jacobi) -> V = Q_W U_R.
    Every product is a GEMM of A or A^T with an orthonormal block, so a
    singular direction is resolved to ~eps sigma_1 / gap instead of the
    Gram's ~eps sigma_1^2 / gap^2 -- one pass resolves what the Gram needs
    one deflation pass per ~6 orders of magnitude for (C3 mode 2: 5 passes).
    Returns None when it does not settle within REFINE_MAX_STEPS steps (the
    caller then runs the deflation passes)."""
    t = _dev.torch()
    dims = tuple(int(v) for v in xd.shape)
    n = dims[mode - 1]
    cols = xd.numel() // max(n, 1)
    if (r > 32 or n < r or cols < 2 * r or xd.numel() > REFINE_NUMEL or start is None
            or int(start.shape[1]) != r):
        return None
    # A = unfold(x, mode) with the other indices in C order as columns
    a = xd.movedim(mode - 1, 0).reshape(n, -1).contiguous()
    v = start.contiguous()
    prev = None
    for _ in range(REFINE_MAX_STEPS):
        # one host read per step: the QR checks, the singular values and the
        # change against the previous step come back together
        zq = _qr_refine_lazy(gemm_dev(a, v, ta=True))          # A^T V -> Q_Z
        wq = _qr_refine_lazy(gemm_dev(a, zq[0]))               # A Q_Z -> Q_W R_W
        ur, sv, _ = svd_small_dev(wq[1])
        vn = gemm_dev(wq[0], ur)
        N.call("bt_sign_fix_f64", _dev.ptr(vn), n, r, _dev.stream())
        parts = [c for c in (zq[2], wq[2]) if c is not None]
        nchk = len(parts)
        parts.append(sv)
        if prev is not None:
            parts.append((vn - prev).abs().amax(dim=0))
        host = _dev.to_host(t.cat(parts))
        if not all(_colscaled_ok(host[3 * i:3 * i + 3]) for i in range(nchk)):
            # a CholeskyQR pivot rejected its block: redo the step on TSQR
            qz, _ = _qr_refine(gemm_dev(a, v, ta=True))
            qw, rw = _qr_refine(gemm_dev(a, qz))
            ur, sv, _ = svd_small_dev(rw)
            vn = gemm_dev(qw, ur)
            N.call("bt_sign_fix_f64", _dev.ptr(vn), n, r, _dev.stream())
            sh = _dev.to_host(sv)
            diff = None if prev is None else _dev.to_host((vn - prev).abs().amax(dim=0))
        else:
            sh = host[3 * nchk:3 * nchk + r]
            diff = None if prev is None else host[3 * nchk + r:]
        v = vn
        if not sh[0] > 0:
            return None
        if diff is not None:
            # a vector is resolved to ~eps sigma_1 / sigma_k: compare each with
            # the previous step at that accuracy (REFINE_TOL floor); the ones
            # below 1e-13 sigma_1 are noise either way
            live = sh > 1e-13 * sh[0]
            tol = np.maximum(REFINE_TOL, 64 * 2.2e-16 * sh[0] / np.maximum(sh, 1e-300))
            if np.all(diff[live] <= tol[live]):
                return v
        prev = v
    return None


def mode_basis_dev(xd, mode: int, r: int, extra_mode: int | None = None, max_passes: int = 16,
                   reduce=None, start=None):
    """Leading r left singular vectors of unfold(x, mode) (decomp.py:220-234),
    sign rule included.  extra_mode: basis of the column concatenation
    [unfold(x, mode), unfold(x, extra_mode)] (tucker_partial
    shared_from="concat"), whose Gram is the sum of the two Grams.

    A Gram + eigensolver pass determines eigenvectors to ~eps*lambda_max/gap,
    so each pass keeps only the directions with lambda > RESOLVE_TAU *
    lambda_max of the current Gram, deflates them out of the tensor and
    re-Grams the remainder (SVD-grade accuracy for the fast-decaying spectra
    of C2/C3).  Once the remainder is at rounding level the
    basis is completed orthonormally (full_matrices completion, too).

    start: optional (n x k) basis close to the answer (HOOI's previous sweep);
    it seeds the first pass's subspace iteration.

    reduce: in-place cross-rank sum applied to every Gram, for a tensor
    sharded along a mode other than ``mode`` (each rank's Gram is then a
    partial sum; the deflation residual is slab-local).  The eigensolves are
    replicated and deterministic, so every rank takes the same branches."""
    modes = [mode] if extra_mode is None else [mode, extra_mode]
    t = _dev.torch()
    n = int(xd.shape[mode - 1])
    if extra_mode is None and reduce is None and REFINE and r <= 32 and n >= 2 * r:
        # warm start (HOOI's previous basis) or, cold, a Gaussian block: the
        # Gram-free subspace iteration settles in a few steps when the
        # spectrum decays fast past r (C3 mode 2: ~1e-3 per index) and hands
        # back to the deflation passes otherwise
        s0 = start if start is not None else gaussian_dev(n, r, 97531)
        v = _refine_basis_qr(xd, mode, r, s0)
        if v is not None:
            if _DEBUG:
                print(f"[mode_basis n={n} r={r}] QR refinement from the "
                      f"{'warm' if start is not None else 'Gaussian'} start", file=sys.stderr)
            return v
    g = _gram_modes(xd, modes, reduce)
    basis = None
    top = None
    hint = None
    for _ in range(max_passes):
        have = 0 if basis is None else int(basis.shape[1])
        need = r - have
        if need <= 0:
            break
        cold = start is None or basis is not None
        # a cold block of >= 48 wanted pairs oversamples to 96 columns and
        # runs simultaneous iteration with two G products per CholeskyQR and
        # a Rayleigh-Ritz only at the start and the end (subspace.cu); C3 mode
        # 1 (64 of 1024, lambda_97 / lambda_64 ~ 0.31): 28 steps, 8.1 ms
        # against 15.9 ms for the tridiagonal solver
        direct = (cold and hint is None and need >= 48 and n <= 1536 and _SUB_DIRECT)
        # a first pass that cannot hold every wanted pair in one block (C2
        # mode 2: 400 of 2047) starts with a 32-pair block: a pass keeps only
        # the pairs above RESOLVE_TAU anyway (16 there), and the next pass's
        # block is sized from this one's spectrum
        h0 = 32 if (hint is None and basis is None and start is None and need > SUB_MAX_BLOCK) else hint
        sub = (_leading_subspace(g, need, RESOLVE_TAU, start if basis is None else None, h0)
               if SUBSPACE and n > SMALL_EIG and not direct else None)
        if sub is not None:
            w, v, k_sub = sub
        else:
            w, v = eigh_dev(g, nvec=need, tau=RESOLVE_TAU)
            k_sub = None
        wh = _dev.to_host(w)
        if top is None:
            top = max(float(wh[0]), 0.0)
        if top == 0.0 or wh[0] <= NOISE_REL * top:
            break                                   # remainder negligible: complete
        k = int(np.sum(wh[:need] > RESOLVE_TAU * wh[0])) if k_sub is None else k_sub
        if _DEBUG:
            print(f"[mode_basis n={n} r={r}] pass: need {need} resolved {k} "
                  f"lambda_top {wh[0]:.3e} ({wh[0] / top:.1e} of first)", file=sys.stderr)
        if basis is None and k >= need:
            return v[:, :need].contiguous()         # one pass resolved everything
        k = max(1, min(need, k))
        hint = _next_pass_hint(wh, k)
        new = v[:, :k].contiguous()
        if basis is not None:
            new = _orth_normalize(basis, new)
        basis = new if basis is None else t.cat([basis, new], dim=1).contiguous()
        if int(basis.shape[1]) >= r:
            break
        res = [_residual(xd, m, basis) for m in modes]
        g = None
        for m, xr in zip(modes, res):
            gm = unfold_gram_dev(xr, m)
            g = gm if g is None else _axpby(1.0, g, 1.0, gm)
        del res
        if reduce is not None:
            reduce(g)
        # trace >= lambda_max: a remainder already at rounding level goes
        # straight to the completion without an eigensolve
        tr = _dev.empty((1,))
        N.call("bt_trace_f64", _dev.ptr(g), n, _dev.ptr(tr), _dev.stream())
        if float(_dev.to_host(tr)[0]) <= NOISE_REL * top:
            break
    have = 0 if basis is None else int(basis.shape[1])
    if have < r:
        extra = _complete(basis, g, r - have)
        basis = extra if basis is None else t.cat([basis, extra], dim=1).contiguous()
    return basis[:, :r].contiguous()


def small_mode_basis_enqueue(xd, mode: int, r: int):
    """First pass of mode_basis_dev for a mode whose extent fits the one-CTA
    Jacobi (n <= SMALL_EIG), enqueued on the current stream without a host
    read: Gram + full eigensolve.  None when mode_basis_dev would start with
    the Gram-free refinement instead.  hosvd runs this for its short modes
    on a side stream beside the long mode's deflation passes (the bases of
    the original unfoldings are independent, decomp.py:247-256)."""
    n = int(xd.shape[mode - 1])
    if n > SMALL_EIG or (REFINE and r <= 32 and n >= 2 * r):
        return None
    g = unfold_gram_dev(xd, mode)
    w, v = eigh_dev(g, nvec=r, tau=RESOLVE_TAU)
    return g, w, v


def small_mode_basis_finish(handle, xd, mode: int, r: int):
    """The host side of that first pass: the basis when the pass resolved
    every wanted pair (the same test mode_basis_dev applies), else the full
    deflation loop from scratch."""
    _, w, v = handle
    wh = _dev.to_host(w)
    top = max(float(wh[0]), 0.0)
    if top > 0.0 and int(np.sum(wh[:r] > RESOLVE_TAU * wh[0])) >= r:
        return v[:, :r].contiguous()
    return mode_basis_dev(xd, mode, r)


def _scaled_gemm(a, b, scale, ta=False):
    """op(a) @ b @ diag(scale) on the engine (the diagonal rides on B's
    per-column scale)."""
    a = a.contiguous()
    b = b.contiguous()
    M = int(a.shape[1] if ta else a.shape[0])
    K = int(a.shape[0] if ta else a.shape[1])
    Nn = int(b.shape[1])
    out = _dev.empty((M, Nn))
    d = N.GemmDesc()
    d.M, d.N, d.Kin, d.Kout, d.batch = M, Nn, K, 1, 1
    d.A = _dev.ptr(a)
    d.sAm, d.sAki = (1, int(a.shape[1])) if ta else (int(a.shape[1]), 1)
    d.B, d.sBn, d.sBki = _dev.ptr(b), 1, Nn
    d.bscale, d.s_scale_ko = _dev.ptr(scale), 0
    d.C, d.sCm, d.sCn = _dev.ptr(out), Nn, 1
    d.alpha, d.beta = 1.0, 0.0
    ws = _dev.workspace(N.load().bt_gemm_f64_ws_bytes(C.byref(d)))
    N.call("bt_gemm_f64", C.byref(d), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    return out


def svd_truncated_dev(ad, r: int):
    """(u, s, v) of a matrix on device via the Gram of its short side
    (decomp.py:149-179): eigenpairs of the Gram (sign-normalised), s =
    sqrt(lambda), the long-side vectors by one engine GEMM scaled by 1/s,
    and the sign rule on u compensated in v."""
    m, n = int(ad.shape[0]), int(ad.shape[1])
    if m <= n:
        w, uu = eigh_dev(unfold_gram_dev(ad, 1))
        u = uu[:, :r].contiguous()
        s, sinv = _dev.empty((r,)), _dev.empty((r,))
        N.call("bt_svals_f64", _dev.ptr(w), r, _dev.ptr(s), _dev.ptr(sinv), _dev.stream())
        v = _scaled_gemm(ad, u, sinv, ta=True)          # a^T u / s   (n x r)
        return u, s, v
    w, vv = eigh_dev(unfold_gram_dev(ad, 2))
    v = vv[:, :r].contiguous()
    s, sinv = _dev.empty((r,)), _dev.empty((r,))
    N.call("bt_svals_f64", _dev.ptr(w), r, _dev.ptr(s), _dev.ptr(sinv), _dev.stream())
    u = _scaled_gemm(ad, v, sinv)                        # a v / s   (m x r)
    N.call("bt_sign_fix_pair_f64", _dev.ptr(u), m, r, _dev.ptr(v), n, _dev.stream())
    return u, s, v


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


def _householder_qr(ad):
    m, n = int(ad.shape[0]), int(ad.shape[1])
    q = _dev.empty((m, n))
    r = _dev.empty((n, n))
    ws = _dev.workspace(N.load().bt_qr_thin_ws_bytes(m, n))
    N.call("bt_qr_thin_f64", _dev.ptr(ad.contiguous()), m, n, _dev.ptr(q), _dev.ptr(r),
           _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    return q, r


QR_CHOL_MAX_COND = 1e6   # CholeskyQR2 is used when the R-diagonal ratio stays below this


def qr_thin_dev(ad):
    """Thin QR with nonnegative diag(R) on device (decomp.py:182-193).

    CholeskyQR2 on the engine: R1 = chol(A^T A)^T, Q1 = A R1^-1, then once
    more on Q1 (orthogonality to working precision for cond(A) up to ~1e7;
    the factorisation is unique for full column rank, so it equals LAPACK's
    Householder result with the sign normalisation).  Falls back to the
    single-CTA Householder kernel when A^T A is not numerically positive
    definite or the diagonal of R spans more than QR_CHOL_MAX_COND."""
    from .decomp import cholesky
    from .errors import NotPositiveDefiniteError

    m, n = int(ad.shape[0]), int(ad.shape[1])
    if n < 8:
        return _householder_qr(ad)
    t = _dev.torch()
    a = ad.contiguous()
    rs = []
    q = a
    for _ in range(2):
        g = gemm_dev(q, q, ta=True)
        g = _axpby(0.5, g, 0.5, g.t().contiguous())
        try:
            low = _dev.to_device(cholesky(g))
        except (NotPositiveDefiniteError, ShapeError):
            return _householder_qr(ad)
        d = _dev.to_host(t.diagonal(low).contiguous())
        if not (d.min() > 0.0) or d.max() / d.min() > QR_CHOL_MAX_COND:
            return _householder_qr(ad)
        linv = _dev.empty((n, n))
        ws = _dev.workspace(N.load().bt_tri_inv_lower_ws_bytes(n))
        N.call("bt_tri_inv_lower_f64", _dev.ptr(low), n, _dev.ptr(linv), _dev.ptr(ws),
               _dev.stream())
        q = gemm_dev(q, linv, tb=True)                   # Q R^-1 = Q L^-T
        rs.append(low.t().contiguous())                   # R = L^T (upper)
    r = gemm_dev(rs[1], rs[0])                            # R = R2 R1 (upper, positive diagonal)
    return q, r
