"""System identification in compressed coordinates (drop-in for
apps.py:46-237): the weighted block-Hankel tensor of the Markov
parameters is Tucker-compressed, the reduced Hankel ``R`` is assembled on the
device, and the realization runs on ``R`` -- all on the GPU.

* ``R``'s singular triplets: an SVD-grade left basis from the deflated Gram
  eigensolver (``_linalg.mode_basis_dev``), singular values as the exact
  column norms ``||R^T u_i||`` (absolute accuracy ~eps sigma_1, like LAPACK's
  SVD), ``v_i = R^T u_i / sigma_i``.
* The shift least squares ``lstsq(theta_fwd, theta_bwd)`` (apps.py:216-218)
  with ``theta = U Sigma^1/2``: ``theta_fwd^T theta_fwd = Sigma^1/2 (U_top^T
  U_top) Sigma^1/2`` where ``U_top^T U_top = I - U_last^T U_last`` is well
  conditioned, so ``A = Sigma^-1/2 (U_top^T U_top)^-1 U_top^T U_bot Sigma^1/2``
  is solved with a Cholesky of that Gram -- the same least-squares solution,
  without squaring Sigma's condition number.
* Output/input maps lifted by engine GEMMs (apps.py:220-224).

Singular vectors carry LAPACK's sign freedom in the reference, so the
realized (A, B, C) match up to a diagonal +-1 similarity; eigenvalues and
the realized Markov parameters are invariant.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _dev
from . import _linalg as L
from . import _native as N
from .blocks import BlockPattern, build_pattern, struct_assemble, struct_expand
from .decomp import cholesky, hosvd, tucker_partial
from .errors import ConvergenceError, ShapeError
from .tensor import ttm_dev

__all__ = ["MarkovSequence", "LtiSystem", "EraResult", "markov_from_lti",
           "hankel_pattern_from_markov", "era_identify_compressed"]


def _arr(x):
    return x if _dev.is_device(x) else np.asarray(x, dtype=np.float64)


@dataclass(frozen=True)
class MarkovSequence:
    """apps.py:46-74: impulse-response parameters h_1 .. h_{2s-1}, (2s-1, d_out, d_in)."""

    params: object

    def __post_init__(self) -> None:
        object.__setattr__(self, "params", _arr(self.params))
        if self.params.ndim != 3:
            raise ShapeError("params must be a (2s-1, d_out, d_in) stack")
        count = int(self.params.shape[0])
        if count < 1 or count % 2 == 0:
            raise ShapeError(f"need an odd number 2s-1 of parameters, got {count}")

    @property
    def s(self) -> int:
        return (int(self.params.shape[0]) + 1) // 2

    @property
    def d_out(self) -> int:
        return int(self.params.shape[1])

    @property
    def d_in(self) -> int:
        return int(self.params.shape[2])


@dataclass(frozen=True)
class LtiSystem:
    """apps.py:77-102: discrete-time state-space triple (A, B, C)."""

    a: object
    b: object
    c: object

    def __post_init__(self) -> None:
        a, b, c = (_arr(m) for m in (self.a, self.b, self.c))
        object.__setattr__(self, "a", a)
        object.__setattr__(self, "b", b)
        object.__setattr__(self, "c", c)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ShapeError("state matrix must be square")
        if b.ndim != 2 or b.shape[0] != a.shape[0]:
            raise ShapeError("input matrix rows must match the state dimension")
        if c.ndim != 2 or c.shape[1] != a.shape[0]:
            raise ShapeError("output matrix columns must match the state dimension")

    @property
    def order(self) -> int:
        return int(self.a.shape[0])

    def eigenvalues(self):
        """Host utility on the (order x order) state matrix (not a path kernel)."""
        return np.linalg.eigvals(_dev.to_host(self.a) if _dev.is_device(self.a) else self.a)


def markov_from_lti(system: LtiSystem, count: int) -> MarkovSequence:
    """apps.py:105-114: h_k = C A^(k-1) B by two engine GEMMs per step."""
    if count < 1 or count % 2 == 0:
        raise ShapeError("count must be odd and positive (it fills an s x s Hankel)")
    a, b, c = (_dev.to_device(m) for m in (system.a, system.b, system.c))
    params = _dev.empty((count, int(c.shape[0]), int(b.shape[1])))
    x = b.contiguous()
    for k in range(count):
        params[k] = L.gemm_dev(c, x)
        if k + 1 < count:
            x = L.gemm_dev(a, x)
    return MarkovSequence(params=_dev.like_input(system.a, params))


def hankel_pattern_from_markov(seq: MarkovSequence):
    """apps.py:117-125."""
    return build_pattern("hankel", seq.s, seq.s, seq.d_out, seq.d_in), seq.params


@dataclass(frozen=True)
class EraResult:
    """apps.py:128-150."""

    system: LtiSystem
    pattern: BlockPattern
    reduced_pattern: BlockPattern
    reduced_hankel: object
    basis_left: object
    basis_right: object
    sing_vals: object
    tera: bool

    def hankel_approx(self):
        """(I (x) U) R (I (x) W^T) as two device mode products of the
        (s, r1, s, r3) view of R."""
        s = self.pattern.ell
        u = _dev.to_device(self.basis_left)
        w = _dev.to_device(self.basis_right)
        r = _dev.to_device(self.reduced_hankel)
        r1, r3 = int(u.shape[1]), int(w.shape[1])
        x = r.reshape(s, r1, s, r3)
        y = ttm_dev(ttm_dev(x.contiguous(), 2, u, int(u.shape[0])), 4, w, int(w.shape[0]))
        out = y.reshape(s * int(u.shape[0]), s * int(w.shape[0]))
        return _dev.like_input(self.reduced_hankel, out)


def _svd_leading(rd, order: int):
    """(sing_vals (all min(M, N)), U[:, :order], V[:, :order]) of R on device."""
    rows, cols = (int(v) for v in rd.shape)
    kmax = min(rows, cols)
    u_all = L.mode_basis_dev(rd.contiguous(), 1, kmax)              # (M, kmax), SVD grade
    rtu = L.gemm_dev(rd, u_all, ta=True)                             # R^T U  (N, kmax)
    sv = _dev.empty((kmax,))
    N.call("bt_col_norms_f64", _dev.ptr(rtu), cols, kmax, _dev.ptr(sv), _dev.stream())
    return sv, u_all, rtu


def era_identify_compressed(seq: MarkovSequence, ranks, order: int, tera: bool = False) -> EraResult:
    """apps.py:153-237 on the GPU."""
    if seq.s < 2:
        raise ShapeError("need s >= 2 Hankel block rows to shift")
    pattern, blocks = hankel_pattern_from_markov(seq)
    r1, r2, r3 = ranks
    bd = _dev.to_device(blocks)
    from .psd import _max_abs

    if _max_abs(bd) == 0.0:
        raise ConvergenceError("all Markov parameters are zero; Hankel is degenerate")
    reduced_pattern = pattern.with_blocks(r1, r3)
    p, dout, din = (int(v) for v in bd.shape)
    if tera:
        t = bd.permute(1, 0, 2).contiguous()                         # (d_out, p, d_in), unweighted
        tk = tucker_partial(t, [r1, None, r3])
        u, w = _dev.to_device(tk.factors[0]), _dev.to_device(tk.factors[2])
        mids = ttm_dev(ttm_dev(bd, 2, u, int(r1), transpose=True), 3, w, int(r3), transpose=True)
        reduced = _dev.to_device(struct_assemble(reduced_pattern, mids))
    else:
        d, _, _ = pattern.device()
        t = _dev.empty((dout, p, din))
        N.call("bt_build_hankel_f64", _dev.ptr(bd), p, dout, din, _dev.ptr(d["eta"]), _dev.ptr(t),
               _dev.stream())
        tk = hosvd(t, [r1, r2, r3])
        u, v, w = (_dev.to_device(f) for f in tk.factors)
        core = _dev.to_device(tk.core)
        items = ttm_dev(core, 2, v, int(v.shape[0]))                  # (r1, p, r3)
        items = items.permute(1, 0, 2).contiguous()                   # (p, r1, r3)
        reduced = _dev.to_device(struct_expand(reduced_pattern, items))
    M, Nn = (int(x) for x in reduced.shape)
    sv, u_all, rtu = _svd_leading(reduced, order)
    if not 1 <= order <= min(M, Nn):
        raise ShapeError(f"model order {order} out of range for a {(M, Nn)} Hankel")
    svh = _dev.to_host(sv)
    cutoff = max(M, Nn) * np.finfo(np.float64).eps * svh[0]
    if svh[order - 1] <= cutoff:
        raise ConvergenceError(f"model order {order} exceeds the numerical rank of the reduced Hankel")
    # sqrt(sigma) and 1/sqrt(sigma): the bt_svals kernel applied to sigma itself
    root, iroot = _dev.empty((order,)), _dev.empty((order,))
    N.call("bt_svals_f64", _dev.ptr(sv), order, _dev.ptr(root), _dev.ptr(iroot), _dev.stream())
    uo = u_all[:, :order].contiguous()
    theta = _dev.empty((M, order))
    N.call("bt_diag_scale_f64", _dev.ptr(uo), M, order, None, _dev.ptr(root), _dev.ptr(theta),
           _dev.stream())
    # gamma^T = sqrt(sigma) V^T with V = R^T U / sigma  ->  gamma = R^T U / sqrt(sigma)
    rto = rtu[:, :order].contiguous()
    gamma = _dev.empty((Nn, order))
    N.call("bt_diag_scale_f64", _dev.ptr(rto), Nn, order, None, _dev.ptr(iroot), _dev.ptr(gamma),
           _dev.stream())
    # shift least squares in the scaled basis (module docstring)
    rows = r1 * (seq.s - 1)
    u_top = uo[:rows].contiguous()
    u_bot = uo[r1:].contiguous()
    gtop = L.gemm_dev(u_top, u_top, ta=True)
    gtop = L._axpby(0.5, gtop, 0.5, gtop.t().contiguous())
    hmix = L.gemm_dev(u_top, u_bot, ta=True)
    low = _dev.to_device(cholesky(gtop))
    linv = _dev.empty((order, order))
    ws = _dev.workspace(N.load().bt_tri_inv_lower_ws_bytes(order))
    N.call("bt_tri_inv_lower_f64", _dev.ptr(low), order, _dev.ptr(linv), _dev.ptr(ws),
           _dev.stream())
    x = L.gemm_dev(linv, L.gemm_dev(linv, hmix), ta=True)            # G^-1 H
    a_til = _dev.empty((order, order))
    N.call("bt_diag_scale_f64", _dev.ptr(x), order, order, _dev.ptr(iroot), _dev.ptr(root),
           _dev.ptr(a_til), _dev.stream())
    c_lift = L.gemm_dev(u, theta[:r1].contiguous())                  # (d_out, order)
    b_lift = L.gemm_dev(gamma[:r3].contiguous(), w, ta=True, tb=True)  # (order, d_in)
    like = seq.params
    system = LtiSystem(a=_dev.like_input(like, a_til), b=_dev.like_input(like, b_lift),
                       c=_dev.like_input(like, c_lift))
    return EraResult(system=system, pattern=pattern, reduced_pattern=reduced_pattern,
                     reduced_hankel=_dev.like_input(like, reduced),
                     basis_left=_dev.like_input(like, u), basis_right=_dev.like_input(like, w),
                     sing_vals=_dev.like_input(like, sv), tera=tera)
