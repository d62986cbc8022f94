"""Tensor primitives (drop-in for tensor.py).

``unfold``/``fold``/``twist``/``squeeze`` are pure layout views with the
reference's first-index-fastest convention (tensor.py:1-16) and stay on the
host for numpy inputs (torch permute/reshape for device inputs).  The
arithmetic ones -- ``mode_multiply`` (tensor.py:75-90) and ``fro_norm``
(tensor.py:107-109) -- run on the GPU: the mode product is a DMMA GEMM over
the C-order tensor in place (no unfolding copy).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _dev
from . import _native as N
from .errors import ShapeError

__all__ = ["unfold", "fold", "mode_multiply", "twist", "squeeze", "fro_norm"]


def _check_mode(mode: int, order: int) -> int:
    if not 1 <= mode <= order:
        raise ShapeError(f"mode {mode} out of range for order-{order} tensor")
    return mode - 1


def unfold(t, mode: int):
    ax = _check_mode(mode, t.ndim)
    if _dev.is_device(t):
        # column index first-index-fastest == reverse C-order of the rest
        rest = [d for d in range(t.ndim) if d != ax][::-1]
        return t.permute(ax, *rest).reshape(t.shape[ax], -1)
    return np.reshape(np.moveaxis(t, ax, 0), (t.shape[ax], -1), order="F")


def fold(mat, mode: int, dims):
    ax = _check_mode(mode, len(dims))
    dims = tuple(int(d) for d in dims)
    rest = dims[:ax] + dims[ax + 1:]
    expected = (dims[ax], int(np.prod(rest, dtype=np.int64)) if rest else 1)
    if tuple(mat.shape) != expected:
        raise ShapeError(f"unfolding of shape {tuple(mat.shape)} cannot fold into {dims} "
                         f"along mode {mode}")
    if _dev.is_device(mat):
        arr = mat.reshape((dims[ax],) + rest[::-1])
        # arr axes: (ax, rest reversed) -> back to natural order
        order = [ax] + [d for d in range(len(dims)) if d != ax][::-1]
        inv = [order.index(d) for d in range(len(dims))]
        return arr.permute(*inv).contiguous()
    arr = np.reshape(mat, (dims[ax], *rest), order="F")
    return np.moveaxis(arr, 0, ax)


def twist(mat):
    if mat.ndim != 2:
        raise ShapeError("twist expects a matrix")
    if _dev.is_device(mat):
        return mat[:, None, :].contiguous()
    return np.ascontiguousarray(mat[:, None, :])


def squeeze(t):
    if t.ndim != 3 or t.shape[1] != 1:
        raise ShapeError(f"squeeze expects an m x 1 x n tensor, got shape {tuple(t.shape)}")
    if _dev.is_device(t):
        return t[:, 0, :].contiguous()
    return np.ascontiguousarray(t[:, 0, :])


def fro_norm_dev(td) -> float:
    """||t||_F of a device tensor (deterministic two-level tree)."""
    n = int(td.numel())
    out = _dev.zeros((1,))
    if n:
        ws = _dev.workspace(N.load().bt_sumsq_ws_bytes(n))
        N.call("bt_sumsq_f64", _dev.ptr(td), n, _dev.ptr(out), _dev.ptr(ws),
               int(ws.numel()) * 8, _dev.stream())
    return float(np.sqrt(_dev.to_host(out)[0]))


def fro_norm(t) -> float:
    return fro_norm_dev(_dev.to_device(t))


def ttm_dev(xd, mode: int, ud, rows: int, transpose: bool = False):
    """y = x x_mode u on device; ud is (rows, extent) or, with transpose,
    (extent, rows) (i.e. u^T given) -- both contiguous."""
    dims = tuple(int(s) for s in xd.shape)
    order = len(dims)
    ax = _check_mode(mode, order)
    out_dims = list(dims)
    out_dims[ax] = int(rows)
    y = _dev.empty(out_dims)
    cd = (C.c_int64 * order)(*dims)
    wsb = N.load().bt_ttm_ws_bytes(cd, order, mode, int(rows))
    ws = _dev.workspace(wsb)
    N.call("bt_ttm_f64", _dev.ptr(xd), cd, order, mode, _dev.ptr(ud), int(rows),
           int(bool(transpose)), _dev.ptr(y), _dev.ptr(ws), int(ws.numel()) * 8, _dev.stream())
    return y


def mode_multiply(t, mode: int, u):
    """tensor.py:75-90: ``t x_mode u`` (``u @ unfold(t, mode)`` refolded)."""
    ax = _check_mode(mode, t.ndim)
    if u.ndim != 2 or u.shape[1] != t.shape[ax]:
        raise ShapeError(f"factor of shape {tuple(u.shape)} does not act on mode {mode} "
                         f"of extent {t.shape[ax]}")
    y = ttm_dev(_dev.to_device(t), mode, _dev.to_device(u), int(u.shape[0]))
    return _dev.like_input(t, y)
