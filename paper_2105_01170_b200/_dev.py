"""Device plumbing: PyTorch provides HBM allocations and the CUDA stream;
nothing here computes.  Arrays cross the API as numpy (reference
semantics: results come back as numpy) or as CUDA torch tensors (kept on
device)."""

from __future__ import annotations

import numpy as np

from . import _native

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


_cuda_ok = False


def require_cuda():
    """torch, after checking once that a CUDA device and the library are there
    (torch.cuda.is_available() costs ~4 us a call -- it was called ~170 times
    per HOOI sweep)."""
    global _cuda_ok
    t = torch()
    if _cuda_ok:
        return t
    if not t.cuda.is_available():
        raise RuntimeError("bt200 needs a CUDA device (sm_100a); there is no CPU fallback")
    _native.load()
    _cuda_ok = True
    return t


def is_device(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def to_device(x, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (fp64 unless dtype given)."""
    t = require_cuda()
    dt = t.float64 if dtype is None else dtype
    if isinstance(x, t.Tensor):
        y = x.to(device="cuda", dtype=dt)
        return y.contiguous()
    arr = np.ascontiguousarray(np.asarray(x))
    return t.from_numpy(arr).to(device="cuda", dtype=dt, non_blocking=False).contiguous()


def empty(shape, dtype=None):
    t = require_cuda()
    return t.empty(tuple(int(s) for s in shape), dtype=t.float64 if dtype is None else dtype,
                   device="cuda")


def zeros(shape, dtype=None):
    t = require_cuda()
    return t.zeros(tuple(int(s) for s in shape), dtype=t.float64 if dtype is None else dtype,
                   device="cuda")


def workspace(nbytes: int):
    """A device scratch buffer of at least nbytes (16-byte aligned)."""
    t = require_cuda()
    n = max(int(nbytes), 16)
    return t.empty((n + 15) // 16 * 2, dtype=t.float64, device="cuda")


def ptr(x) -> int:
    return 0 if x is None else int(x.data_ptr())


_raw_stream = None


def stream() -> int:
    """The current CUDA stream's handle.  torch.cuda.current_stream() builds a
    Stream object (~15 us); the raw-handle query behind it is ~1 us -- every
    library call takes the stream, ~60 calls per HOOI sweep."""
    global _raw_stream
    t = torch()
    if _raw_stream is None:
        fn = getattr(t._C, "_cuda_getCurrentRawStream", None)
        _raw_stream = fn if fn is not None else False
    if _raw_stream:
        return int(_raw_stream(t.cuda.current_device()))
    return int(t.cuda.current_stream().cuda_stream)


def to_host(x) -> np.ndarray:
    return x.detach().cpu().numpy()


def like_input(ref, dev_tensor):
    """Return dev_tensor as a CUDA tensor if ref was on device, else numpy."""
    return dev_tensor if is_device(ref) else to_host(dev_tensor)


def transpose(x):
    """x (rows, cols) device tensor -> contiguous (cols, rows) copy, by the
    library's tiled transpose kernel (layout plumbing of the matvec RHS)."""
    if x.ndim != 2:
        raise ValueError(f"transpose expects a matrix, got shape {tuple(x.shape)}")
    # the kernel moves 8-byte elements: anything but fp64 goes through
    # to_device's conversion first (an int / fp32 tensor would otherwise be
    # reinterpreted as doubles)
    x = to_device(x).contiguous()
    rows, cols = int(x.shape[0]), int(x.shape[1])
    out = empty((cols, rows))
    _native.call("bt_transpose_f64", ptr(x), rows, cols, ptr(out), stream())
    return out
