"""ctypes binding of libbt200.so (the C-ABI in include/bt200.h).

The product path has no CPU fallback: if the shared library or a CUDA
device is missing, every compute entry point raises.  Device memory and
streams come from PyTorch (plumbing only); all arithmetic runs in the
library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import (ConvergenceError, NotPositiveDefiniteError, PatternMismatchError,
                     ShapeError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbt200.so")

BT_OK, BT_E_SHAPE, BT_E_PATTERN, BT_E_NOT_PD, BT_E_CONV, BT_E_CUDA, BT_E_VALUE = range(7)

_i64 = C.c_int64
_dp = C.c_void_p  # device pointers are passed as integers


class GemmDesc(C.Structure):
    _fields_ = [("M", _i64), ("N", _i64), ("Kin", _i64), ("Kout", _i64), ("batch", _i64),
                ("A", _dp), ("sAm", _i64), ("sAko", _i64), ("sAki", _i64), ("sAb", _i64),
                ("B", _dp), ("sBn", _i64), ("sBko", _i64), ("sBki", _i64), ("sBb", _i64),
                ("bscale", _dp), ("s_scale_ko", _i64), ("s_scale_b", _i64),
                ("ascale", _dp), ("s_ascale_ko", _i64), ("s_ascale_b", _i64),
                ("C", _dp), ("sCm", _i64), ("sCn", _i64), ("sCb", _i64),
                ("alpha", C.c_double), ("beta", C.c_double), ("symmetric", C.c_int),
                ("splits", C.c_int)]


class PatternDev(C.Structure):
    _fields_ = [("ell", _i64), ("q", _i64), ("m", _i64), ("n", _i64), ("p", _i64), ("nnz", _i64),
                ("cell_class", _dp), ("cell_order", _dp), ("rep_cell", _dp), ("eta", _dp),
                ("class_ptr", _dp), ("class_cells", _dp)]


class CpProblem(C.Structure):
    _fields_ = [("x", _dp), ("I", _i64), ("J", _i64), ("K", _i64), ("R", _i64),
                ("norm_x", C.c_double)]


_P = C.POINTER
_SIGS = {
    "bt_version": (C.c_int, []),
    "bt_last_error": (C.c_char_p, []),
    "bt_launch_count": (_i64, []),
    "bt_gemm_f64_ws_bytes": (_i64, [_P(GemmDesc)]),
    "bt_gemm_f64": (C.c_int, [_P(GemmDesc), _dp, _i64, _dp]),
    "bt_gather_ws_bytes": (_i64, [_P(PatternDev)]),
    "bt_gather_blocks_f64": (C.c_int, [_dp, _i64, _P(PatternDev), C.c_double, C.c_int, _dp, _dp,
                                       _P(_i64), _dp]),
    "bt_scatter_blocks_f64": (C.c_int, [_dp, _i64, _i64, _i64, _P(PatternDev), _dp, _i64, _dp]),
    "bt_build_hankel_f64": (C.c_int, [_dp, _i64, _i64, _i64, _dp, _dp, _dp]),
    "bt_build_gneiting_f64": (C.c_int, [_dp, _i64, _i64, C.c_double, _dp, _dp, _dp]),
    "bt_build_psf_f64": (C.c_int, [_dp, _i64, _i64, _dp, _dp]),
    "bt_build_cp_model_f64": (C.c_int, [_dp, _dp, _dp, _i64, _i64, _i64, _i64, _i64, _i64,
                                        C.c_double, C.c_uint64, _dp, _dp, _i64, _dp]),
    "bt_cp_als_ws_bytes": (_i64, [_P(CpProblem)]),
    "bt_cp_tree_variant": (C.c_int, [_P(CpProblem)]),
    "bt_cp_als_f64": (C.c_int, [_P(CpProblem), _dp, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int,
                                _P(C.c_double), _P(C.c_int), _P(C.c_int), _P(C.c_double), _dp,
                                _i64, _dp]),
    "bt_cp_state_ws_bytes": (_i64, [_P(CpProblem)]),
    "bt_cp_state_create": (C.c_int, [_P(CpProblem), _dp, _dp, _dp, _dp, C.c_int, C.c_int, _dp, _i64,
                                     _dp, _P(C.c_void_p)]),
    "bt_cp_state_destroy": (C.c_int, [C.c_void_p]),
    "bt_cp_init_local": (C.c_int, [C.c_void_p, C.c_double, _dp]),
    "bt_cp_init_finish": (C.c_int, [C.c_void_p, _dp]),
    "bt_cp_mttkrp": (C.c_int, [C.c_void_p, C.c_int, _dp]),
    "bt_cp_solve": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp]),
    "bt_cp_solve_finish": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp]),
    "bt_cp_residual": (C.c_int, [C.c_void_p, _dp]),
    "bt_cp_residual_finish": (C.c_int, [C.c_void_p, C.c_int, _dp]),
    "bt_cp_read_fit": (C.c_int, [C.c_void_p, C.c_int, _P(C.c_double)]),
    "bt_cp_state_finish": (C.c_int, [C.c_void_p, C.c_int, _P(C.c_double)]),
    "bt_mttkrp_ws_bytes": (_i64, [_P(CpProblem), C.c_int]),
    "bt_mttkrp_f64": (C.c_int, [_P(CpProblem), C.c_int, _dp, _dp, _dp, _dp, _dp, _i64, _dp]),
    "bt_pinv_sym_f64": (C.c_int, [_dp, _i64, _dp, _dp]),
    "bt_unfold_gram_ws_bytes": (_i64, [_P(_i64), C.c_int, C.c_int]),
    "bt_unfold_gram_f64": (C.c_int, [_dp, _P(_i64), C.c_int, C.c_int, _dp, _dp, _i64, _dp]),
    "bt_syevd_ws_bytes": (_i64, [_i64]),
    "bt_syevd_f64": (C.c_int, [_dp, _i64, _dp, _dp, _dp, _i64, _dp]),
    "bt_syevx_ws_bytes": (_i64, [_i64, _i64]),
    "bt_syevx_f64": (C.c_int, [_dp, _i64, _i64, C.c_double, _dp, _dp, _dp, _i64, _dp]),
    "bt_qr_thin_ws_bytes": (_i64, [_i64, _i64]),
    "bt_qr_thin_f64": (C.c_int, [_dp, _i64, _i64, _dp, _dp, _dp, _i64, _dp]),
    "bt_block_digest_f64": (C.c_int, [_dp, _i64, _i64, _i64, _i64, _i64, C.c_double, _dp, _dp,
                                      _dp, _dp]),
    "bt_block_group_ws_bytes": (_i64, [_i64]),
    "bt_block_group": (C.c_int, [_dp, _dp, _dp, _i64, _dp, _dp, _dp, _i64, _dp]),
    "bt_block_match_f64": (C.c_int, [_dp, _i64, _i64, _i64, _i64, _i64, _dp, C.c_double, C.c_int,
                                     _dp, _dp]),
    "bt_fill_normal_f64": (C.c_int, [_dp, _i64, C.c_uint64, _dp]),
    "bt_diag_scale_f64": (C.c_int, [_dp, _i64, _i64, _dp, _dp, _dp, _dp]),
    "bt_col_norms_f64": (C.c_int, [_dp, _i64, _i64, _dp, _dp]),
    "bt_transpose_f64": (C.c_int, [_dp, _i64, _i64, _dp, _dp]),
    "bt_svd_small_f64": (C.c_int, [_dp, _i64, _dp, _dp, _dp, _dp]),
    "bt_tsqr_ws_bytes": (_i64, [_i64, _i64]),
    "bt_chol_small_f64": (C.c_int, [_dp, _i64, _dp, _dp, _dp, _dp]),
    "bt_complete_basis_ws_bytes": (_i64, [_i64, _i64, _i64]),
    "bt_complete_basis_f64": (C.c_int, [_dp, _i64, _i64, _i64, C.c_uint64, _dp, _P(C.c_int), _dp,
                                        _i64, _dp]),
    "bt_tsqr_f64": (C.c_int, [_dp, _i64, _i64, _dp, _dp, _dp, _i64, _dp]),
    "bt_reverse_axes_f64": (C.c_int, [_dp, _P(_i64), C.c_int, _dp, _dp]),
    "bt_sign_fix_pair_f64": (C.c_int, [_dp, _i64, _i64, _dp, _i64, _dp]),
    "bt_svals_f64": (C.c_int, [_dp, _i64, _dp, _dp, _dp]),
    "bt_ritz_resid_f64": (C.c_int, [_dp, _dp, _dp, _i64, _i64, _i64, _dp, _dp]),
    "bt_cholesky_ws_bytes": (_i64, [_i64]),
    "bt_cholesky_f64": (C.c_int, [_dp, _i64, _dp, _dp, _P(_i64), _dp]),
    "bt_tri_inv_lower_ws_bytes": (_i64, [_i64]),
    "bt_tri_inv_lower_f64": (C.c_int, [_dp, _i64, _dp, _dp, _dp]),
    "bt_ttm_ws_bytes": (_i64, [_P(_i64), C.c_int, C.c_int, _i64]),
    "bt_ttm_f64": (C.c_int, [_dp, _P(_i64), C.c_int, C.c_int, _dp, _i64, C.c_int, _dp, _dp, _i64,
                             _dp]),
    "bt_matvec_kron_ws_bytes": (_i64, [_P(PatternDev), _i64, _i64]),
    "bt_matvec_kron_f64": (C.c_int, [_P(PatternDev), _dp, _dp, _dp, _dp, _i64, _dp, _i64, _dp,
                                     _dp, _i64, _dp]),
    "bt_matvec_blr_ws_bytes": (_i64, [_P(PatternDev), _i64, _i64, _i64]),
    "bt_matvec_blr_f64": (C.c_int, [_P(PatternDev), _dp, _dp, _dp, _i64, _dp, _i64, _dp, _dp,
                                    _i64, _dp, _dp, _i64, _dp]),
    "bt_ml_matvec_ws_bytes": (_i64, [_i64, _P(_i64), _P(_i64), _i64]),
    "bt_ml_matvec_f64": (C.c_int, [_i64, _P(_i64), _P(_i64), _dp, _dp, _dp, _dp, _i64, _dp, _dp,
                                   _i64, _dp]),
    "bt_maxabs_f64": (C.c_int, [_dp, _i64, _dp, _dp, _i64, _dp]),
    "bt_transpose_check_f64": (C.c_int, [_dp, _i64, _i64, _dp, C.c_double, _dp, _P(_i64), _dp]),
    "bt_inv_sqrt_f64": (C.c_int, [_dp, _i64, _dp, _dp]),
    "bt_sym_scale_f64": (C.c_int, [_dp, _i64, _dp, _dp, _dp]),
    "bt_trace_f64": (C.c_int, [_dp, _i64, _dp, _dp]),
    "bt_copy_cells_f64": (C.c_int, [_dp, _i64, _dp, _i64, _i64, _i64, _i64, _dp, _dp]),
    "bt_cp_small_clocks": (C.c_int, [_dp]),
    "bt_leading_subspace_ws_bytes": (_i64, [_i64, _i64, _i64]),
    "bt_leading_subspace_f64": (C.c_int, [_dp, _i64, _i64, C.c_double, _dp, _i64, _i64, _dp, _dp,
                                          _P(_i64), _P(_i64), _P(C.c_int), _dp, _i64, _dp]),
    "bt_sign_fix_f64": (C.c_int, [_dp, _i64, _i64, _dp]),
    "bt_col_normalize_f64": (C.c_int, [_dp, _i64, _i64, _dp]),
    "bt_axpby_f64": (C.c_int, [_i64, C.c_double, _dp, C.c_double, _dp, _dp, _dp]),
    "bt_sumsq_ws_bytes": (_i64, [_i64]),
    "bt_sumsq_f64": (C.c_int, [_dp, _i64, _dp, _dp, _i64, _dp]),
    "bt_peak_dmma": (C.c_int, [_i64, C.c_int, C.c_int, _dp, _P(C.c_double), _dp]),
    "bt_peak_dmma_chains": (C.c_int, [_i64, C.c_int, C.c_int, C.c_int, _dp, _P(C.c_double), _dp]),
    "bt_peak_dfma": (C.c_int, [_i64, C.c_int, C.c_int, _dp, _P(C.c_double), _dp]),
}

_lib = None


def exported_symbols():
    return list(_SIGS)


def load(path: str = LIB_PATH):
    """Load (once) and type the shared library.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"bt200 native library not found at {path}; run "
            "`python -m paper_2105_01170_b200.build` (there is no CPU fallback)")
    lib = C.CDLL(path)
    missing = []
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    _MISSING[:] = missing
    return lib


_MISSING: list = []


def missing_symbols():
    load()
    return list(_MISSING)


_EXC = {BT_E_SHAPE: ShapeError, BT_E_PATTERN: PatternMismatchError,
        BT_E_NOT_PD: NotPositiveDefiniteError, BT_E_CONV: ConvergenceError,
        BT_E_CUDA: RuntimeError, BT_E_VALUE: ValueError}


def check(status: int, what: str = "") -> None:
    if status == BT_OK:
        return
    msg = (_lib.bt_last_error() or b"").decode(errors="replace")
    raise _EXC.get(status, RuntimeError)(f"{what}: {msg}" if what else msg)


def call(name: str, *args):
    lib = load()
    if name in _MISSING:
        raise RuntimeError(f"libbt200.so does not export {name}; rebuild")
    check(getattr(lib, name)(*args), name)
