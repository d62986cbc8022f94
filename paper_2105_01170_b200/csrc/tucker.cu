// K7 / K9: unfolding Gram (SYRK) and mode products (TTM) over a C-order
// tensor in place -- the reference forms `unfold(t, k)` copies
// (tensor.py:52) and calls LAPACK SVD on them (decomp.py:172/227) or
// `u @ unfold` (tensor.py:90).  Both reduce to the DMMA engine with the
// tensor viewed as (outer, n_mode, inner).
#include "gemm.cuh"

#include <algorithm>
#include <cstdlib>

int bt_gemm_run(BtGemmArgs g, int64_t batch, cudaStream_t st, int want_splits, int64_t ws_elems);
int64_t bt_gemm_ws_elems(BtGemmArgs g, int64_t batch);
int64_t bt_syrk_tma_ws_elems(int64_t n, int64_t kt_total);
int bt_syrk_tma(const double* x, int64_t outer, int64_t n, int64_t inner, double* g, double* ws,
                int64_t ws_elems, cudaStream_t st);
// BT_SYRK_TMA=0: unfolding Grams on the cp.async engine (A/B runs)
static bool use_syrk_tma() {
  static const bool v = !(getenv("BT_SYRK_TMA") && getenv("BT_SYRK_TMA")[0] == '0');
  return v;
}
int bt_gemm_at_tma_ex(const double* a, int64_t lda, int64_t sAb, const double* b, int64_t ldb,
                      double* c, int64_t ldc, int64_t sCb, int64_t M, int64_t N, int64_t Kdim,
                      int64_t batch, int transpose_out, cudaStream_t st);

namespace {

struct View3 {
  int64_t outer, n, inner;
};

bool view3(const int64_t* dims, int order, int mode, View3& v) {
  if (order < 1 || mode < 1 || mode > order) return false;
  v.outer = 1;
  v.inner = 1;
  for (int d = 0; d < mode - 1; ++d) v.outer *= dims[d];
  v.n = dims[mode - 1];
  for (int d = mode; d < order; ++d) v.inner *= dims[d];
  return true;
}

// G[i][i'] = sum_{o,c} X(o,i,c) X(o,i',c)
BtGemmArgs gram_args(const double* x, const View3& v, double* g) {
  BtGemmArgs a{};
  a.M = v.n;
  a.N = v.n;
  if (v.inner > 1) {
    // K-contiguous rows of length inner, outer blocks as ko
    a.Kin = v.inner;
    a.Kout = v.outer;
    a.A = BtOperand{x, v.inner, v.n * v.inner, 1, 0};
    a.B = BtOperand{x, v.inner, v.n * v.inner, 1, 0};
  } else {
    // last mode: m contiguous, reduction over outer with stride n
    a.Kin = v.outer;
    a.Kout = 1;
    a.A = BtOperand{x, 1, 0, v.n, 0};
    a.B = BtOperand{x, 1, 0, v.n, 0};
  }
  a.C = g;
  a.sCm = v.n;
  a.sCn = 1;
  a.alpha = 1.0;
  a.beta = 0.0;
  a.symmetric = 1;
  return a;
}

// Y(o, r, c) = sum_i U[r][i] X(o, i, c)    (u given as (rows, n) or u^T as (n, rows))
BtGemmArgs ttm_args(const double* x, const View3& v, const double* u, int64_t rows, int transpose,
                    double* y, int64_t& batch) {
  BtGemmArgs a{};
  a.alpha = 1.0;
  a.beta = 0.0;
  if (v.inner == 1) {
    // Y[o][r] = sum_i X[o][i] U[r][i]
    batch = 1;
    a.M = v.outer;
    a.N = rows;
    a.Kin = v.n;
    a.Kout = 1;
    a.A = BtOperand{x, v.n, 0, 1, 0};
    a.B = transpose ? BtOperand{u, 1, 0, rows, 0} : BtOperand{u, v.n, 0, 1, 0};
    a.C = y;
    a.sCm = rows;
    a.sCn = 1;
  } else {
    batch = v.outer;
    a.M = rows;
    a.N = v.inner;
    a.Kin = v.n;
    a.Kout = 1;
    a.A = transpose ? BtOperand{u, 1, 0, rows, 0} : BtOperand{u, v.n, 0, 1, 0};
    a.B = BtOperand{x, 1, 0, v.inner, v.n * v.inner};
    a.C = y;
    a.sCm = v.inner;
    a.sCn = 1;
    a.sCb = rows * v.inner;
  }
  return a;
}

}  // namespace

extern "C" int64_t bt_unfold_gram_ws_bytes(const int64_t* dims, int order, int mode) {
  View3 v;
  if (!view3(dims, order, mode, v)) return 0;
  int64_t e = bt_gemm_ws_elems(gram_args(nullptr, v, nullptr), 1);
  if (v.inner > 1)
    e = std::max(e, bt_syrk_tma_ws_elems(v.n, v.outer * ((v.inner + 15) / 16)));
  return e * 8;
}

extern "C" int bt_unfold_gram_f64(const double* x, const int64_t* dims, int order, int mode,
                                  double* g, void* ws, int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_unfold_gram_f64");
  View3 v;
  BT_REQUIRE(view3(dims, order, mode, v), BT_E_SHAPE, "mode %d out of range for order-%d tensor",
             mode, order);
  if (use_syrk_tma() && v.inner > 1 && v.n >= 64) {
    // K-contiguous rows: the TMA-fed SYRK (lower 128-tiles, split reduction)
    const int rc = bt_syrk_tma(x, v.outer, v.n, v.inner, g, static_cast<double*>(ws), ws_bytes / 8,
                               bt_stream(stream));
    if (rc != BT_E_VALUE) return rc;
  }
  BtGemmArgs a = gram_args(x, v, g);
  a.ws = static_cast<double*>(ws);
  return bt_gemm_run(a, 1, bt_stream(stream), 0, ws_bytes / 8);
}

extern "C" int64_t bt_ttm_ws_bytes(const int64_t* dims, int order, int mode, int64_t rows) {
  View3 v;
  if (!view3(dims, order, mode, v)) return 0;
  int64_t batch = 1;
  BtGemmArgs a = ttm_args(nullptr, v, nullptr, rows, 0, nullptr, batch);
  int64_t total = 0;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    const int64_t w = bt_gemm_ws_elems(a, nb);
    total = w > total ? w : total;
  }
  return total * 8;
}

int bt_ttm_last_tma(const double* x, int64_t rows, int64_t K, const double* u, int64_t R, double* y,
                    cudaStream_t st);

extern "C" int bt_ttm_f64(const double* x, const int64_t* dims, int order, int mode,
                          const double* u, int64_t rows, int transpose, double* y, void* ws,
                          int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_ttm_f64");
  View3 v;
  BT_REQUIRE(view3(dims, order, mode, v), BT_E_SHAPE, "mode %d out of range for order-%d tensor",
             mode, order);
  BT_REQUIRE(rows >= 0, BT_E_SHAPE, "ttm: negative row count");
  // Y(o, :, :) = U^T X(o, :, :) over a non-last mode with u given as U
  // (n x rows): the TMA-fed transposed-A kernel, C^T stored -- X(o) is read in
  // place as (n x inner) with inner contiguous (BT_TTM_TMA=0: the engine)
  static const bool ttm_tma = !(getenv("BT_TTM_TMA") && getenv("BT_TTM_TMA")[0] == '0');
  if (ttm_tma && transpose && v.inner > 1 && rows > 0 && v.n > 0 && v.outer <= 65535) {
    const int rc = bt_gemm_at_tma_ex(x, v.inner, v.n * v.inner, u, rows, y, v.inner, rows * v.inner,
                                     v.inner, rows, v.n, v.outer, 1, bt_stream(stream));
    if (rc != BT_E_VALUE) return rc;
  }
  // last mode, u given as U (n x rows) with more than 32 columns: the C5
  // tree kernel without its reduction epilogue (TMA-staged X and U tiles,
  // 128 x 64 output tiles); narrower outputs stay on the engine's 128 x 32 /
  // 128 x 16 tile classes
  static const bool last_tma = !(getenv("BT_TTM_LAST_TMA") && getenv("BT_TTM_LAST_TMA")[0] == '0');
  if (ttm_tma && last_tma && transpose && v.inner == 1 && rows > 32 && v.n > 0 && v.outer > 0) {
    const int rc = bt_ttm_last_tma(x, v.outer, v.n, u, rows, y, bt_stream(stream));
    if (rc != BT_E_VALUE) return rc;
  }
  int64_t batch = 1;
  BtGemmArgs a = ttm_args(x, v, u, rows, transpose, y, batch);
  a.ws = static_cast<double*>(ws);
  // the grid's z dimension caps one launch at 65535 batches
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    BtGemmArgs c = a;
    c.B.ptr = a.B.ptr + b0 * a.B.s_b;
    c.C = a.C + b0 * a.sCb;
    BT_TRY(bt_gemm_run(c, nb, bt_stream(stream), 0, ws_bytes / 8));
  }
  return BT_OK;
}
