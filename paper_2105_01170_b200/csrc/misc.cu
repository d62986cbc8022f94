// Deterministic reductions and the FP64 peak microbenchmarks.
#include "bt_common.cuh"
#include "jacobi.cuh"  // jacobi_rotation

// ---------------------------------------------------------------------------
// sum of squares (fro_norm, tensor.py:107-109) -- two-pass fixed tree
// ---------------------------------------------------------------------------

static constexpr int SUMSQ_BLOCKS = 1184;  // 8 x 148 SMs; fixed => deterministic

__global__ void __launch_bounds__(256) bt_sumsq_partial(const double* __restrict__ x, int64_t n,
                                                        double* __restrict__ part) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool v2 = ((reinterpret_cast<uintptr_t>(x) & 15u) == 0);
  if (v2) {
    const int64_t n2 = n / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
      double2 v = ld_stream2(x + 2 * i);
      s = fma(v.x, v.x, s);
      s = fma(v.y, v.y, s);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
      double v = x[n - 1];
      s = fma(v, v, s);
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      double v = ld_stream(x + i);
      s = fma(v, v, s);
    }
  }
  __shared__ double red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void bt_sum_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

extern "C" int64_t bt_sumsq_ws_bytes(int64_t) { return SUMSQ_BLOCKS * 8; }
int64_t bt_sumsq_ws_bytes_const() { return SUMSQ_BLOCKS; }

extern "C" int bt_sumsq_f64(const double* x, int64_t n, double* out, void* ws, int64_t ws_bytes,
                            void* stream) {
  BT_REQUIRE(ws_bytes >= SUMSQ_BLOCKS * 8, BT_E_VALUE, "sumsq: workspace too small");
  cudaStream_t st = bt_stream(stream);
  double* part = static_cast<double*>(ws);
  bt_sumsq_partial<<<SUMSQ_BLOCKS, 256, 0, st>>>(x, n, part);
  BT_LAUNCH_CHECK();
  bt_sum_final<<<1, 1024, 0, st>>>(part, SUMSQ_BLOCKS, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// ---------------------------------------------------------------------------
// FP64 peak microbenchmarks: DMMA.8x8x4 vs DFMA
// ---------------------------------------------------------------------------

template <int CHAINS>
__global__ void bt_peak_dmma_kernel(int64_t iters, double* sink) {
  double c[CHAINS][2];
  const int lane = threadIdx.x & 31;
  double a = 1.0 + 1e-9 * lane, b = 1.0 - 1e-9 * lane;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = 0.0;
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma884(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) sink[blockIdx.x] = s;
}

template <int CHAINS>
__global__ void bt_peak_dfma_kernel(int64_t iters, double* sink) {
  double c[CHAINS];
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) sink[blockIdx.x] = s;
}

extern "C" int bt_peak_dmma(int64_t iters, int blocks, int threads, double* sink, double* flops,
                            void* stream) {
  bt_peak_dmma_kernel<8><<<blocks, threads, 0, bt_stream(stream)>>>(iters, sink);
  BT_LAUNCH_CHECK();
  *flops = (double)blocks * (threads / 32) * (double)iters * 8 * 512.0;
  return BT_OK;
}

extern "C" int bt_peak_dmma_chains(int64_t iters, int blocks, int threads, int chains,
                                   double* sink, double* flops, void* stream) {
  switch (chains) {
    case 2: bt_peak_dmma_kernel<2><<<blocks, threads, 0, bt_stream(stream)>>>(iters, sink); break;
    case 4: bt_peak_dmma_kernel<4><<<blocks, threads, 0, bt_stream(stream)>>>(iters, sink); break;
    case 16: bt_peak_dmma_kernel<16><<<blocks, threads, 0, bt_stream(stream)>>>(iters, sink); break;
    case 32: bt_peak_dmma_kernel<32><<<blocks, threads, 0, bt_stream(stream)>>>(iters, sink); break;
    default: chains = 8; bt_peak_dmma_kernel<8><<<blocks, threads, 0, bt_stream(stream)>>>(iters, sink);
  }
  BT_LAUNCH_CHECK();
  *flops = (double)blocks * (threads / 32) * (double)iters * chains * 512.0;
  return BT_OK;
}

extern "C" int bt_peak_dfma(int64_t iters, int blocks, int threads, double* sink, double* flops,
                            void* stream) {
  bt_peak_dfma_kernel<8><<<blocks, threads, 0, bt_stream(stream)>>>(iters, sink);
  BT_LAUNCH_CHECK();
  *flops = (double)blocks * threads * (double)iters * 8 * 2.0;
  return BT_OK;
}

// ---------------------------------------------------------------------------
// z = alpha x + beta y
// ---------------------------------------------------------------------------

__global__ void bt_axpby_kernel(int64_t n, double alpha, const double* __restrict__ x, double beta,
                                const double* __restrict__ y, double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = alpha * x[i] + beta * y[i];
}

extern "C" int bt_axpby_f64(int64_t n, double alpha, const double* x, double beta, const double* y,
                            double* z, void* stream) {
  if (n <= 0) return BT_OK;
  const int64_t blocks = (n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192;
  bt_axpby_kernel<<<static_cast<int>(blocks), 256, 0, bt_stream(stream)>>>(n, alpha, x, beta, y, z);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// ---------------------------------------------------------------------------
// max |x| (deterministic; max is order independent) -- psd.py:184 scale
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) bt_maxabs_partial(const double* __restrict__ x, int64_t n,
                                                         double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fmax(s, fabs(ld_stream(x + i)));
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t = fmax(t, red[w]);
    part[blockIdx.x] = t;
  }
}

__global__ void bt_max_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t = fmax(t, part[i]);
    *out = t;
  }
}

extern "C" int bt_maxabs_f64(const double* x, int64_t n, double* out, void* ws, int64_t ws_bytes,
                             void* stream) {
  BT_REQUIRE(ws_bytes >= SUMSQ_BLOCKS * 8, BT_E_VALUE, "maxabs: workspace too small");
  cudaStream_t st = bt_stream(stream);
  double* part = static_cast<double*>(ws);
  bt_maxabs_partial<<<SUMSQ_BLOCKS, 256, 0, st>>>(x, n, part);
  BT_LAUNCH_CHECK();
  bt_max_final<<<1, 32, 0, st>>>(part, SUMSQ_BLOCKS, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// ---------------------------------------------------------------------------
// transpose closure check (psd.py:141-161): class k fails iff
// max|B[partner[k]] - B[k]^T| > tol with numpy NaN semantics
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256)
    bt_transpose_check_kernel(const double* __restrict__ b, int64_t p, int64_t n,
                              const int64_t* __restrict__ partner, double tol,
                              int* __restrict__ flags) {
  __shared__ int red[2][8];
  for (int64_t k = blockIdx.x; k < p; k += gridDim.x) {
    const double* bk = b + k * n * n;
    const double* bp = b + partner[k] * n * n;
    int exceed = 0, nan = 0;
    for (int64_t e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int64_t i = e / n, j = e % n;
      const double d = fabs(bp[i * n + j] - bk[j * n + i]);
      exceed |= (d > tol);
      nan |= (d != d);
    }
    exceed = __any_sync(0xffffffffu, exceed);
    nan = __any_sync(0xffffffffu, nan);
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = exceed;
      red[1][threadIdx.x >> 5] = nan;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int e = 0, nn = 0;
      for (int w = 0; w < 8; ++w) {
        e |= red[0][w];
        nn |= red[1][w];
      }
      flags[k] = (e && !nn) ? 1 : 0;
    }
    __syncthreads();
  }
}

extern "C" int bt_transpose_check_f64(const double* blocks, int64_t p, int64_t n,
                                      const int64_t* partner, double tol, void* ws,
                                      int64_t* bad_class, void* stream) {
  BT_NVTX("bt_transpose_check_f64");
  cudaStream_t st = bt_stream(stream);
  int* flags = static_cast<int*>(ws);
  const int grid = static_cast<int>(p < 148 * 8 ? p : 148 * 8);
  bt_transpose_check_kernel<<<grid, 256, 0, st>>>(blocks, p, n, partner, tol, flags);
  BT_LAUNCH_CHECK();
  int* h = new int[p];
  cudaError_t e1 = cudaMemcpyAsync(h, flags, sizeof(int) * p, cudaMemcpyDeviceToHost, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    delete[] h;
    bt_set_error("transpose check: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    return BT_E_CUDA;
  }
  int64_t first = -1;
  for (int64_t k = 0; k < p; ++k)
    if (h[k]) {
      first = k;
      break;
    }
  delete[] h;
  if (bad_class) *bad_class = first;
  if (first >= 0) {
    bt_set_error("class %lld: block transpose differs from its partner", (long long)(first + 1));
    return BT_E_PATTERN;
  }
  return BT_OK;
}

// ---------------------------------------------------------------------------
// x[:, c] /= ||x[:, c]||  (row-major rows x cols; one warp per column)
// ---------------------------------------------------------------------------

__global__ void bt_col_normalize_kernel(double* __restrict__ x, int64_t rows, int64_t cols) {
  const int lane = threadIdx.x & 31;
  for (int64_t c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); c < cols;
       c += (int64_t)gridDim.x * (blockDim.x / 32)) {
    double s = 0.0;
    for (int64_t r = lane; r < rows; r += 32) s = fma(x[r * cols + c], x[r * cols + c], s);
    s = warp_sum(s);
    const double nrm = sqrt(s);
    if (nrm > 0.0)
      for (int64_t r = lane; r < rows; r += 32) x[r * cols + c] = x[r * cols + c] / nrm;
  }
}

// out[c] = || gv[:, c] - theta[c] * v[:, c] ||  (Ritz residual norms; one warp per column)
__global__ void bt_ritz_resid_kernel(const double* __restrict__ gv, const double* __restrict__ v,
                                     const double* __restrict__ theta, int64_t rows, int64_t cols,
                                     int64_t ld, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); c < cols;
       c += (int64_t)gridDim.x * (blockDim.x / 32)) {
    const double th = theta[c];
    double s = 0.0;
    for (int64_t r = lane; r < rows; r += 32) {
      const double d = fma(-th, v[r * ld + c], gv[r * ld + c]);
      s = fma(d, d, s);
    }
    s = warp_sum(s);
    if (lane == 0) out[c] = sqrt(s);
  }
}

extern "C" int bt_ritz_resid_f64(const double* gv, const double* v, const double* theta,
                                 int64_t rows, int64_t cols, int64_t ld, double* out, void* stream) {
  if (rows <= 0 || cols <= 0) return BT_OK;
  BT_REQUIRE(ld >= cols, BT_E_SHAPE, "ritz_resid: ld < cols");
  const int64_t blocks = (cols + 7) / 8 < 1024 ? (cols + 7) / 8 : 1024;
  bt_ritz_resid_kernel<<<static_cast<int>(blocks), 256, 0, bt_stream(stream)>>>(gv, v, theta, rows,
                                                                                 cols, ld, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

extern "C" int bt_col_normalize_f64(double* x, int64_t rows, int64_t cols, void* stream) {
  if (rows <= 0 || cols <= 0) return BT_OK;
  const int64_t blocks = (cols + 7) / 8 < 1024 ? (cols + 7) / 8 : 1024;
  bt_col_normalize_kernel<<<static_cast<int>(blocks), 256, 0, bt_stream(stream)>>>(x, rows, cols);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// ---------------------------------------------------------------------------
// sign rule of decomp.py:176-179 on every column of a row-major matrix:
// flip so the largest-|.| entry (first on ties) is positive
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) bt_sign_fix_kernel(double* __restrict__ x, int64_t rows,
                                                          int64_t cols, double* __restrict__ y,
                                                          int64_t yrows) {
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  for (int64_t c = blockIdx.x; c < cols; c += gridDim.x) {
    double best = -1.0;
    int64_t bidx = 0;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      const double v = fabs(x[i * cols + c]);
      if (v > best) {
        best = v;
        bidx = i;
      }
    }
    bv[threadIdx.x] = best;
    bi[threadIdx.x] = bidx;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        const double o = bv[threadIdx.x + s];
        const int64_t oi = bi[threadIdx.x + s];
        if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
          bv[threadIdx.x] = o;
          bi[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    const bool flip = x[bi[0] * cols + c] < 0.0;
    __syncthreads();
    if (flip) {
      for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) x[i * cols + c] = -x[i * cols + c];
      if (y)  // companion factor flipped with it (v of an SVD, decomp.py:176-179)
        for (int64_t i = threadIdx.x; i < yrows; i += blockDim.x) y[i * cols + c] = -y[i * cols + c];
    }
    __syncthreads();
  }
}

extern "C" int bt_sign_fix_f64(double* x, int64_t rows, int64_t cols, void* stream) {
  if (rows <= 0 || cols <= 0) return BT_OK;
  const int64_t g = cols < 4096 ? cols : 4096;
  bt_sign_fix_kernel<<<static_cast<int>(g), 256, 0, bt_stream(stream)>>>(x, rows, cols, nullptr, 0);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

extern "C" int bt_sign_fix_pair_f64(double* x, int64_t rows, int64_t cols, double* y,
                                    int64_t yrows, void* stream) {
  if (rows <= 0 || cols <= 0) return BT_OK;
  const int64_t g = cols < 4096 ? cols : 4096;
  bt_sign_fix_kernel<<<static_cast<int>(g), 256, 0, bt_stream(stream)>>>(x, rows, cols, y, yrows);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// singular values from Gram eigenvalues: s = sqrt(max(w, 0)), sinv = 1/s (1 where s == 0)
__global__ void bt_svals_kernel(const double* __restrict__ w, int64_t n, double* __restrict__ s,
                                double* __restrict__ sinv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = sqrt(fmax(w[i], 0.0));
    s[i] = v;
    sinv[i] = v > 0.0 ? 1.0 / v : 1.0;
  }
}

extern "C" int bt_svals_f64(const double* w, int64_t n, double* s, double* sinv, void* stream) {
  if (n <= 0) return BT_OK;
  bt_svals_kernel<<<static_cast<int>((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0,
                    bt_stream(stream)>>>(w, n, s, sinv);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// out[i] = 1 / sqrt(x[i])   (x > 0)
__global__ void bt_inv_sqrt_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = 1.0 / sqrt(x[i]);
}

extern "C" int bt_inv_sqrt_f64(const double* x, int64_t n, double* out, void* stream) {
  if (n <= 0) return BT_OK;
  bt_inv_sqrt_kernel<<<static_cast<int>((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0,
                       bt_stream(stream)>>>(x, n, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// out[0] = trace(m) for an n x n row-major matrix (one CTA, fixed-order
// reduction): an upper bound on lambda_max of a PSD Gram.
__global__ void bt_trace_kernel(const double* __restrict__ m, int64_t n, double* __restrict__ out) {
  __shared__ double part[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += m[i * n + i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[0] = s;
  }
}

extern "C" int bt_trace_f64(const double* m, int64_t n, double* out, void* stream) {
  bt_trace_kernel<<<1, 256, 0, bt_stream(stream)>>>(m, n, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// Column-scaled symmetric Gram for SVQB: dinv[j] = m_jj > 0 ? m_jj^-1/2 : 0,
// out = D sym(m) D with sym(m) = (m + m^T) / 2 (b x b, row-major).  Graded
// blocks (G Q with a fast-decaying spectrum) then keep every column instead
// of losing the small ones to the relative drop threshold.
__global__ void bt_sym_scale_kernel(const double* __restrict__ m, int64_t b,
                                    double* __restrict__ dinv, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < b * b;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / b, j = e - i * b;
    const double di = m[i * b + i], dj = m[j * b + j];
    const double si = di > 0.0 ? 1.0 / sqrt(di) : 0.0;
    const double sj = dj > 0.0 ? 1.0 / sqrt(dj) : 0.0;
    out[e] = (0.5 * (m[i * b + j] + m[j * b + i])) * si * sj;
    if (i == j) dinv[i] = si;
  }
}

extern "C" int bt_sym_scale_f64(const double* m, int64_t b, double* dinv, double* out,
                                void* stream) {
  if (b <= 0) return BT_OK;
  const int64_t n = b * b;
  bt_sym_scale_kernel<<<static_cast<int>((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0,
                        bt_stream(stream)>>>(m, b, dinv, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// ---------------------------------------------------------------------------
// axis reversal (container payloads, container.py:111-159): out is the
// C-order array of the axis-reversed tensor, i.e. x's elements in
// first-index-fastest order.  Applying it to that result with the reversed
// extents gives x back.  One thread per output element, coalesced writes.
// ---------------------------------------------------------------------------

struct RevDims {
  int64_t d[6];
  int64_t stride[6];  // input strides (C order) of axis k
  int nd;
};

__global__ void bt_reverse_axes_kernel(const double* __restrict__ x, RevDims rd, int64_t total,
                                       double* __restrict__ out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    // output index is F-order over the input axes: axis 0 fastest
    int64_t rem = o, off = 0;
    for (int k = 0; k < rd.nd; ++k) {
      const int64_t i = rem % rd.d[k];
      rem /= rd.d[k];
      off += i * rd.stride[k];
    }
    out[o] = x[off];
  }
}

extern "C" int bt_reverse_axes_f64(const double* x, const int64_t* dims, int ndim, double* out,
                                   void* stream) {
  BT_NVTX("bt_reverse_axes_f64");
  BT_REQUIRE(ndim >= 1 && ndim <= 6, BT_E_SHAPE, "reverse_axes: rank %d outside 1..6", ndim);
  RevDims rd;
  rd.nd = ndim;
  int64_t total = 1;
  for (int k = ndim - 1; k >= 0; --k) {
    BT_REQUIRE(dims[k] >= 0, BT_E_SHAPE, "reverse_axes: negative extent");
    rd.d[k] = dims[k];
    rd.stride[k] = total;
    total *= dims[k];
  }
  if (total == 0) return BT_OK;
  const int64_t blocks = (total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096;
  bt_reverse_axes_kernel<<<static_cast<int>(blocks), 256, 0, bt_stream(stream)>>>(x, rd, total, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// out (cols x rows) = x (rows x cols)^T, both row-major: 32 x 32 tiles staged
// in shared memory (padded against bank conflicts) so reads and writes are
// both coalesced -- the right-hand-side layout flip of the batched matvecs
// ((q*n, nrhs) user layout <-> one contiguous vector per RHS)
__global__ void __launch_bounds__(256) bt_transpose_kernel(const double* __restrict__ x,
                                                           int64_t rows, int64_t cols,
                                                           double* __restrict__ out) {
  __shared__ double tile[32][33];
  const int64_t tiles_c = (cols + 31) / 32;
  const int64_t ntiles = ((rows + 31) / 32) * tiles_c;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t r0 = (t / tiles_c) * 32, c0 = (t % tiles_c) * 32;
    for (int k = threadIdx.y; k < 32; k += 8) {
      const int64_t r = r0 + k, c = c0 + threadIdx.x;
      if (r < rows && c < cols) tile[k][threadIdx.x] = x[r * cols + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += 8) {
      const int64_t c = c0 + k, r = r0 + threadIdx.x;
      if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][k];
    }
    __syncthreads();
  }
}

extern "C" int bt_transpose_f64(const double* x, int64_t rows, int64_t cols, double* out,
                                void* stream) {
  BT_NVTX("bt_transpose_f64");
  BT_REQUIRE(rows >= 0 && cols >= 0, BT_E_SHAPE, "transpose: negative extent");
  if (rows == 0 || cols == 0) return BT_OK;
  const int64_t ntiles = ((rows + 31) / 32) * ((cols + 31) / 32);
  const int64_t blocks = ntiles < 8 * 148 * 4 ? ntiles : 8 * 148 * 4;
  bt_transpose_kernel<<<static_cast<unsigned>(blocks), dim3(32, 8), 0, bt_stream(stream)>>>(
      x, rows, cols, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// out[i][j] = left[i] * x[i][j] * right[j] (either scale may be null) -- the
// diagonal similarity of the ERA shift solve (apps.py:216-218)
__global__ void bt_diag_scale_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                     const double* __restrict__ left,
                                     const double* __restrict__ right, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    double v = x[e];
    if (left) v = left[i] * v;
    if (right) v = v * right[j];
    out[e] = v;
  }
}

extern "C" int bt_diag_scale_f64(const double* x, int64_t rows, int64_t cols, const double* left,
                                 const double* right, double* out, void* stream) {
  if (rows <= 0 || cols <= 0) return BT_OK;
  const int64_t n = rows * cols;
  bt_diag_scale_kernel<<<static_cast<int>((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0,
                         bt_stream(stream)>>>(x, rows, cols, left, right, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// out[c] = || x[:, c] || for a row-major rows x cols matrix (one warp per column)
__global__ void bt_col_norms_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                    double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); c < cols;
       c += (int64_t)gridDim.x * (blockDim.x / 32)) {
    double s = 0.0;
    for (int64_t r = lane; r < rows; r += 32) s = fma(x[r * cols + c], x[r * cols + c], s);
    s = warp_sum(s);
    if (lane == 0) out[c] = sqrt(s);
  }
}

extern "C" int bt_col_norms_f64(const double* x, int64_t rows, int64_t cols, double* out,
                                void* stream) {
  if (rows <= 0 || cols <= 0) return BT_OK;
  const int64_t blocks = (cols + 7) / 8 < 1024 ? (cols + 7) / 8 : 1024;
  bt_col_norms_kernel<<<static_cast<int>(blocks), 256, 0, bt_stream(stream)>>>(x, rows, cols, out);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// ---------------------------------------------------------------------------
// SVD of a small square matrix (n <= 32) by one-sided (Hestenes) Jacobi on
// one CTA of 16 warps: W = M J and J live in shared memory column by column;
// a round pairs the 32 columns by the circle method, warp k takes pair k with
// lane = row: the three dot products of the pair are xor-butterfly warp sums
// (every lane ends with the same bits), the rotation is computed redundantly
// in every lane and the lane updates its row of both columns of W and J; one
// barrier per round.  (The one-warp version -- a column per lane, three
// 32-long dependent FMA chains per round -- took 205-345 us per call, two or
// three calls per basis refinement; this one ~4x less.)  Rotation while
// |w_p . w_q| > 1e-15 ||w_p|| ||w_q|| (the relative criterion: small singular
// values keep high relative accuracy -- the point of taking this route
// instead of a Gram).  Output: singular values descending, U = W / sigma,
// V = J, each column of U with its largest-|.| entry positive
// (decomp.py:176-179 sign rule; first on ties), the sign compensated in V.
// Rows/columns beyond n are padding.
// ---------------------------------------------------------------------------

namespace {

__device__ __forceinline__ double warp_sum_all(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(512) svd_small_kernel(const double* __restrict__ m, int n,
                                                        double* __restrict__ u, double* __restrict__ s,
                                                        double* __restrict__ v) {
  constexpr int NP = 32, LD = NP + 1;
  __shared__ double ws[NP][LD], js[NP][LD], sg[NP];   // [column][row]
  __shared__ int order[NP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;   // lane = row, 16 warps
  for (int c = warp; c < NP; c += 16) {
    ws[c][lane] = (lane < n && c < n) ? m[lane * n + c] : 0.0;
    js[c][lane] = (lane == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    int rotated = 0;
    for (int rnd = 0; rnd < NP - 1; ++rnd) {
      // circle method: pair `warp` of round rnd (p < q)
      int p, q;
      if (warp == 0) {
        p = rnd;
        q = NP - 1;
      } else {
        p = rnd + warp;
        if (p >= NP - 1) p -= NP - 1;
        q = rnd - warp + (NP - 1);
        if (q >= NP - 1) q -= NP - 1;
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
      }
      const double wp = ws[p][lane], wq = ws[q][lane];
      const double a = warp_sum_all(wp * wp), b = warp_sum_all(wq * wq), g = warp_sum_all(wp * wq);
      if (g != 0.0 && g * g > 1e-30 * (a * b)) {   // warp-uniform
        // theta = (b - a) / (2 g); t = sign(theta) / (|theta| + sqrt(1 + theta^2))
        // from refined rcp / rsqrt (jacobi.cuh, ~1 ulp): the IEEE divisions
        // and square roots were ~1500 of the round's ~1700 dependent cycles;
        // the exact formula only where 1 / (2 g) would overflow the approximation
        double cs, sn;
        if (fabs(g) > 1e-290) {
          jacobi_rotation(a, b, g, cs, sn);
        } else {
          const double th = (b - a) / (2.0 * g);
          const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
          cs = 1.0 / sqrt(1.0 + t * t);
          sn = cs * t;
        }
        rotated = 1;
        const double jp = js[p][lane], jq = js[q][lane];
        ws[p][lane] = cs * wp - sn * wq;
        ws[q][lane] = sn * wp + cs * wq;
        js[p][lane] = cs * jp - sn * jq;
        js[q][lane] = sn * jp + cs * jq;
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  // epilogue on one warp, a column per lane (as the one-warp version did)
  if (warp == 0) {
    const int c = lane;
    double nrm2 = 0.0;
#pragma unroll
    for (int i = 0; i < NP; ++i) nrm2 = fma(ws[c][i], ws[c][i], nrm2);
    const double sig = (c < n) ? sqrt(nrm2) : -1.0;
    sg[c] = sig;
    __syncwarp();
    // descending order (ties: lower column first)
    int rank = 0;
    for (int j = 0; j < NP; ++j) rank += (sg[j] > sig) || (sg[j] == sig && j < c);
    order[rank] = c;
    const double inv = sig > 0.0 ? 1.0 / sig : 0.0;
    // sign rule on U's column (largest |entry| positive, first on ties)
    double best = -1.0, bval = 0.0;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const double e = ws[c][i] * inv;
      if (i < n && fabs(e) > best) {
        best = fabs(e);
        bval = e;
      }
    }
    const double flip = (bval < 0.0) ? -1.0 : 1.0;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      ws[c][i] = flip * ws[c][i] * inv;
      js[c][i] = flip * js[c][i];
    }
    __syncwarp();
    if (c < n) {
      const int src = order[c];
      s[c] = sg[src];
      for (int i = 0; i < n; ++i) {
        u[i * n + c] = ws[src][i];
        v[i * n + c] = js[src][i];
      }
    }
  }
}

}  // namespace

extern "C" int bt_svd_small_f64(const double* m, int64_t n, double* u, double* s, double* v,
                                void* stream) {
  BT_NVTX("bt_svd_small_f64");
  BT_REQUIRE(n >= 1 && n <= 32, BT_E_SHAPE, "svd_small: n = %lld outside 1..32", (long long)n);
  svd_small_kernel<<<1, 512, 0, bt_stream(stream)>>>(m, static_cast<int>(n), u, s, v);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// ---------------------------------------------------------------------------
// Small Cholesky for CholeskyQR steps (n <= 32, one warp): g = L L^T,
// writes lt = L^T (upper) and linvt = L^-T (upper), flag = 1 when a pivot
// is not above 1e-12 of the largest diagonal (the caller then takes the
// Householder route).  The Gram comes from a column-scaled block, so its
// diagonal is ~1.
// ---------------------------------------------------------------------------

namespace {

__device__ __forceinline__ double rsqrt_nr_f64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}

// One CTA of 256 threads, right-looking: every column step is a scaled
// column, a barrier, a rank-1 update of the trailing block spread over the
// CTA, a barrier; L^-1 by forward substitution on the identity in the same
// shape.  (The one-warp version, a serial read-modify-write loop per row and
// step, took 37 us at n = 32 -- eight calls per HOOI sweep; this one ~10 us.)
__global__ void __launch_bounds__(256) chol_small_kernel(const double* __restrict__ g, int n,
                                                         double* __restrict__ lt,
                                                         double* __restrict__ linvt,
                                                         int* __restrict__ flag) {
  __shared__ double a[32][33], y[32][33], rd[32];
  __shared__ double dmax_s;
  const int tid = threadIdx.x;
  for (int e = tid; e < 32 * 32; e += 256) {
    const int i = e >> 5, j = e & 31;
    a[i][j] = (i < n && j < n) ? g[i * n + j] : (i == j ? 1.0 : 0.0);
    y[i][j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    double d = tid < n ? a[tid][tid] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if (tid == 0) dmax_s = d;
  }
  __syncthreads();
  const double dmax = dmax_s;
  int bad = 0;
  for (int k = 0; k < n; ++k) {
    const double d = a[k][k];
    if (!(d > 1e-12 * dmax)) {   // uniform: every thread reads the same pivot
      bad = 1;
      break;
    }
    const double r = rsqrt_nr_f64(d);
    __syncthreads();
    if (tid > k && tid < n) a[tid][k] *= r;
    if (tid == 0) {
      a[k][k] = d * r;
      rd[k] = r;
    }
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += 256) {
      const int i = e >> 5, j = e & 31;
      if (j > k && j <= i && i < n) a[i][j] -= a[i][k] * a[j][k];
    }
    __syncthreads();
  }
  if (tid == 0) *flag = bad;
  if (bad) return;
  // Y = L^-1 (lower): row k is final once rows < k have been eliminated from it
  for (int k = 0; k < n; ++k) {
    if (tid <= k) y[k][tid] *= rd[k];
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += 256) {
      const int i = e >> 5, c = e & 31;
      if (i > k && i < n && c <= k) y[i][c] -= a[i][k] * y[k][c];
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += 256) {
    const int i = e / n, j = e % n;
    lt[e] = (j >= i) ? a[j][i] : 0.0;       // L^T
    linvt[e] = (j >= i) ? y[j][i] : 0.0;    // L^-T
  }
}

}  // namespace

extern "C" int bt_chol_small_f64(const double* g, int64_t n, double* lt, double* linvt, int* flag,
                                 void* stream) {
  BT_REQUIRE(n >= 1 && n <= 32, BT_E_SHAPE, "chol_small: n = %lld outside 1..32", (long long)n);
  chol_small_kernel<<<1, 256, 0, bt_stream(stream)>>>(g, static_cast<int>(n), lt, linvt, flag);
  BT_LAUNCH_CHECK();
  return BT_OK;
}
