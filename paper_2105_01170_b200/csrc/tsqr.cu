// Tall-skinny Householder QR (TSQR) for m x n, n <= 32: the orthonormal
// factor of a basis refinement step (_linalg._refine_basis_qr), where
// CholeskyQR would square the conditioning (the blocks there span singular
// values over 10+ orders of magnitude) and the one-CTA Householder kernel of
// qr.cu is latency bound at thousands of rows.
//
//   level 1: the rows split into blocks of TS_RB; each CTA factors its block
//            in shared memory (Householder, warp per column for the
//            reflector dots) and keeps its reflectors;
//   level 2: one CTA factors the stacked n x n R factors (nb * n rows);
//   Q:       block i's rows of Q = H_i [Q2_i; 0] (its reflectors applied to
//            its n-row slice of level 2's Q).
// R's diagonal is made nonnegative (numpy/LAPACK's qr normalised as in
// decomp.py:182-193).  Deterministic: fixed reduction orders, no atomics.
#include "bt_common.cuh"

namespace {

constexpr int TS_RB = 512;      // rows per level-1 block
constexpr int TS_NMAX = 32;
constexpr int TS_THREADS = 256;

// Householder QR of a (rows x n) block in shared memory a (leading dim lda =
// n + 1): reflector k is
// stored in place below the diagonal with v_k = 1 implied, tau[k] its
// scalar; the upper triangle ends up as R (diagonal alpha_k).
__device__ void smem_householder(double* a, int rows, int n, int lda, double* tau, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < n; ++k) {
    // ||a_k[k:]||^2 by warp 0..: block reduction
    double s = 0.0;
    for (int i = k + 1 + threadIdx.x; i < rows; i += blockDim.x) s = fma(a[i * lda + k], a[i * lda + k], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tail2 = 0.0;
      for (int w = 0; w < nw; ++w) tail2 += red[w];
      const double x0 = a[k * lda + k];
      if (tail2 == 0.0) {
        tau[k] = 0.0;            // already triangular in this column
        red[32] = 1.0;
      } else {
        const double nrm = sqrt(x0 * x0 + tail2);
        const double alpha = (x0 > 0.0) ? -nrm : nrm;
        const double v0 = x0 - alpha;
        tau[k] = -v0 / alpha;    // H = I - tau v v^T with v = [1, x_tail / v0]
        red[32] = 1.0 / v0;
        a[k * lda + k] = alpha;
      }
    }
    __syncthreads();
    const double sc = red[32], tk = tau[k];
    if (tk != 0.0)
      for (int i = k + 1 + threadIdx.x; i < rows; i += blockDim.x) a[i * lda + k] *= sc;
    __syncthreads();
    if (tk != 0.0) {
      // trailing columns j > k: warp per column, w = v^T a_j, a_j -= tau w v
      for (int j = k + 1 + warp; j < n; j += nw) {
        double d = (lane == 0) ? a[k * lda + j] : 0.0;
        for (int i = k + 1 + lane; i < rows; i += 32) d = fma(a[i * lda + k], a[i * lda + j], d);
        d = warp_sum(d) * tk;
        if (lane == 0) a[k * lda + j] -= d;
        for (int i = k + 1 + lane; i < rows; i += 32) a[i * lda + j] -= d * a[i * lda + k];
      }
    }
    __syncthreads();
  }
}

// apply H_0 ... H_{n-1} (reflectors in a's lower part) to c (rows x n, ldc):
// c = H_0 (H_1 (... H_{n-1} c)), i.e. Q c
__device__ void smem_apply_q(const double* a, int rows, int n, int lda, const double* tau, double* c,
                             int ldc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = n - 1; k >= 0; --k) {
    const double tk = tau[k];
    if (tk != 0.0) {
      for (int j = warp; j < n; j += nw) {
        double d = (lane == 0) ? c[k * ldc + j] : 0.0;
        for (int i = k + 1 + lane; i < rows; i += 32) d = fma(a[i * lda + k], c[i * ldc + j], d);
        d = warp_sum(d) * tk;
        if (lane == 0) c[k * ldc + j] -= d;
        for (int i = k + 1 + lane; i < rows; i += 32) c[i * ldc + j] -= d * a[i * lda + k];
      }
    }
    __syncthreads();
  }
}

// level 1: block b of x (m x n) -> reflectors (refl[b]: TS_RB x n), tau
// (taus[b]: n), R into the stacked matrix rs (b * n .. b * n + n rows)
__global__ void __launch_bounds__(TS_THREADS)
    tsqr_local_kernel(const double* __restrict__ x, int64_t m, int n, double* __restrict__ refl,
                      double* __restrict__ taus, double* __restrict__ rs) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double tau[TS_NMAX], red[33];
  const int lda = n + 1;
  double* a = sm;
  const int64_t r0 = (int64_t)blockIdx.x * TS_RB;
  const int rows = static_cast<int>(m - r0 < TS_RB ? m - r0 : TS_RB);
  for (int e = threadIdx.x; e < TS_RB * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    a[i * lda + j] = (i < rows) ? x[(r0 + i) * n + j] : 0.0;
  }
  __syncthreads();
  smem_householder(a, TS_RB, n, lda, tau, red);
  double* rb = rs + (int64_t)blockIdx.x * n * n;
  double* vb = refl + (int64_t)blockIdx.x * TS_RB * n;
  for (int e = threadIdx.x; e < TS_RB * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    vb[e] = a[i * lda + j];
    if (i < n) rb[e] = (j >= i) ? a[i * lda + j] : 0.0;
  }
  if (threadIdx.x < n) taus[(int64_t)blockIdx.x * n + threadIdx.x] = tau[threadIdx.x];
}

// level 2 (one CTA): QR of the stacked R (rows = nb * n); writes R (sign
// normalised, n x n), the explicit Q2 (rows x n, columns flipped with R's
// rows) and the sign vector
__global__ void __launch_bounds__(TS_THREADS)
    tsqr_top_kernel(const double* __restrict__ rs, int rows, int n, double* __restrict__ r,
                    double* __restrict__ q2) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double tau[TS_NMAX], red[33], sgn[TS_NMAX];
  const int lda = n + 1;
  double* a = sm;
  double* c = sm + rows * lda;
  for (int e = threadIdx.x; e < rows * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    a[i * lda + j] = rs[e];
    c[i * lda + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  smem_householder(a, rows, n, lda, tau, red);
  if (threadIdx.x < n) sgn[threadIdx.x] = (a[threadIdx.x * lda + threadIdx.x] < 0.0) ? -1.0 : 1.0;
  smem_apply_q(a, rows, n, lda, tau, c, lda);
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    r[e] = (j >= i) ? sgn[i] * a[i * lda + j] : 0.0;
  }
  for (int e = threadIdx.x; e < rows * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    q2[e] = c[i * lda + j] * sgn[j];
  }
}

// Q rows of block b: H_b [Q2_b; 0]
__global__ void __launch_bounds__(TS_THREADS)
    tsqr_q_kernel(const double* __restrict__ refl, const double* __restrict__ taus,
                  const double* __restrict__ q2, int64_t m, int n, double* __restrict__ q) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double tau[TS_NMAX];
  const int lda = n + 1;
  double* c = sm;   // the reflectors are read from global memory (L2)
  const int64_t r0 = (int64_t)blockIdx.x * TS_RB;
  const int rows = static_cast<int>(m - r0 < TS_RB ? m - r0 : TS_RB);
  const double* vb = refl + (int64_t)blockIdx.x * TS_RB * n;
  for (int e = threadIdx.x; e < TS_RB * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    c[i * lda + j] = (i < n) ? q2[((int64_t)blockIdx.x * n + i) * n + j] : 0.0;
  }
  if (threadIdx.x < n) tau[threadIdx.x] = taus[(int64_t)blockIdx.x * n + threadIdx.x];
  __syncthreads();
  smem_apply_q(vb, TS_RB, n, n, tau, c, lda);
  for (int e = threadIdx.x; e < rows * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    q[(r0 + i) * n + j] = c[i * lda + j];
  }
}

}  // namespace

extern "C" int64_t bt_tsqr_ws_bytes(int64_t m, int64_t n) {
  const int64_t nb = bt_cdiv(m, TS_RB);
  return (nb * TS_RB * n + nb * n + nb * n * n + nb * n * n + 16) * 8;
}

extern "C" int bt_tsqr_f64(const double* x, int64_t m, int64_t n, double* q, double* r, void* ws,
                           int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_tsqr_f64");
  BT_REQUIRE(n >= 1 && n <= TS_NMAX && m >= n, BT_E_SHAPE, "tsqr: needs m >= n, 1 <= n <= 32");
  const int64_t nb = bt_cdiv(m, TS_RB);
  const int64_t top_rows = nb * n;
  const size_t top_sm = sizeof(double) * 2 * top_rows * (n + 1);
  BT_REQUIRE(top_sm <= 220 * 1024, BT_E_SHAPE, "tsqr: %lld rows exceed one level of stacking",
             (long long)m);
  BT_REQUIRE(ws_bytes >= bt_tsqr_ws_bytes(m, n), BT_E_VALUE, "tsqr: workspace too small");
  cudaStream_t st = bt_stream(stream);
  double* w = static_cast<double*>(ws);
  double* refl = w;
  double* taus = refl + nb * TS_RB * n;
  double* rs = taus + nb * n;
  double* q2 = rs + nb * n * n;
  const int ni = static_cast<int>(n);
  const size_t blk_sm = sizeof(double) * TS_RB * (n + 1);
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(tsqr_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       220 * 1024));
    BT_CUDA_CHECK(cudaFuncSetAttribute(tsqr_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       220 * 1024));
    BT_CUDA_CHECK(cudaFuncSetAttribute(tsqr_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       220 * 1024));
    attr = true;
  }
  tsqr_local_kernel<<<static_cast<unsigned>(nb), TS_THREADS, blk_sm, st>>>(x, m, ni, refl, taus, rs);
  BT_LAUNCH_CHECK();
  tsqr_top_kernel<<<1, TS_THREADS, top_sm, st>>>(rs, static_cast<int>(top_rows), ni, r, q2);
  BT_LAUNCH_CHECK();
  tsqr_q_kernel<<<static_cast<unsigned>(nb), TS_THREADS, blk_sm, st>>>(refl, taus, q2, m, ni, q);
  BT_LAUNCH_CHECK();
  return BT_OK;
}
