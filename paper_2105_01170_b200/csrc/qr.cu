// Thin QR with a nonnegative R diagonal (decomp.py:182-193, used by
// blr_from_kruskal and the "qr" Kron split, reconstruct.py:212-216, 257-259).
// The operands are tall-skinny (extent x CP rank), so one CTA runs
// Householder QR in global memory: per column a block reduction for the
// reflector and warp-per-column dot products for the trailing update, then
// Q is formed by back-accumulating the reflectors; finally rows of R / columns
// of Q are flipped so diag(R) >= 0 (numpy's LAPACK result normalised the
// same way by the reference).
#include "bt_common.cuh"

namespace {

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// a: m x n (row-major, overwritten), vws: m x n reflectors, tau: n
__global__ void __launch_bounds__(256)
    householder_qr_kernel(double* a, int64_t m, int64_t n, double* vws, double* tau, double* q,
                          double* r) {
  __shared__ double red[8];
  __shared__ double sh[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t k = 0; k < n; ++k) {
    double s = 0.0;
    for (int64_t i = k + threadIdx.x; i < m; i += blockDim.x) s += a[i * n + k] * a[i * n + k];
    const double nrm2 = block_sum(s, red);
    if (threadIdx.x == 0) {
      const double x0 = a[k * n + k];
      const double nrm = sqrt(nrm2);
      const double alpha = (x0 > 0.0) ? -nrm : nrm;
      const double v0 = x0 - alpha;
      const double vn2 = nrm2 - x0 * x0 + v0 * v0;
      sh[0] = alpha;
      sh[1] = v0;
      sh[2] = (vn2 > 0.0) ? 2.0 / vn2 : 0.0;
      tau[k] = sh[2];
    }
    __syncthreads();
    const double v0 = sh[1], tk = sh[2];
    for (int64_t i = k + threadIdx.x; i < m; i += blockDim.x)
      vws[i * n + k] = (i == k) ? v0 : a[i * n + k];
    __syncthreads();
    // trailing columns: warp per column
    for (int64_t j = k + 1 + warp; j < n; j += blockDim.x >> 5) {
      double d = 0.0;
      for (int64_t i = k + lane; i < m; i += 32) d += vws[i * n + k] * a[i * n + j];
      d = warp_sum(d) * tk;
      for (int64_t i = k + lane; i < m; i += 32) a[i * n + j] -= d * vws[i * n + k];
    }
    __syncthreads();
    if (threadIdx.x == 0) a[k * n + k] = (tk > 0.0) ? sh[0] : a[k * n + k];
    for (int64_t i = k + 1 + threadIdx.x; i < m; i += blockDim.x) a[i * n + k] = 0.0;
    __syncthreads();
  }
  // Q = H_0 ... H_{n-1} [I_n; 0]
  for (int64_t idx = threadIdx.x; idx < m * n; idx += blockDim.x)
    q[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
  __syncthreads();
  for (int64_t k = n - 1; k >= 0; --k) {
    const double tk = tau[k];
    if (tk == 0.0) continue;
    for (int64_t j = warp; j < n; j += blockDim.x >> 5) {
      double d = 0.0;
      for (int64_t i = k + lane; i < m; i += 32) d += vws[i * n + k] * q[i * n + j];
      d = warp_sum(d) * tk;
      for (int64_t i = k + lane; i < m; i += 32) q[i * n + j] -= d * vws[i * n + k];
    }
    __syncthreads();
  }
  // sign normalisation: diag(R) >= 0
  for (int64_t idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int64_t i = idx / n, j = idx % n;
    const double d = a[i * n + i];
    const double sg = (d < 0.0) ? -1.0 : 1.0;
    r[idx] = (j >= i) ? sg * a[i * n + j] : 0.0;
  }
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int64_t j = idx % n;
    const double d = a[j * n + j];
    if (d < 0.0) q[idx] = -q[idx];
  }
}

}  // namespace

extern "C" int64_t bt_qr_thin_ws_bytes(int64_t m, int64_t n) { return (2 * m * n + n + 2) * 8; }

extern "C" int bt_qr_thin_f64(const double* a, int64_t m, int64_t n, double* q, double* r,
                              void* ws, int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_qr_thin_f64");
  BT_REQUIRE(n >= 1 && m >= n, BT_E_SHAPE, "qr_thin expects a tall or square matrix");
  BT_REQUIRE(ws_bytes >= bt_qr_thin_ws_bytes(m, n), BT_E_VALUE, "qr_thin: workspace too small");
  cudaStream_t st = bt_stream(stream);
  double* w = static_cast<double*>(ws);
  double* acopy = w;
  double* v = w + m * n;
  double* tau = v + m * n;
  BT_CUDA_CHECK(cudaMemcpyAsync(acopy, a, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, st));
  householder_qr_kernel<<<1, 256, 0, st>>>(acopy, m, n, v, tau, q, r);
  BT_LAUNCH_CHECK();
  return BT_OK;
}
