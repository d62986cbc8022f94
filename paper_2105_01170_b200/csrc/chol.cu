// Cholesky factorisation and lower-triangular inverse (decomp.py:196-212
// `cholesky`, psd.py:248-257 `spd_compress` anchor factor and the
// L^-1 B L^-T scalings of its remainder blocks).
//
// Blocked right-looking Cholesky with 64-wide panels: the diagonal block is
// factored (and inverted) in shared memory by one CTA, the panel below it is
// L21 = A21 L11^-T (one DMMA GEMM against the explicit 64 x 64 inverse), and
// the trailing matrix takes A22 -= L21 L21^T (one DMMA GEMM).  The inverse
// L^-1 is blocked forward substitution over block rows with the same two
// GEMM shapes.  Only the lower triangle of the input is read (LAPACK potrf
// convention); a non-positive pivot returns BT_E_NOT_PD with the 1-based
// pivot index, read back once at the end (a failed panel poisons nothing:
// later panels see the device flag and return immediately).
#include "bt_common.cuh"
#include "gemm.cuh"

int bt_gemm_run(BtGemmArgs g, int64_t batch, cudaStream_t st, int want_splits, int64_t ws_elems);

namespace {

constexpr int NB = 64;            // panel width
constexpr int LDS = NB + 1;       // padded smem row

// Factor the kb x kb diagonal block at (k0, k0) of l (row-major, ld n) in
// shared memory; write L11 back (lower; upper left untouched) and its
// inverse (kb x kb, ld NB, zero upper) to dinv.  info: 0 or 1-based pivot.
__global__ void __launch_bounds__(256)
    potrf_diag_kernel(double* __restrict__ l, int64_t n, int64_t k0, int kb,
                      double* __restrict__ dinv, int64_t* __restrict__ info) {
  extern __shared__ double smem_chol[];
  double* s = smem_chol;
  double* x = smem_chol + NB * LDS;
  __shared__ int bad;
  if (*info != 0) return;  // an earlier panel failed
  const int tid = threadIdx.x;
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    const int i = e / kb, j = e % kb;
    s[i * LDS + j] = (j <= i) ? l[(k0 + i) * n + k0 + j] : 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int k = 0; k < kb; ++k) {
    if (tid == 0) {
      const double d = s[k * LDS + k];
      if (!(d > 0.0)) {
        bad = 1;
        *info = k0 + k + 1;
      } else {
        s[k * LDS + k] = sqrt(d);
      }
    }
    __syncthreads();
    if (bad) return;
    const double dk = s[k * LDS + k];
    for (int i = k + 1 + tid; i < kb; i += blockDim.x) s[i * LDS + k] /= dk;
    __syncthreads();
    const int m = kb - k - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = k + 1 + e / m, j = k + 1 + e % m;
      if (j <= i) s[i * LDS + j] -= s[i * LDS + k] * s[j * LDS + k];
    }
    __syncthreads();
  }
  // inverse: column j by forward substitution (one thread per column)
  if (tid < kb) {
    const int j = tid;
    for (int i = 0; i < kb; ++i) {
      double v = (i == j) ? 1.0 : 0.0;
      if (i > j) {
        for (int k = j; k < i; ++k) v -= s[i * LDS + k] * x[k * LDS + j];
      }
      x[i * LDS + j] = (i < j) ? 0.0 : v / s[i * LDS + i];
    }
  }
  __syncthreads();
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    const int i = e / kb, j = e % kb;
    if (j <= i) l[(k0 + i) * n + k0 + j] = s[i * LDS + j];
    dinv[i * NB + j] = x[i * LDS + j];
  }
}

// inverse of every kb x kb diagonal block of a lower-triangular l (one CTA per block)
__global__ void __launch_bounds__(64)
    diag_inv_kernel(const double* __restrict__ l, int64_t n, double* __restrict__ dinv) {
  extern __shared__ double smem_chol[];
  double* s = smem_chol;
  double* x = smem_chol + NB * LDS;
  const int64_t k0 = (int64_t)blockIdx.x * NB;
  const int kb = (int)((n - k0) < NB ? (n - k0) : NB);
  const int tid = threadIdx.x;
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    const int i = e / kb, j = e % kb;
    s[i * LDS + j] = (j <= i) ? l[(k0 + i) * n + k0 + j] : 0.0;
  }
  __syncthreads();
  if (tid < kb) {
    const int j = tid;
    for (int i = 0; i < kb; ++i) {
      double v = (i == j) ? 1.0 : 0.0;
      if (i > j) {
        for (int k = j; k < i; ++k) v -= s[i * LDS + k] * x[k * LDS + j];
      }
      x[i * LDS + j] = (i < j) ? 0.0 : v / s[i * LDS + i];
    }
  }
  __syncthreads();
  double* out = dinv + (int64_t)blockIdx.x * NB * NB;
  for (int e = tid; e < kb * kb; e += blockDim.x) out[(e / kb) * NB + e % kb] = x[(e / kb) * LDS + e % kb];
}

__global__ void copy_lower_kernel(const double* __restrict__ a, int64_t n, double* __restrict__ l) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n;
       e += (int64_t)gridDim.x * blockDim.x)
    l[e] = a[e];
}

__global__ void zero_upper_kernel(double* __restrict__ l, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n;
       e += (int64_t)gridDim.x * blockDim.x)
    if (e % n > e / n) l[e] = 0.0;
}

// rows [i0, i0+bi) of the identity (bi x w, ld w)
__global__ void identity_rows_kernel(double* __restrict__ t, int64_t i0, int bi, int64_t w) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < bi * w;
       e += (int64_t)gridDim.x * blockDim.x)
    t[e] = (e % w == i0 + e / w) ? 1.0 : 0.0;
}

BtGemmArgs plain_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t sAm,
                      int64_t sAk, const double* B, int64_t sBn, int64_t sBk, double* C,
                      int64_t sCm, double alpha, double beta) {
  BtGemmArgs g;
  memset(&g, 0, sizeof(g));
  g.M = M;
  g.N = N;
  g.Kin = K;
  g.Kout = 1;
  g.A = BtOperand{A, sAm, 0, sAk, 0};
  g.B = BtOperand{B, sBn, 0, sBk, 0};
  g.C = C;
  g.sCm = sCm;
  g.sCn = 1;
  g.alpha = alpha;
  g.beta = beta;
  return g;
}

int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr size_t kSmem = 2 * NB * LDS * sizeof(double);

int set_smem() {
  static int done = 0;
  if (!done) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(potrf_diag_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    BT_CUDA_CHECK(cudaFuncSetAttribute(diag_inv_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    done = 1;
  }
  return BT_OK;
}

}  // namespace

extern "C" int64_t bt_cholesky_ws_bytes(int64_t n) {
  // info + dinv (NB x NB) + panel (n x NB)
  return 64 + (int64_t)NB * NB * 8 + (n > 0 ? n : 0) * NB * 8;
}

extern "C" int bt_cholesky_f64(const double* a, int64_t n, double* l, void* ws, int64_t* bad_pivot,
                               void* stream) {
  BT_NVTX("bt_cholesky_f64");
  BT_REQUIRE(n >= 1, BT_E_SHAPE, "cholesky: empty matrix");
  cudaStream_t st = bt_stream(stream);
  int64_t* info = static_cast<int64_t*>(ws);
  double* dinv = reinterpret_cast<double*>(static_cast<char*>(ws) + 64);
  double* panel = dinv + NB * NB;
  BT_TRY(set_smem());
  BT_CUDA_CHECK(cudaMemsetAsync(info, 0, sizeof(int64_t), st));
  if (a != l) {
    copy_lower_kernel<<<148 * 4, 256, 0, st>>>(a, n, l);
    BT_LAUNCH_CHECK();
  }
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int kb = (int)((n - k0) < NB ? (n - k0) : NB);
    potrf_diag_kernel<<<1, 256, kSmem, st>>>(l, n, k0, kb, dinv, info);
    BT_LAUNCH_CHECK();
    const int64_t m2 = n - k0 - kb;
    if (m2 == 0) break;
    // panel = A21 * L11^-T : panel[i][c] = sum_j A21[i][j] dinv[c][j]
    double* a21 = l + (k0 + kb) * n + k0;
    int rc = bt_gemm_run(plain_gemm(m2, kb, kb, a21, n, 1, dinv, NB, 1, panel, NB, 1.0, 0.0), 1,
                         st, 1, 0);
    if (rc != BT_OK) return rc;
    BT_CUDA_CHECK(cudaMemcpy2DAsync(a21, n * sizeof(double), panel, NB * sizeof(double),
                                    kb * sizeof(double), m2, cudaMemcpyDeviceToDevice, st));
    // A22 -= panel panel^T  (full square; only the lower triangle is used)
    rc = bt_gemm_run(plain_gemm(m2, m2, kb, panel, NB, 1, panel, NB, 1, l + (k0 + kb) * (n + 1), n,
                                -1.0, 1.0),
                     1, st, 1, 0);
    if (rc != BT_OK) return rc;
  }
  zero_upper_kernel<<<148 * 4, 256, 0, st>>>(l, n);
  BT_LAUNCH_CHECK();
  int64_t h = 0;
  BT_CUDA_CHECK(cudaMemcpyAsync(&h, info, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  BT_CUDA_CHECK(cudaStreamSynchronize(st));
  if (bad_pivot) *bad_pivot = h;
  if (h != 0) {
    bt_set_error("%lld-th leading minor is not positive definite", (long long)h);
    return BT_E_NOT_PD;
  }
  return BT_OK;
}

extern "C" int64_t bt_tri_inv_lower_ws_bytes(int64_t n) {
  // diagonal-block inverses + one block row of the right-hand side
  return (cdiv64(n, NB) * NB * NB + (int64_t)NB * (n > 0 ? n : 0)) * 8;
}

// X = L^-1 by block rows: X_i = D_i^-1 (E_i - L_{i,<i} X_{<i}), columns < i0+bi.
extern "C" int bt_tri_inv_lower_f64(const double* l, int64_t n, double* linv, void* ws,
                                    void* stream) {
  BT_NVTX("bt_tri_inv_lower_f64");
  BT_REQUIRE(n >= 1, BT_E_SHAPE, "tri_inv: empty matrix");
  cudaStream_t st = bt_stream(stream);
  const int64_t nblk = cdiv64(n, NB);
  double* dinv = static_cast<double*>(ws);
  double* t = dinv + nblk * NB * NB;
  BT_TRY(set_smem());
  diag_inv_kernel<<<static_cast<unsigned>(nblk), 64, kSmem, st>>>(l, n, dinv);
  BT_LAUNCH_CHECK();
  BT_CUDA_CHECK(cudaMemsetAsync(linv, 0, n * n * sizeof(double), st));
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t i0 = b * NB;
    const int bi = (int)((n - i0) < NB ? (n - i0) : NB);
    const int64_t w = i0 + bi;  // nonzero columns of this block row
    identity_rows_kernel<<<static_cast<unsigned>(cdiv64(bi * w, 256)), 256, 0, st>>>(t, i0, bi, w);
    BT_LAUNCH_CHECK();
    if (i0 > 0) {
      // t -= L[i0:i0+bi, 0:i0] X[0:i0, 0:w]  (B(k, n) = X[k][n]: unit stride along n)
      int rc = bt_gemm_run(plain_gemm(bi, w, i0, l + i0 * n, n, 1, linv, 1, n, t, w, -1.0, 1.0), 1,
                           st, 1, 0);
      if (rc != BT_OK) return rc;
    }
    // X[i0:i0+bi, 0:w] = D_b^-1 t  (A(m, k) = dinv[m][k], B(k, n) = t[k][n])
    int rc = bt_gemm_run(plain_gemm(bi, w, bi, dinv + b * NB * NB, NB, 1, t, 1, w, linv + i0 * n,
                                    n, 1.0, 0.0),
                         1, st, 1, 0);
    if (rc != BT_OK) return rc;
  }
  return BT_OK;
}
