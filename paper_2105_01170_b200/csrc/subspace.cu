// K8 (leading eigenpairs of a deflation pass): block subspace iteration with
// Rayleigh-Ritz on a symmetric n x n Gram, driven from the host side of the
// library so that one iteration costs its kernels plus two small D2H reads
// (the Python loop it replaces spent more time in launch overhead than the
// GPU spent computing).  Same algorithm and acceptance rule as the reference
// restatement in _linalg.py: the leading left singular vectors that
// decomp.py:220-234 takes from LAPACK's SVD, per deflation pass.
//
//   Q0 = SVQB(Gaussian [ , warm start columns])
//   repeat:  Q = SVQB(G Q);  H = Q^T G Q;  H = S diag(theta) S^T (one-CTA
//            Jacobi);  V = Q S;  accept the leading k pairs once every
//            ||G v - theta v|| <= 32 eps theta_1
//
// SVQB is the column-scaled variant (D = diag(Y^T Y)^-1/2; eigen-decomposition
// of D Y^T Y D; drop directions below 1e3 eps of the largest; one
// Newton-Schulz step).  Status: 0 converged, 1 not converged / too slow (the
// caller falls back to bt_syevx_f64), 2 not applicable (block shape).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemm.cuh"
#include "jacobi.cuh"  // rsqrt_nr

int bt_gemm_run(BtGemmArgs g, int64_t batch, cudaStream_t st, int want_splits, int64_t ws_elems);
int bt_syevd_sweeps(const double* a, int64_t n, double* w, double* v, void* ws, int64_t ws_bytes,
                    void* stream, int max_sweeps);
int64_t bt_gemm_ws_elems(BtGemmArgs g, int64_t batch);

extern "C" {
int64_t bt_syevd_ws_bytes(int64_t n);
int bt_syevd_f64(const double* a, int64_t n, double* w, double* v, void* ws, int64_t ws_bytes,
                 void* stream);
int bt_inv_sqrt_f64(const double* x, int64_t n, double* out, void* stream);
int bt_sym_scale_f64(const double* m, int64_t b, double* dinv, double* out, void* stream);
int bt_sign_fix_f64(double* x, int64_t rows, int64_t cols, void* stream);
int bt_fill_normal_f64(double* out, int64_t n, uint64_t key, void* stream);
int bt_ritz_resid_f64(const double* gv, const double* v, const double* theta, int64_t rows,
                      int64_t cols, int64_t ld, double* out, void* stream);
}

namespace {

constexpr int SUB_OVERSAMPLE = 16;
constexpr int SUB_MAX_BLOCK = 96;
constexpr int SUB_MAX_ITERS = 10;
// a cold block of many wanted pairs (C3 mode 1: 64 of 1024) oversamples by
// half the wanted count (capped by SUB_MAX_BLOCK) and may take more
// iterations: at b = 96 it converges at lambda_97 / lambda_64 ~ 0.31 per
// iteration, ~0.2 ms each, well under the tridiagonal solver's ~15 ms
constexpr int SUB_MAX_ITERS_COLD = 32;
constexpr int RR_ROUGH_SWEEPS = 4;
// BT_RR_ROUGH=<n>: Jacobi sweeps of a cold block's first (rough) Rayleigh-Ritz (A/B switch)
static int rr_rough_sweeps() {
  static const int v = [] {
    const char* e = std::getenv("BT_RR_ROUGH");
    const int n = e ? std::atoi(e) : RR_ROUGH_SWEEPS;
    return n >= 1 ? n : RR_ROUGH_SWEEPS;
  }();
  return v;
}

// BT_SUB_SKIP_RR=0: a Rayleigh-Ritz every iteration for cold blocks too
bool no_skip_rr() {
  static const bool v = getenv("BT_SUB_SKIP_RR") && getenv("BT_SUB_SKIP_RR")[0] == '0';
  return v;
}

int64_t block_for(int64_t n, int64_t want, bool cold) {
  const int64_t over = cold ? std::max<int64_t>(SUB_OVERSAMPLE, want / 2) : SUB_OVERSAMPLE;
  return std::min(n, std::min<int64_t>(std::min<int64_t>(want, SUB_MAX_BLOCK - SUB_OVERSAMPLE) + over,
                                       SUB_MAX_BLOCK));
}
constexpr double SUB_RESID = 32.0;
constexpr double EPS = 2.220446049250313e-16;
constexpr double SVQB_DROP = 1e3 * EPS;

// out = (h + h^T) / 2  (b x b)
__global__ void sym_kernel(const double* __restrict__ h, int64_t b, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < b * b;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / b, j = e - i * b;
    out[e] = 0.5 * h[i * b + j] + 0.5 * h[j * b + i];
  }
}

// out = 1.5 I - 0.5 m  (Newton-Schulz correction, b x b)
__global__ void ns_kernel(const double* __restrict__ m, int64_t b, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < b * b;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / b, j = e - i * b;
    out[e] = 1.5 * (i == j ? 1.0 : 0.0) - 0.5 * m[e];
  }
}

// dst[r][c] = src[r][c] for c < cols  (row strides ld_dst / ld_src)
__global__ void copy_cols_kernel(const double* __restrict__ src, int64_t ld_src, int64_t rows,
                                 int64_t cols, double* __restrict__ dst, int64_t ld_dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    dst[r * ld_dst + c] = src[r * ld_src + c];
  }
}

// One-CTA Cholesky of a (column-scaled, unit-diagonal) Gram m (b <= 96) and
// the inverse of its transposed factor: rinv = L^-T, so Y D rinv has
// orthonormal columns (CholeskyQR).  status = 0 ok, 1 when a pivot falls
// below CHOL_MIN_PIVOT (cond(m) too large for one CholeskyQR + Newton-Schulz
// step: the caller takes the eigenvalue-based SVQB instead); a failure also
// sets *sticky when given (the deferred check of the power steps).
//
// Blocked right-looking, 32-column panels (m padded with identity to a
// multiple of 32): warp 0 factors the diagonal block in registers (lane =
// row, pivots and L columns by shuffle) and inverts it (lane = column of
// L11^-1, L11 rows broadcast from shared memory); all warps form
// L21 = A21 L11^-T and the trailing update.  The off-diagonal blocks of X = L^-1 follow by block
// distance: X_ij = -X_ii sum_{j <= k < i} L_ik X_kj.  Three panels and
// ~10 CTA barriers at b = 96: 54 us, where the element-wise version took one
// barrier per column and ran 131 us (the three one-warp diagonal blocks are
// most of what is left).
constexpr double CHOL_MIN_PIVOT = 1e-6;
constexpr int CHOL_MAXB = 96;
constexpr int CHOL_CB = 32;
constexpr int CHOL_THREADS = 256;

__global__ void __launch_bounds__(CHOL_THREADS)
    chol_rinv_kernel(const double* __restrict__ m, int b, double* __restrict__ rinv,
                     int* __restrict__ status, int* __restrict__ sticky) {
  constexpr int CB = CHOL_CB;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double chol_sm[];
  const int bp = (b + CB - 1) / CB * CB, P = bp / CB, ld = bp + 1;
  double* a = chol_sm;      // L (lower); upper off-diagonal blocks: scratch T
  double* x = a + bp * ld;  // X = L^-1 (lower)
  __shared__ double rdiag[CHOL_MAXB];
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  if (tid == 0) bad = 0;
  // m (b x b, in L2) -> a: eight loads in flight per thread
  for (int e0 = tid; e0 < bp * bp; e0 += 8 * nt) {
    double vv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * nt, i = e / bp, j = e - i * bp;
      vv[u] = (e < bp * bp && i < b && j < b) ? m[i * b + j] : (i == j ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * nt, i = e / bp, j = e - i * bp;
      if (e < bp * bp) {
        a[i * ld + j] = vv[u];
        x[i * ld + j] = 0.0;
      }
    }
  }
  __syncthreads();
  for (int p = 0; p < P; ++p) {
    const int o = p * CB;
    if (warp == 0) {
      // lane = row; fully unrolled (a rolled k loop with shifted registers
      // measured 1.7x slower: one warp, latency bound either way)
      double r[CB];
#pragma unroll
      for (int j = 0; j < CB; ++j) r[j] = a[(o + lane) * ld + o + j];
      bool ok = true;
      double rdg = 0.0;
#pragma unroll
      for (int k = 0; k < CB; ++k) {
        const double piv = __shfl_sync(FULL, r[k], k);
        ok = ok && (piv > CHOL_MIN_PIVOT);
        const double rk = rsqrt_nr(fmax(piv, CHOL_MIN_PIVOT));
        const double lik = (lane >= k) ? r[k] * rk : 0.0;
        if (lane == k) rdg = rk;
        r[k] = lik;
#pragma unroll
        for (int j = k + 1; j < CB; ++j) r[j] = fma(-lik, __shfl_sync(FULL, lik, j), r[j]);
      }
#pragma unroll
      for (int j = 0; j < CB; ++j) a[(o + lane) * ld + o + j] = r[j];
      rdiag[o + lane] = rdg;
      if (lane == 0 && !ok) bad = 1;
      __syncwarp();
      // column `lane` of L11^-1: x_jj = 1 / l_jj, x_ij = -(sum_{j <= k < i} l_ik x_kj) / l_ii
      // (four partial sums: the chain per row is the last term only)
      double xc[CB];
#pragma unroll
      for (int i = 0; i < CB; ++i) {
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < i - 1; ++k) s4[k & 3] = fma(a[(o + i) * ld + o + k], xc[k], s4[k & 3]);
        double s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        if (i >= 1) s = fma(a[(o + i) * ld + o + i - 1], xc[i - 1], s);
        const double ri = rdiag[o + i];
        xc[i] = (i == lane) ? ri : ((i > lane) ? -s * ri : 0.0);
      }
#pragma unroll
      for (int i = 0; i < CB; ++i) x[(o + i) * ld + o + lane] = xc[i];
    }
    __syncthreads();
    if (bad) break;
    // L21 = A21 L11^-T, a warp per row
    for (int rr = o + CB + warp; rr < bp; rr += nw) {
      const double av = a[rr * ld + o + lane];
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < CB; ++k)
        s4[k & 3] = fma(__shfl_sync(FULL, av, k), x[(o + lane) * ld + o + k], s4[k & 3]);
      a[rr * ld + o + lane] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    }
    __syncthreads();
    // trailing lower triangle: A22 -= L21 L21^T, 4 x 4 blocks per thread
    const int t0 = o + CB, nq = (bp - t0) / 4;
    for (int e = tid; e < nq * nq; e += nt) {
      const int bi = e / nq, bj = e - bi * nq;
      if (bj > bi) continue;
      const int i0 = t0 + 4 * bi, j0 = t0 + 4 * bj;
      double acc[4][4] = {};
#pragma unroll 4
      for (int k = 0; k < CB; ++k) {
        double ai[4], aj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ai[u] = a[(i0 + u) * ld + o + k];
          aj[u] = a[(j0 + u) * ld + o + k];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int w = 0; w < 4; ++w) acc[u][w] = fma(ai[u], aj[w], acc[u][w]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (j0 + w <= i0 + u) a[(i0 + u) * ld + j0 + w] -= acc[u][w];
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) {
      *status = 1;
      if (sticky != nullptr) *sticky = 1;
    }
    return;
  }
  // off-diagonal blocks of X by block distance d (4 x 4 register blocks)
  constexpr int QB = CB / 4;
  for (int d = 1; d < P; ++d) {
    const int cnt = (P - d) * QB * QB;
    for (int e = tid; e < cnt; e += nt) {
      const int i = d + e / (QB * QB), rc = e % (QB * QB), r0 = 4 * (rc / QB), c0 = 4 * (rc % QB), j = i - d;
      double acc[4][4] = {};
      for (int k = j * CB; k < i * CB; ++k) {
        double ar[4], xk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ar[u] = a[(i * CB + r0 + u) * ld + k];
          xk[u] = x[k * ld + j * CB + c0 + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int w = 0; w < 4; ++w) acc[u][w] = fma(ar[u], xk[w], acc[u][w]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) a[(j * CB + r0 + u) * ld + i * CB + c0 + w] = acc[u][w];  // T_ij in the free upper block (j, i)
    }
    __syncthreads();
    for (int e = tid; e < cnt; e += nt) {
      const int i = d + e / (QB * QB), rc = e % (QB * QB), r0 = 4 * (rc / QB), c0 = 4 * (rc % QB), j = i - d;
      double acc[4][4] = {};
      for (int t = 0; t < r0 + 4; ++t) {
        double xr[4], tk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          xr[u] = x[(i * CB + r0 + u) * ld + i * CB + t];   // zero above the diagonal
          tk[u] = a[(j * CB + t) * ld + i * CB + c0 + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int w = 0; w < 4; ++w) acc[u][w] = fma(xr[u], tk[w], acc[u][w]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) x[(i * CB + r0 + u) * ld + j * CB + c0 + w] = -acc[u][w];
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e - i * b;
    rinv[e] = (j >= i) ? x[j * ld + i] : 0.0;  // L^-T: upper triangular
  }
  if (tid == 0) *status = 0;
}

unsigned grid_for(int64_t n) { return static_cast<unsigned>(std::min<int64_t>(bt_cdiv(n, 256), 4096)); }

// C (M x N, row-major, ld N) = op(A) op(B) with explicit strides, as
// _linalg._gemm builds it
BtGemmArgs gemm_args(int64_t M, int64_t N, int64_t K, const double* A, int64_t sAm, int64_t sAk,
                     const double* B, int64_t sBk, int64_t sBn, double* C) {
  BtGemmArgs g{};
  g.M = M;
  g.N = N;
  g.Kin = K;
  g.Kout = 1;
  g.A = BtOperand{A, sAm, 0, sAk, 0};
  g.B = BtOperand{B, sBn, 0, sBk, 0};
  g.C = C;
  g.sCm = N;
  g.sCn = 1;
  g.alpha = 1.0;
  g.beta = 0.0;
  return g;
}

struct Plan {
  int64_t b, n;
  int64_t off_q, off_y, off_gq, off_gv, off_m, off_ms, off_s, off_w2, off_v2, off_dinv,
      off_sv, off_h, off_hs, off_w, off_res, off_flag, off_gws, off_ews, total;
  int64_t gemm_ws, eig_ws;
};

Plan plan(int64_t n, int64_t b) {
  Plan p{};
  p.n = n;
  p.b = b;
  int64_t o = 0;
  auto take = [&](int64_t k) {
    const int64_t at = o;
    o += (k + 1) / 2 * 2;
    return at;
  };
  p.off_q = take(n * b);
  p.off_y = take(n * b);
  p.off_gq = take(n * b);
  p.off_gv = take(n * b);
  p.off_m = take(b * b);
  p.off_ms = take(b * b);
  p.off_s = take(b * b);
  p.off_w2 = take(b);
  p.off_v2 = take(b * b);
  p.off_dinv = take(b);
  p.off_sv = take(b);
  p.off_h = take(b * b);
  p.off_hs = take(b * b);
  p.off_w = take(b);
  p.off_res = take(b);
  p.off_flag = take(2);
  // GEMM split-K partials: the largest of the shapes used below
  int64_t gw = 0;
  gw = std::max(gw, bt_gemm_ws_elems(gemm_args(n, b, n, nullptr, n, 1, nullptr, b, 1, nullptr), 1));
  gw = std::max(gw, bt_gemm_ws_elems(gemm_args(b, b, n, nullptr, 1, b, nullptr, b, 1, nullptr), 1));
  gw = std::max(gw, bt_gemm_ws_elems(gemm_args(n, b, b, nullptr, b, 1, nullptr, b, 1, nullptr), 1));
  p.gemm_ws = gw;
  p.off_gws = take(gw);
  p.eig_ws = (bt_syevd_ws_bytes(b) + 7) / 8;
  p.off_ews = take(p.eig_ws);
  p.total = o;
  return p;
}

struct Ctx {
  const Plan& p;
  double* ws;
  cudaStream_t st;
  bool cholqr;
  double* at(int64_t off) const { return ws + off; }
  int gemm(BtGemmArgs g) const {
    g.ws = ws + p.off_gws;
    return bt_gemm_run(g, 1, st, 0, p.gemm_ws);
  }
  int eig(const double* a, int64_t b, double* w, double* v, int max_sweeps = 60) const {
    return bt_syevd_sweeps(a, b, w, v, ws + p.off_ews, p.eig_ws * 8, st, max_sweeps);
  }
};

bool skip_polish() {
  static const bool on = !(getenv("BT_SUB_POLISH_ALL") && getenv("BT_SUB_POLISH_ALL")[0] == '1');
  return on;
}

// Column-scaled SVQB of y (n x b, row-major) into q (n x keep); returns keep
// (0 when y is numerically zero) through *keep and the dropped count.
int svqb(const Ctx& c, const double* y, int64_t n, int64_t b, double* q, int64_t* keep_out,
         int64_t* dropped, int* sticky = nullptr) {
  const Plan& p = c.p;
  double* m = c.at(p.off_m);
  double* ms = c.at(p.off_ms);
  double* dinv = c.at(p.off_dinv);
  double* w2 = c.at(p.off_w2);
  double* v2 = c.at(p.off_v2);
  double* sv = c.at(p.off_sv);
  BT_TRY(c.gemm(gemm_args(b, b, n, y, 1, b, y, b, 1, m)));          // Y^T Y
  BT_TRY(bt_sym_scale_f64(m, b, dinv, ms, c.st));
  double* out = c.at(p.off_gv);  // scratch n x keep (gv is free here)
  if (b <= CHOL_MAXB && c.cholqr) {
    // well-conditioned block (the usual case once Q holds Ritz vectors):
    // CholeskyQR  Q = Y D L^-T  + the Newton-Schulz polish
    int* flag = reinterpret_cast<int*>(c.at(p.off_flag));
    const int64_t bp = (b + CHOL_CB - 1) / CHOL_CB * CHOL_CB;
    const size_t smb = sizeof(double) * 2 * bp * (bp + 1);
    static bool attr = false;
    if (!attr) {
      BT_CUDA_CHECK(cudaFuncSetAttribute(chol_rinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(double) * 2 * CHOL_MAXB *
                                                          (CHOL_MAXB + 1))));
      attr = true;
    }
    chol_rinv_kernel<<<1, CHOL_THREADS, smb, c.st>>>(ms, static_cast<int>(b), v2, flag, sticky);
    BT_LAUNCH_CHECK();
    int hflag = 0;
    if (sticky == nullptr) {
      // a deferred check (sticky given) assumes success; the caller reads the
      // sticky flag once after its run of steps
      BT_CUDA_CHECK(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, c.st));
      BT_CUDA_CHECK(cudaStreamSynchronize(c.st));
    }
    if (hflag == 0) {
      // the silent power steps (sticky given) skip the Newton-Schulz polish:
      // their block is re-orthonormalised by the next step anyway, and the
      // last iteration before the Rayleigh-Ritz check polishes
      const bool polish = sticky == nullptr || !skip_polish();
      BtGemmArgs g = gemm_args(n, b, b, y, b, 1, v2, b, 1, polish ? out : q);
      g.ascale = dinv;
      BT_TRY(c.gemm(g));
      if (!polish) {
        *keep_out = b;
        return BT_OK;
      }
      BT_TRY(c.gemm(gemm_args(b, b, n, out, 1, b, out, b, 1, m)));
      ns_kernel<<<grid_for(b * b), 256, 0, c.st>>>(m, b, ms);
      BT_LAUNCH_CHECK();
      BT_TRY(c.gemm(gemm_args(n, b, b, out, b, 1, ms, b, 1, q)));
      *keep_out = b;
      return BT_OK;
    }
  }
  BT_TRY(c.eig(ms, b, w2, v2));
  std::vector<double> wh(b);
  BT_CUDA_CHECK(cudaMemcpyAsync(wh.data(), w2, sizeof(double) * b, cudaMemcpyDeviceToHost, c.st));
  BT_CUDA_CHECK(cudaStreamSynchronize(c.st));
  if (!(wh[0] > 0.0)) {
    *keep_out = 0;
    return BT_OK;
  }
  int64_t keep = 0;
  for (int64_t i = 0; i < b; ++i) keep += wh[i] > SVQB_DROP * wh[0];
  *dropped += b - keep;
  BT_TRY(bt_inv_sqrt_f64(w2, keep, sv, c.st));
  // Y D V[:, :keep] diag(s): D on A's reduction index, s on B's columns
  BtGemmArgs g = gemm_args(n, keep, b, y, b, 1, v2, b, 1, out);
  g.ascale = dinv;
  g.bscale = sv;
  BT_TRY(c.gemm(g));
  // one Newton-Schulz step: Q = out (1.5 I - 0.5 out^T out)
  BT_TRY(c.gemm(gemm_args(keep, keep, n, out, 1, keep, out, keep, 1, m)));
  ns_kernel<<<grid_for(keep * keep), 256, 0, c.st>>>(m, keep, ms);
  BT_LAUNCH_CHECK();
  BT_TRY(c.gemm(gemm_args(n, keep, keep, out, keep, 1, ms, keep, 1, q)));
  *keep_out = keep;
  return BT_OK;
}

}  // namespace

extern "C" int64_t bt_leading_subspace_ws_bytes(int64_t n, int64_t need, int64_t hint) {
  const int64_t want = hint > 0 ? std::max<int64_t>(1, std::min(need, hint)) : need;
  const int64_t b = block_for(n, want, true);   // the larger of the two block sizes
  if (b < 2 || b > SUB_MAX_BLOCK || 2 * b > n) return 0;
  return plan(n, b).total * 8;
}

extern "C" int bt_leading_subspace_f64(const double* g, int64_t n, int64_t need, double tau,
                                       const double* start, int64_t start_cols, int64_t hint,
                                       double* w, double* v, int64_t* bq_out, int64_t* k_out,
                                       int* status, void* wsv, int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_leading_subspace_f64");
  *status = 2;
  *bq_out = 0;
  *k_out = 0;
  const int64_t want = hint > 0 ? std::max<int64_t>(1, std::min(need, hint)) : need;
  const bool cold = start == nullptr || start_cols <= 0;
  const int64_t b = block_for(n, want, cold && hint <= 0);
  if (b < 2 || b > SUB_MAX_BLOCK || 2 * b > n) return BT_OK;
  const int max_iters = (cold && hint <= 0 && want >= 48) ? SUB_MAX_ITERS_COLD : SUB_MAX_ITERS;
  const Plan p = plan(n, b);
  BT_REQUIRE(ws_bytes >= p.total * 8, BT_E_VALUE, "leading_subspace: workspace too small");
  static const bool no_chol = getenv("BT_SUB_CHOLQR") && getenv("BT_SUB_CHOLQR")[0] == '0';
  const Ctx c{p, static_cast<double*>(wsv), bt_stream(stream), !no_chol};
  const bool dbg = getenv("BT_BASIS_DEBUG") != nullptr;
  double* q = c.at(p.off_q);
  double* y = c.at(p.off_y);
  double* gq = c.at(p.off_gq);
  double* h = c.at(p.off_h);
  double* hs = c.at(p.off_hs);
  double* sm = c.at(p.off_s);
  double* res = c.at(p.off_res);
  *status = 1;
  // Gaussian start block (Philox key as _linalg.gaussian_dev), warm columns in front
  BT_TRY(bt_fill_normal_f64(y, n * b, static_cast<uint64_t>(20210501 + n), c.st));
  if (start != nullptr && start_cols > 0) {
    const int64_t ks = std::min<int64_t>(start_cols, b - SUB_OVERSAMPLE);
    if (ks > 0) {
      copy_cols_kernel<<<grid_for(n * ks), 256, 0, c.st>>>(start, start_cols, n, ks, y, b);
      BT_LAUNCH_CHECK();
    }
  }
  int64_t bq = 0, dropped = 0;
  BT_TRY(svqb(c, y, n, b, q, &bq, &dropped));
  if (bq == 0) return BT_OK;
  double prev = -1.0;
  int steps_since_rr = 1;
  // silent power steps between Rayleigh-Ritz checks: for the cold many-pair
  // block (C3 mode 1) and, since C2's deflation passes spent 8 full
  // Rayleigh-Ritz iterations of ~300 us on a block that converges 10x per
  // 18 us G product, for every cold block (BT_SUB_SKIP_RR_ALL=0: only the former)
  static const bool skip_all = !(getenv("BT_SUB_SKIP_RR_ALL") && getenv("BT_SUB_SKIP_RR_ALL")[0] == '0');
  const bool skip_rr = (max_iters == SUB_MAX_ITERS_COLD || (cold && skip_all)) && !no_skip_rr();
  std::vector<double> wh(b), rh(b);
  for (int it = 0; it < max_iters; ++it) {
    BT_TRY(c.gemm(gemm_args(n, bq, n, g, n, 1, q, bq, 1, y)));       // G Q
    dropped = 0;
    int64_t nq = 0;
    BT_TRY(svqb(c, y, n, bq, q, &nq, &dropped));
    if (nq == 0) return BT_OK;
    bq = nq;
    BT_TRY(c.gemm(gemm_args(n, bq, n, g, n, 1, q, bq, 1, gq)));      // G Q
    BT_TRY(c.gemm(gemm_args(bq, bq, n, q, 1, bq, gq, bq, 1, h)));    // Q^T G Q
    sym_kernel<<<grid_for(bq * bq), 256, 0, c.st>>>(h, bq, hs);
    BT_LAUNCH_CHECK();
    // the first Rayleigh-Ritz of a cold many-pair block only orients the
    // block and estimates the rate: a few Jacobi sweeps (its pairs are never
    // accepted, see below)
    const bool rough = skip_rr && it == 0 && start == nullptr;
    BT_TRY(c.eig(hs, bq, w, sm, rough ? rr_rough_sweeps() : 60));       // descending
    BT_TRY(c.gemm(gemm_args(n, bq, bq, q, bq, 1, sm, bq, 1, v)));    // V = Q S
    double* gv = c.at(p.off_gv);
    BT_TRY(c.gemm(gemm_args(n, bq, bq, gq, bq, 1, sm, bq, 1, gv)));  // G V = (G Q) S
    BT_TRY(bt_ritz_resid_f64(gv, v, w, n, bq, bq, res, c.st));
    BT_CUDA_CHECK(cudaMemcpyAsync(wh.data(), w, sizeof(double) * bq, cudaMemcpyDeviceToHost, c.st));
    BT_CUDA_CHECK(cudaMemcpyAsync(rh.data(), res, sizeof(double) * bq, cudaMemcpyDeviceToHost, c.st));
    BT_CUDA_CHECK(cudaStreamSynchronize(c.st));
    const double top = wh[0];
    if (!(top > 0.0)) return BT_OK;
    // accept at most b - 16 pairs, and never the whole retained block unless
    // SVQB dropped directions (those sit below ~sqrt(1e3 eps) of the top)
    const int64_t lim = std::min<int64_t>(std::min<int64_t>(need, b - SUB_OVERSAMPLE),
                                          dropped ? bq : bq - 1);
    int64_t k = 0;
    for (int64_t i = 0; i < lim; ++i) k += wh[i] > tau * top;
    double worst = 0.0;
    for (int64_t i = 0; i < std::max<int64_t>(k, 1); ++i) worst = std::max(worst, rh[i]);
    const double target = SUB_RESID * EPS * top;
    if (dbg)
      fprintf(stderr, "[subspace n=%lld b=%lld] it %d: k %lld max resid/theta1 %.2e\n",
              (long long)n, (long long)b, it, (long long)k, worst / top);
    if (worst <= target && !rough) {
      BT_TRY(bt_sign_fix_f64(v, n, bq, c.st));
      *bq_out = bq;
      *k_out = k;
      *status = 0;
      return BT_OK;
    }
    if (prev < 0.0 && start == nullptr && dropped == 0 && k >= 1 && worst > 0.0 &&
        wh[bq - 1] > 0.0) {
      // cold start: the residual of pair k falls roughly like
      // (lambda_{b+1} / lambda_k)^it with the last Ritz value standing in for
      // lambda_{b+1}; a slowly decaying block edge goes straight to the
      // tridiagonal solver
      const double rate0 = wh[bq - 1] / wh[k - 1];
      if (rate0 >= 1.0 ||
          std::log(target / worst) / std::log(std::max(rate0, 1e-300)) > 1.5 * (max_iters - 1))
        return BT_OK;
    }
    if (prev > 0.0 && worst > 0.0) {
      // linear convergence factor per step (several steps since the last RR
      // when Rayleigh-Ritz is skipped)
      const double rate = std::pow(worst / prev, 1.0 / static_cast<double>(steps_since_rr));
      const int left = max_iters - 1 - it;
      if (rate >= 1.0 || std::log(target / worst) / std::log(std::max(rate, 1e-300)) > left)
        return BT_OK;  // too slow: the tridiagonal path wins
    }
    // next block = the Ritz vectors (v stays the caller's output buffer)
    BT_CUDA_CHECK(cudaMemcpyAsync(q, v, sizeof(double) * n * bq, cudaMemcpyDeviceToDevice, c.st));
    if (skip_rr && worst > 0.0 && k >= 1) {
      // cold block of many pairs: plain simultaneous iteration (G Q, then
      // CholeskyQR -- Q's columns stay near the eigenvectors, so the
      // column-scaled Gram stays well conditioned) for the predicted number
      // of steps, and the Rayleigh-Ritz + residual check only after them
      // before any measured rate: sqrt(theta_b / theta_k) -- the Ritz ratio
      // itself overestimates the speed (C3 mode 1: 0.155 vs 0.31 measured)
      double rate = std::sqrt(wh[bq - 1] / wh[k - 1]);
      if (prev > 0.0) rate = std::pow(worst / prev, 1.0 / static_cast<double>(steps_since_rr));
      int m = 0;
      if (rate > 0.0 && rate < 1.0)
        m = static_cast<int>(std::ceil(std::log(target / worst) / std::log(rate))) - 1;
      m = std::max(0, std::min(m, max_iters - 2 - it));
      // two applications of G per orthonormalisation (Q's columns are near
      // eigenvectors, so the column-scaled G^2 Q stays well conditioned)
      double* gq2 = c.at(p.off_gq);
      // CholeskyQR failures are checked once after the run (sticky flag)
      int* sticky = reinterpret_cast<int*>(c.at(p.off_flag)) + 1;
      BT_CUDA_CHECK(cudaMemsetAsync(sticky, 0, sizeof(int), c.st));
      for (int j = 0; j < m; j += 2) {
        const bool two = j + 1 < m;
        BT_TRY(c.gemm(gemm_args(n, bq, n, g, n, 1, q, bq, 1, two ? gq2 : y)));   // G Q
        if (two) BT_TRY(c.gemm(gemm_args(n, bq, n, g, n, 1, gq2, bq, 1, y)));   // G (G Q)
        int64_t nq = 0, dr = 0;
        BT_TRY(svqb(c, y, n, bq, q, &nq, &dr, sticky));
        if (nq != bq) return BT_OK;  // the block lost directions: let the caller fall back
      }
      if (m > 0) {
        int hs = 0;
        BT_CUDA_CHECK(cudaMemcpyAsync(&hs, sticky, sizeof(int), cudaMemcpyDeviceToHost, c.st));
        BT_CUDA_CHECK(cudaStreamSynchronize(c.st));
        if (hs != 0) return BT_OK;  // a step lost conditioning: the caller falls back
      }
      it += m;
      steps_since_rr = m + 1;
      if (dbg)
        fprintf(stderr, "[subspace n=%lld b=%lld] %d power steps without Rayleigh-Ritz (rate %.3f)\n",
                (long long)n, (long long)b, m, rate);
    }
    prev = worst;
  }
  return BT_OK;
}

// ---------------------------------------------------------------------------
// Orthonormal completion of a basis (decomp.py:220-234 full_matrices branch
// and the deflation's rounding-level remainder): `need` columns orthogonal to
// basis (n x k) from a Philox Gaussian block, in blocks of <= 32 columns:
// project out the basis and the columns already made (twice), then
// column-scaled CholeskyQR2 with the one-warp Cholesky -- all on the stream,
// one host read of the failure flags at the end (status 1: a block was
// rejected and the caller takes its own path).
// ---------------------------------------------------------------------------

extern "C" int bt_chol_small_f64(const double* g, int64_t n, double* lt, double* linvt, int* flag,
                                 void* stream);
extern "C" int bt_sign_fix_f64(double* x, int64_t rows, int64_t cols, void* stream);

namespace {

// gs = D g D with D = diag(g_ii^-1/2) (b x b); d out
__global__ void scale_gram_kernel(const double* __restrict__ g, int b, double* __restrict__ gs,
                                  double* __restrict__ d) {
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e / b, j = e % b;
    const double di = rsqrt(g[i * b + i]), dj = rsqrt(g[j * b + j]);
    gs[e] = g[e] * di * dj;
    if (i == j) d[i] = di;
  }
}

// m = diag(d) linvt  (b x b)
__global__ void scale_rows_kernel(const double* __restrict__ linvt, const double* __restrict__ d, int b,
                                  double* __restrict__ m) {
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) m[e] = d[e / b] * linvt[e];
}

}  // namespace

// columns per completion block: the one-CTA blocked CholeskyQR factor
// (chol_rinv_kernel, 54 us at 96 columns) instead of 32-column blocks on the
// one-warp Cholesky (37 us each, three times as many projections)
constexpr int64_t COMP_BS = CHOL_MAXB;
constexpr int COMP_PASSES = 2;   // projection passes per block (twice is enough: one pass leaves ~eps of the
                                 // block along the basis, which the ERA rank test at n eps sigma_1 sees)

extern "C" int64_t bt_complete_basis_ws_bytes(int64_t n, int64_t k, int64_t need) {
  const int64_t rows = k + need, B = COMP_BS;
  BtGemmArgs g1 = gemm_args(rows, B, n, nullptr, 1, rows, nullptr, B, 1, nullptr);
  BtGemmArgs g2 = gemm_args(n, B, rows, nullptr, rows, 1, nullptr, B, 1, nullptr);
  BtGemmArgs g3 = gemm_args(B, B, n, nullptr, 1, B, nullptr, B, 1, nullptr);
  const int64_t gw = std::max(bt_gemm_ws_elems(g1, 1), std::max(bt_gemm_ws_elems(g2, 1),
                                                                 bt_gemm_ws_elems(g3, 1)));
  return (2 * n * B + rows * B + 4 * B * B + B + 64 + gw + 64) * 8;
}

extern "C" int bt_complete_basis_f64(const double* basis, int64_t n, int64_t k, int64_t need,
                                     uint64_t key, double* out, int* status, void* wsv,
                                     int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_complete_basis_f64");
  *status = 1;
  BT_REQUIRE(n >= 1 && k >= 0 && need >= 1 && k + need <= n, BT_E_SHAPE,
             "complete_basis: %lld + %lld columns exceed %lld rows", (long long)k, (long long)need,
             (long long)n);
  BT_REQUIRE(ws_bytes >= bt_complete_basis_ws_bytes(n, k, need), BT_E_VALUE,
             "complete_basis: workspace too small");
  cudaStream_t st = bt_stream(stream);
  const int64_t B = COMP_BS;
  double* w = static_cast<double*>(wsv);
  double* t0 = w;                 // n x B working block
  double* t1 = t0 + n * B;        // n x B
  double* cproj = t1 + n * B;     // (k + need) x B
  double* gm = cproj + (k + need) * B;
  double* gs = gm + B * B;
  double* rinv = gs + B * B;
  double* mm = rinv + B * B;
  double* dv = mm + B * B;
  int* flags = reinterpret_cast<int*>(dv + B);
  double* gws = dv + B + 64;
  const int64_t gw_elems = ws_bytes / 8 - (gws - w);
  auto run = [&](BtGemmArgs g) {
    g.ws = gws;
    return bt_gemm_run(g, 1, st, 0, gw_elems);
  };
  const int64_t nblk = (need + B - 1) / B;
  BT_REQUIRE(2 * nblk <= 64, BT_E_SHAPE, "complete_basis: %lld columns exceed %lld", (long long)need,
             (long long)(32 * B));
  BT_CUDA_CHECK(cudaFuncSetAttribute(chol_rinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sizeof(double) * 2 * CHOL_MAXB * (CHOL_MAXB + 1))));
  BT_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(int) * 2 * nblk, st));
  BT_TRY(bt_fill_normal_f64(out, n * need, key, st));
  for (int64_t j0 = 0; j0 < need; j0 += B) {
    const int64_t b = std::min<int64_t>(B, need - j0);
    // working copy of the block
    copy_cols_kernel<<<grid_for(n * b), 256, 0, st>>>(out + j0, need, n, b, t0, b);
    BT_LAUNCH_CHECK();
    for (int pass = 0; pass < COMP_PASSES; ++pass) {
      // against the input basis, then the completed columns 0 .. j0
      const double* qs[2] = {basis, out};
      const int64_t qk[2] = {k, j0};
      const int64_t qld[2] = {k, need};
      for (int p = 0; p < 2; ++p) {
        if (qk[p] == 0) continue;
        BT_TRY(run(gemm_args(qk[p], b, n, qs[p], 1, qld[p], t0, b, 1, cproj)));   // Q^T T
        BtGemmArgs up = gemm_args(n, b, qk[p], qs[p], qld[p], 1, cproj, b, 1, t0); // T -= Q C
        up.alpha = -1.0;
        up.beta = 1.0;
        BT_TRY(run(up));
      }
    }
    // column-scaled CholeskyQR2: T <- T D L^-T, twice
    const int64_t bp = (b + CHOL_CB - 1) / CHOL_CB * CHOL_CB;
    const size_t smb = sizeof(double) * 2 * bp * (bp + 1);
    for (int it = 0; it < 2; ++it) {
      BT_TRY(run(gemm_args(b, b, n, t0, 1, b, t0, b, 1, gm)));                    // T^T T
      scale_gram_kernel<<<1, 1024, 0, st>>>(gm, static_cast<int>(b), gs, dv);
      BT_LAUNCH_CHECK();
      chol_rinv_kernel<<<1, CHOL_THREADS, smb, st>>>(gs, static_cast<int>(b), rinv,
                                                     flags + 2 * (j0 / B) + it, nullptr);
      BT_LAUNCH_CHECK();
      scale_rows_kernel<<<1, 1024, 0, st>>>(rinv, dv, static_cast<int>(b), mm);
      BT_LAUNCH_CHECK();
      BT_TRY(run(gemm_args(n, b, b, t0, b, 1, mm, b, 1, t1)));                    // T D L^-T
      std::swap(t0, t1);
    }
    copy_cols_kernel<<<grid_for(n * b), 256, 0, st>>>(t0, b, n, b, out + j0, need);
    BT_LAUNCH_CHECK();
  }
  BT_TRY(bt_sign_fix_f64(out, n, need, st));
  std::vector<int> hf(2 * nblk);
  BT_CUDA_CHECK(cudaMemcpyAsync(hf.data(), flags, sizeof(int) * 2 * nblk, cudaMemcpyDeviceToHost, st));
  BT_CUDA_CHECK(cudaStreamSynchronize(st));
  int bad = 0;
  for (int f : hf) bad |= f;
  *status = bad ? 1 : 0;
  return BT_OK;
}
