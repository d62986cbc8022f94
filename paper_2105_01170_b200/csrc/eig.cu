// K8: FP64 symmetric eigensolver for the unfolding Grams (replaces the
// LAPACK SVD of decomp.py:172/227 in _mode_basis / svd_truncated).
//
//   n <= 96 : one CTA, cyclic Jacobi fully in shared memory.
//   n  > 96 : block Jacobi.  The matrix is padded to a multiple of 64 with a
//             decoupled diagonal strictly below the spectrum; per round the
//             n/64 disjoint block pairs (32-wide blocks, circle-method
//             ordering) are diagonalised on chip (64x64 Jacobi in smem) and
//             the resulting 64x64 rotations are applied as A <- J^T A J and
//             V <- V J by DMMA tile GEMMs (each 64x64 tile is updated in place
//             from its own entries only, so the update needs no copy).
// Output: eigenvalues descending; eigenvectors as columns, each flipped so
// its largest-|.| entry (first on ties) is positive (decomp.py:176-179).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "jacobi.cuh"

extern "C" int bt_sumsq_f64(const double* x, int64_t n, double* out, void* ws, int64_t ws_bytes,
                            void* stream);
int64_t bt_sumsq_ws_bytes_const();

namespace {

constexpr int EB = 32;       // Jacobi block width
constexpr int EP = 2 * EB;   // pair width (subproblem size)
constexpr int ELD = 68;      // smem leading dim, == 4 (mod 16)
constexpr int SMALL_N = 96;
constexpr double ABS_TOL = 1e-15;  // rotate only |a_pq| > ABS_TOL * ||A||_F (~4.5 eps: noise floor)
constexpr int OFFN_BLOCKS = 296;
constexpr int INNER_SWEEPS = 2;  // Jacobi sweeps per 64x64 pair subproblem and round

// ---------------------------------------------------------------------------
// small path
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(1024)
    syevd_small_kernel(const double* __restrict__ a, int n, const double* __restrict__ sumsq,
                       double* __restrict__ dout, double* __restrict__ qout, int np, int max_sweeps) {
  extern __shared__ __align__(16) double sm[];
  const int ld = np + 1;
  double* s = sm;
  double* q = s + np * ld;
  double* cs = q + np * ld;
  double* sn = cs + np / 2;
  int* pp = reinterpret_cast<int*>(sn + np / 2);
  int* qq = pp + np / 2;
  const double nrm = sqrt(*sumsq);
  const double pad = -1.0 - 2.0 * nrm;
  for (int idx = threadIdx.x; idx < np * np; idx += blockDim.x) {
    const int r = idx / np, c = idx % np;
    s[r * ld + c] = (r < n && c < n) ? a[r * n + c] : (r == c ? pad : 0.0);
  }
  __syncthreads();
  jacobi_fast(s, q, np, ld, cs, sn, pp, qq, max_sweeps, ABS_TOL * nrm, 1e-15);
  __syncthreads();
  for (int i = threadIdx.x; i < np; i += blockDim.x) dout[i] = s[i * ld + i];
  for (int idx = threadIdx.x; idx < np * np; idx += blockDim.x)
    qout[idx] = q[(idx / np) * ld + idx % np];
}

// ---------------------------------------------------------------------------
// block path
// ---------------------------------------------------------------------------

__global__ void pad_kernel(const double* __restrict__ a, int64_t n, int64_t np,
                           const double* __restrict__ sumsq, double* __restrict__ ap,
                           double* __restrict__ v) {
  const double pad = -1.0 - 2.0 * sqrt(*sumsq);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < np * np;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / np, c = idx % np;
    ap[idx] = (r < n && c < n) ? a[r * n + c] : (r == c ? pad : 0.0);
    v[idx] = (r == c) ? 1.0 : 0.0;
  }
}

__device__ __forceinline__ int64_t pair_index(int nb, int rnd, int k, int l) {
  int P, Q;
  rr_pair(nb, rnd, k, P, Q);
  return (l < EB) ? static_cast<int64_t>(P) * EB + l : static_cast<int64_t>(Q) * EB + (l - EB);
}

// One (or a few) cyclic sweeps of two-sided Jacobi on the 64x64 pair
// subproblem, specialised for n = 64 and 8 warps: every warp computes all 32
// rotations of a round redundantly (lane = pair), so only two barriers per
// round remain (after the row update, after the column + Q update).
constexpr int SLD = EP + 1;  // 65: conflict-light row/column access

__device__ __forceinline__ void pair_of(int rnd, int k, int& p, int& q) {
  const int m = EP - 1;
  if (k == 0) {
    p = rnd;
    q = m;
  } else {
    p = (rnd + k) % m;
    q = (rnd - k + m) % m;
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

__global__ void __launch_bounds__(256)
    solve_pairs_kernel(const double* __restrict__ ap, int64_t np, int nb, int rnd,
                       const double* __restrict__ sumsq, double* __restrict__ jout,
                       int* __restrict__ flag, int inner_sweeps) {
  extern __shared__ __align__(16) double sm[];
  double* s = sm;
  double* q = sm + EP * SLD;
  __shared__ int rot_any;
  const int k = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int idx = threadIdx.x; idx < EP * EP; idx += blockDim.x) {
    const int r = idx / EP, c = idx % EP;
    s[r * SLD + c] = ap[pair_index(nb, rnd, k, r) * np + pair_index(nb, rnd, k, c)];
    q[r * SLD + c] = (r == c) ? 1.0 : 0.0;
  }
  if (threadIdx.x == 0) rot_any = 0;
  __syncthreads();
  const double abs_tol = ABS_TOL * sqrt(*sumsq);
  int any = 0;
  for (int sweep = 0; sweep < inner_sweeps; ++sweep) {
    for (int r = 0; r < EP - 1; ++r) {
      int p, qq;
      pair_of(r, lane, p, qq);
      const double apq = s[p * SLD + qq], app = s[p * SLD + p], aqq = s[qq * SLD + qq];
      double c = 1.0, sn = 0.0;
      if (apq != 0.0 && fabs(apq) > abs_tol && fabs(apq) > 1e-15 * sqrt(fabs(app) * fabs(aqq))) {
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        c = 1.0 / sqrt(t * t + 1.0);
        sn = t * c;
        any = 1;
      }
      // rows p, q: warp w owns columns [8w, 8w + 8)
      if (sn != 0.0) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = warp * 8 + jj;
          const double x = s[p * SLD + j], y = s[qq * SLD + j];
          s[p * SLD + j] = c * x - sn * y;
          s[qq * SLD + j] = sn * x + c * y;
        }
      }
      __syncthreads();
      // columns p, q of s and q: warp w owns rows [8w, 8w + 8)
      if (sn != 0.0) {
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) {
          const int i = warp * 8 + ii;
          double x = s[i * SLD + p], y = s[i * SLD + qq];
          s[i * SLD + p] = c * x - sn * y;
          s[i * SLD + qq] = sn * x + c * y;
          x = q[i * SLD + p];
          y = q[i * SLD + qq];
          q[i * SLD + p] = c * x - sn * y;
          q[i * SLD + qq] = sn * x + c * y;
        }
      }
      __syncthreads();
    }
  }
  if (any) rot_any = 1;  // benign race: every writer stores 1
  __syncthreads();
  const int rot = rot_any;
  double* j = jout + static_cast<int64_t>(k) * EP * EP;
  for (int idx = threadIdx.x; idx < EP * EP; idx += blockDim.x)
    j[idx] = q[(idx / EP) * SLD + idx % EP];
  if (threadIdx.x == 0) {
    jout[(int64_t)(nb / 2) * EP * EP + k] = rot ? 1.0 : 0.0;  // per-pair "rotated" mark
    if (rot) *flag = 1;
  }
}

// C(64x64) = op(X) * Y with X, Y, in smem (ld ELD); 8 warps of 16x32 each.
// xt: op(X)[m][k] = X[k][m] (transposed read) else X[m][k].
__device__ __forceinline__ void tile_gemm64(const double* X, bool xt, const double* Y,
                                            double (&acc)[2][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int m0 = (warp & 3) * 16, n0 = (warp >> 2) * 32;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < EP; kk += 4) {
    double a[2], b[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int m = m0 + i * 8 + gq;
      a[i] = xt ? X[(kk + tq) * ELD + m] : X[m * ELD + kk + tq];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = Y[(kk + tq) * ELD + n0 + j * 8 + gq];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
}

// tiles [0, P^2): A[I_p, I_q] <- J_p^T A[I_p, I_q] J_q ; tiles beyond: V[rows, I_q] <- V J_q
__global__ void __launch_bounds__(256)
    apply_pairs_kernel(double* __restrict__ ap, double* __restrict__ v, int64_t np, int nb,
                       int rnd, const double* __restrict__ jin) {
  extern __shared__ __align__(16) double sm[];
  double* Jp = sm;
  double* Jq = Jp + EP * ELD;
  double* T = Jq + EP * ELD;
  const int P = nb / 2;
  const int64_t t = blockIdx.x;
  const double* mark = jin + (int64_t)P * EP * EP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int m0 = (warp & 3) * 16, n0 = (warp >> 2) * 32;
  double acc[2][4][2];
  if (t < (int64_t)P * P) {
    const int p = static_cast<int>(t / P), q = static_cast<int>(t % P);
    if (mark[p] == 0.0 && mark[q] == 0.0) return;  // both rotations are the identity
    for (int idx = threadIdx.x; idx < EP * EP; idx += blockDim.x) {
      const int r = idx / EP, c = idx % EP;
      Jp[r * ELD + c] = jin[(int64_t)p * EP * EP + idx];
      Jq[r * ELD + c] = jin[(int64_t)q * EP * EP + idx];
      T[r * ELD + c] = ap[pair_index(nb, rnd, p, r) * np + pair_index(nb, rnd, q, c)];
    }
    __syncthreads();
    tile_gemm64(Jp, true, T, acc);  // J_p^T A
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = m0 + i * 8 + gq, n = n0 + j * 8 + 2 * tq;
        T[m * ELD + n] = acc[i][j][0];
        T[m * ELD + n + 1] = acc[i][j][1];
      }
    __syncthreads();
    tile_gemm64(T, false, Jq, acc);  // (J_p^T A) J_q
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = m0 + i * 8 + gq, n = n0 + j * 8 + 2 * tq;
        const int64_t gr = pair_index(nb, rnd, p, m);
        ap[gr * np + pair_index(nb, rnd, q, n)] = acc[i][j][0];
        ap[gr * np + pair_index(nb, rnd, q, n + 1)] = acc[i][j][1];
      }
  } else {
    const int64_t u = t - (int64_t)P * P;
    const int64_t rb = u / P;
    const int q = static_cast<int>(u % P);
    if (mark[q] == 0.0) return;
    for (int idx = threadIdx.x; idx < EP * EP; idx += blockDim.x) {
      const int r = idx / EP, c = idx % EP;
      Jq[r * ELD + c] = jin[(int64_t)q * EP * EP + idx];
      T[r * ELD + c] = v[(rb * EP + r) * np + pair_index(nb, rnd, q, c)];
    }
    __syncthreads();
    tile_gemm64(T, false, Jq, acc);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = m0 + i * 8 + gq, n = n0 + j * 8 + 2 * tq;
        double* row = v + (rb * EP + m) * np;
        row[pair_index(nb, rnd, q, n)] = acc[i][j][0];
        row[pair_index(nb, rnd, q, n + 1)] = acc[i][j][1];
      }
  }
}

// sum of squares of the off-diagonal entries (fixed-order two-level tree)
__global__ void __launch_bounds__(256)
    offnorm_partial(const double* __restrict__ ap, int64_t np, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < np * np;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double v = ap[idx];
    if (idx / np != idx % np) s = fma(v, v, s);
  }
  __shared__ double red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void offnorm_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += part[i];
    *out = t;
  }
}

__global__ void diag_kernel(const double* __restrict__ ap, int64_t np, double* __restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = ap[i * np + i];
}

// ---------------------------------------------------------------------------
// sort (descending, stable by index) + sign rule + output
// ---------------------------------------------------------------------------

__global__ void rank_kernel(const double* __restrict__ d, int64_t np, int64_t* __restrict__ perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double di = d[i];
    int64_t rk = 0;
    for (int64_t j = 0; j < np; ++j) {
      const double dj = d[j];
      rk += (dj > di) || (dj == di && j < i);
    }
    perm[rk] = i;
  }
}

__global__ void __launch_bounds__(256)
    output_kernel(const double* __restrict__ d, const double* __restrict__ q, int64_t np,
                  int64_t n, const int64_t* __restrict__ perm, double* __restrict__ w,
                  double* __restrict__ vout) {
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  for (int64_t c = blockIdx.x; c < n; c += gridDim.x) {
    const int64_t src = perm[c];
    double best = -1.0;
    int64_t bidx = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double x = fabs(q[i * np + src]);
      if (x > best) {
        best = x;
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
    const double lead = q[bi[0] * np + src];
    const double sgn = (lead < 0.0) ? -1.0 : 1.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) vout[i * n + c] = sgn * q[i * np + src];
    if (threadIdx.x == 0) w[c] = d[src];
    __syncthreads();
  }
}

size_t small_smem(int np) { return (size_t)(2 * np * (np + 1) + np) * 8 + (size_t)np * 4; }
size_t pair_smem() { return (size_t)(2 * EP * (EP + 1) + EP) * 8 + (size_t)EP * 4; }
size_t apply_smem() { return (size_t)3 * EP * ELD * 8; }

struct EigPlan {
  int64_t n, np;
  bool small;
  int64_t off_ap, off_v, off_d, off_perm, off_j, off_ss, off_sumws, off_flag, off_offn, total;
};

EigPlan eig_plan(int64_t n) {
  EigPlan p;
  p.n = n;
  // BT_EIG_SMALL_N=<n> (<= 96): sizes above n take the multi-CTA block-Jacobi path (A/B switch)
  static const int small_n = [] {
    const char* e = getenv("BT_EIG_SMALL_N");
    const int v = e ? atoi(e) : SMALL_N;
    return (v >= 2 && v <= SMALL_N) ? v : SMALL_N;
  }();
  p.small = n <= small_n;
  p.np = p.small ? n + (n & 1) : bt_cdiv(n, EP) * EP;
  int64_t o = 0;
  auto take = [&](int64_t k) {
    int64_t at = o;
    o += (k + 1) / 2 * 2;
    return at;
  };
  p.off_ap = take(p.small ? 0 : p.np * p.np);
  p.off_v = take(p.np * p.np);
  p.off_d = take(p.np);
  p.off_perm = take(p.np);
  const int64_t pairs = p.np / EP;
  p.off_j = take(p.small ? 0 : pairs * EP * EP + pairs + 2);
  p.off_ss = take(2);
  p.off_sumws = take(bt_sumsq_ws_bytes_const());
  p.off_flag = take(2);
  p.off_offn = take(OFFN_BLOCKS + 2);
  p.total = o;
  return p;
}

}  // namespace

extern "C" int64_t bt_syevd_ws_bytes(int64_t n) { return eig_plan(n).total * 8; }

// max_sweeps caps the one-CTA Jacobi (n <= 96; 60 = run to convergence): a
// truncated solve still returns an orthogonal V and the Rayleigh quotients of
// its columns, which is all a first Rayleigh-Ritz of a subspace iteration
// needs (subspace.cu)
int bt_syevd_sweeps(const double* a, int64_t n, double* w, double* v, void* wsv, int64_t ws_bytes,
                    void* stream, int max_sweeps);

extern "C" int bt_syevd_f64(const double* a, int64_t n, double* w, double* v, void* wsv,
                            int64_t ws_bytes, void* stream) {
  return bt_syevd_sweeps(a, n, w, v, wsv, ws_bytes, stream, 60);
}

int bt_syevd_sweeps(const double* a, int64_t n, double* w, double* v, void* wsv, int64_t ws_bytes,
                    void* stream, int max_sweeps) {
  BT_NVTX("bt_syevd_f64");
  BT_REQUIRE(n >= 1, BT_E_SHAPE, "syevd: empty matrix");
  cudaStream_t st = bt_stream(stream);
  EigPlan p = eig_plan(n);
  BT_REQUIRE(ws_bytes >= p.total * 8, BT_E_VALUE, "syevd: workspace too small");
  double* ws = static_cast<double*>(wsv);
  double* ss = ws + p.off_ss;
  BT_TRY(bt_sumsq_f64(a, n * n, ss, ws + p.off_sumws, bt_sumsq_ws_bytes_const() * 8, st));
  double* q = ws + p.off_v;
  double* d = ws + p.off_d;
  if (p.small) {
    const size_t sm = small_smem(static_cast<int>(p.np));
    static bool attr = false;
    if (!attr) {
      BT_CUDA_CHECK(cudaFuncSetAttribute(syevd_small_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(small_smem(SMALL_N))));
      attr = true;
    }
    syevd_small_kernel<<<1, 1024, sm, st>>>(a, static_cast<int>(n), ss, d, q,
                                           static_cast<int>(p.np), max_sweeps);
    BT_LAUNCH_CHECK();
  } else {
    static bool attr = false;
    if (!attr) {
      BT_CUDA_CHECK(cudaFuncSetAttribute(solve_pairs_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         2 * EP * SLD * 8));
      BT_CUDA_CHECK(cudaFuncSetAttribute(apply_pairs_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(apply_smem())));
      attr = true;
    }
    double* ap = ws + p.off_ap;
    double* jb = ws + p.off_j;
    int* flag = reinterpret_cast<int*>(ws + p.off_flag);
    pad_kernel<<<static_cast<unsigned>(std::min<int64_t>(bt_cdiv(p.np * p.np, 256), 8192)), 256,
                 0, st>>>(a, n, p.np, ss, ap, q);
    BT_LAUNCH_CHECK();
    const int nb = static_cast<int>(p.np / EB);
    const int pairs = nb / 2;
    const int64_t tiles = (int64_t)pairs * pairs + (p.np / EP) * pairs;
    // Convergence: the rotation threshold is far below the rounding noise the
    // tile GEMMs inject (~eps ||A||), so the sweep loop stops on the
    // off-diagonal norm: below ~eps*sqrt(n)*||A||_F, or stagnating at the
    // noise floor once it is below 1e-10 ||A||_F.
    double* offn = ws + p.off_offn;
    double h2[2] = {0.0, 0.0};
    BT_CUDA_CHECK(cudaMemcpyAsync(&h2[0], ss, sizeof(double), cudaMemcpyDeviceToHost, st));
    BT_CUDA_CHECK(cudaStreamSynchronize(st));
    const double normf = sqrt(h2[0]);
    bool done = false;
    double prev = INFINITY;
    for (int sweep = 0; sweep < 40 && !done; ++sweep) {
      BT_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int), st));
      for (int rnd = 0; rnd < nb - 1; ++rnd) {
        solve_pairs_kernel<<<pairs, 256, 2 * EP * SLD * 8, st>>>(ap, p.np, nb, rnd, ss, jb, flag,
                                                                  INNER_SWEEPS);
        BT_LAUNCH_CHECK();
        apply_pairs_kernel<<<static_cast<unsigned>(tiles), 256, apply_smem(), st>>>(ap, q, p.np,
                                                                                    nb, rnd, jb);
        BT_LAUNCH_CHECK();
      }
      offnorm_partial<<<OFFN_BLOCKS, 256, 0, st>>>(ap, p.np, offn);
      BT_LAUNCH_CHECK();
      offnorm_final<<<1, 32, 0, st>>>(offn, OFFN_BLOCKS, offn + OFFN_BLOCKS);
      BT_LAUNCH_CHECK();
      int h = 0;
      double off2 = 0.0;
      BT_CUDA_CHECK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
      BT_CUDA_CHECK(cudaMemcpyAsync(&off2, offn + OFFN_BLOCKS, sizeof(double),
                                    cudaMemcpyDeviceToHost, st));
      BT_CUDA_CHECK(cudaStreamSynchronize(st));
      const double off = sqrt(off2);
      if (getenv("BT_EIG_DEBUG"))
        fprintf(stderr, "[syevd n=%lld] sweep %d off/normF %.3e rotated %d\n", (long long)n,
                sweep, off / normf, h);
      done = (h == 0) || (off <= 2.2e-16 * sqrt(static_cast<double>(n)) * normf) ||
             (off <= 1e-10 * normf && off > 0.5 * prev);
      prev = off;
    }
    BT_REQUIRE(done, BT_E_CONV, "syevd: block Jacobi did not converge in 40 sweeps");
    diag_kernel<<<static_cast<unsigned>(bt_cdiv(p.np, 256)), 256, 0, st>>>(ap, p.np, d);
    BT_LAUNCH_CHECK();
  }
  int64_t* perm = reinterpret_cast<int64_t*>(ws + p.off_perm);
  rank_kernel<<<static_cast<unsigned>(bt_cdiv(p.np, 128)), 128, 0, st>>>(d, p.np, perm);
  BT_LAUNCH_CHECK();
  output_kernel<<<static_cast<unsigned>(std::min<int64_t>(n, 4096)), 256, 0, st>>>(d, q, p.np, n,
                                                                                  perm, w, v);
  BT_LAUNCH_CHECK();
  return BT_OK;
}
