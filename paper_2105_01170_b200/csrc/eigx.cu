// K8 (leading eigenpairs): Householder tridiagonalisation + bisection +
// inverse iteration + back-transformation, for the Gram matrices of the
// Tucker path when only the leading nvec eigenvectors are needed (the
// reference's LAPACK SVD, decomp.py:172/227, returns them for the leading r).
//
//   1. T = Q^T A Q by n-2 Householder reflectors (per step: reflector in one
//      CTA, SYMV p = tau A22 v by warps-per-row, rank-2 update A22 -= v w^T +
//      w v^T; the 8-30 MB matrix stays in L2).
//   2. the nvec largest eigenvalues of T by Sturm-count bisection (one thread
//      per eigenvalue, absolute accuracy ~eps ||T||).
//   3. their eigenvectors by inverse iteration on T - lambda I (tridiagonal LU
//      with partial pivoting), one warp per cluster of close eigenvalues
//      with modified Gram-Schmidt inside the cluster (LAPACK dstein's rule:
//      gap <= 1e-3 ||T||).
//   4. V = Q Y, one warp per vector applying the reflectors in reverse.
// Output as bt_syevd_f64: eigenvalues descending, vectors sign-normalised
// (largest-|.| entry positive, first on ties, decomp.py:176-179).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "bt_common.cuh"

namespace cg = cooperative_groups;

namespace {

__device__ double block_reduce_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// Whole tridiagonalisation in one cooperative launch (one 1024-thread CTA
// per SM, two grid-wide barriers per reflector): every CTA recomputes the
// reflector of column k redundantly from row k (A is kept exactly symmetric),
// the SYMV and the rank-2 update are split into (row, 256-column chunk) work
// items over all warps of the grid for memory-level parallelism, with
// per-chunk SYMV partials summed in a fixed order (deterministic).
constexpr int TCHUNK = 256;

__global__ void __launch_bounds__(1024)
    tridiag_coop_kernel(double* __restrict__ a, int64_t n, double* __restrict__ d,
                        double* __restrict__ e, double* __restrict__ tau,
                        double* __restrict__ vref, double* __restrict__ ppart,
                        double* __restrict__ part) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double smv[];
  double* vs = smv;       // v (n)
  double* ws = smv + n;   // w (n)
  __shared__ double red[32];
  __shared__ double sh[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int64_t gwarps = (int64_t)gridDim.x * nw;
  const int64_t gw = (int64_t)blockIdx.x * nw + warp;
  const int64_t nchunk = (n + TCHUNK - 1) / TCHUNK;
  for (int64_t k = 0; k + 2 < n; ++k) {
    const int64_t m0 = k + 1;
    const double* rowk = a + k * n;
    // -- reflector (redundant per CTA)
    double s = 0.0;
    for (int64_t i = m0 + 1 + threadIdx.x; i < n; i += blockDim.x) s = fma(rowk[i], rowk[i], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tail2 = 0.0;
      for (int w2 = 0; w2 < nw; ++w2) tail2 += red[w2];
      const double x0 = rowk[m0];
      if (tail2 == 0.0) {
        sh[0] = 0.0;
        sh[1] = x0;
        sh[2] = 0.0;
      } else {
        const double nrm = sqrt(x0 * x0 + tail2);
        const double beta = (x0 >= 0.0) ? -nrm : nrm;
        sh[0] = (beta - x0) / beta;
        sh[1] = beta;
        sh[2] = 1.0 / (x0 - beta);
      }
      if (blockIdx.x == 0) {
        d[k] = rowk[k];
        tau[k] = sh[0];
        e[k] = sh[1];
      }
    }
    __syncthreads();
    const double t = sh[0], sc = sh[2];
    for (int64_t i = m0 + threadIdx.x; i < n; i += blockDim.x) vs[i] = (i == m0) ? 1.0 : rowk[i] * sc;
    if (blockIdx.x == 0)
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        vref[k * n + i] = (i < m0) ? 0.0 : ((i == m0) ? 1.0 : rowk[i] * sc);
    __syncthreads();
    // -- SYMV partials: item (row i, chunk c) -> ppart[i * nchunk + c]
    const int64_t c0 = m0 / TCHUNK;
    const int64_t nc = nchunk - c0;
    const int64_t items = (n - m0) * nc;
    for (int64_t it = gw; it < items; it += gwarps) {
      const int64_t i = m0 + it / nc;
      const int64_t c = c0 + it % nc;
      const int64_t j0 = max(m0, c * TCHUNK), j1 = min(n, (c + 1) * TCHUNK);
      const double* row = a + i * n;
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < TCHUNK / 32; ++q) {
        const int64_t j = j0 + lane + 32 * q;
        if (j < j1) acc = fma(row[j], vs[j], acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) ppart[i * nchunk + c] = acc;
    }
    grid.sync();
    // -- p = t * sum_c ppart (every CTA, fixed order), p^T v, w = p - (t/2)(p^T v) v
    double local = 0.0;
    for (int64_t i = m0 + threadIdx.x; i < n; i += blockDim.x) {
      double acc = 0.0;
      for (int64_t c = c0; c < nchunk; ++c) acc += ppart[i * nchunk + c];
      acc *= t;
      ws[i] = acc;
      local = fma(acc, vs[i], local);
    }
    local = warp_sum(local);
    if (lane == 0) red[warp] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
      double ptv = 0.0;
      for (int w2 = 0; w2 < nw; ++w2) ptv += red[w2];
      sh[0] = 0.5 * t * ptv;
    }
    __syncthreads();
    const double alpha = sh[0];
    for (int64_t i = m0 + threadIdx.x; i < n; i += blockDim.x) ws[i] = ws[i] - alpha * vs[i];
    __syncthreads();
    // -- rank-2 update over the same (row, chunk) items
    for (int64_t it = gw; it < items; it += gwarps) {
      const int64_t i = m0 + it / nc;
      const int64_t c = c0 + it % nc;
      const int64_t j0 = max(m0, c * TCHUNK), j1 = min(n, (c + 1) * TCHUNK);
      double* row = a + i * n;
      const double vi = vs[i], wi = ws[i];
#pragma unroll
      for (int q = 0; q < TCHUNK / 32; ++q) {
        const int64_t j = j0 + lane + 32 * q;
        if (j < j1) row[j] -= vi * ws[j] + wi * vs[j];
      }
    }
    grid.sync();
  }
}

// Single-CTA tridiagonalisation for small n (<= 512): block barriers instead
// of grid barriers (the multi-CTA version is barrier-latency bound there).
__global__ void __launch_bounds__(1024)
    tridiag_cta_kernel(double* __restrict__ a, int64_t n, double* __restrict__ d,
                       double* __restrict__ e, double* __restrict__ tau,
                       double* __restrict__ vref) {
  extern __shared__ __align__(16) double smv[];
  double* vs = smv;
  double* ps = smv + n;
  __shared__ double red[32];
  __shared__ double sh[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  for (int64_t k = 0; k + 2 < n; ++k) {
    const int64_t m0 = k + 1;
    const double* rowk = a + k * n;
    double s = 0.0;
    for (int64_t i = m0 + 1 + threadIdx.x; i < n; i += blockDim.x) s = fma(rowk[i], rowk[i], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tail2 = 0.0;
      for (int w = 0; w < nwarps; ++w) tail2 += red[w];
      const double x0 = rowk[m0];
      if (tail2 == 0.0) {
        sh[0] = 0.0;
        sh[1] = x0;
        sh[2] = 0.0;
      } else {
        const double nrm = sqrt(x0 * x0 + tail2);
        const double beta = (x0 >= 0.0) ? -nrm : nrm;
        sh[0] = (beta - x0) / beta;
        sh[1] = beta;
        sh[2] = 1.0 / (x0 - beta);
      }
      d[k] = rowk[k];
      tau[k] = sh[0];
      e[k] = sh[1];
    }
    __syncthreads();
    const double t = sh[0], sc = sh[2];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double v = (i < m0) ? 0.0 : ((i == m0) ? 1.0 : rowk[i] * sc);
      vs[i] = v;
      vref[k * n + i] = v;
    }
    __syncthreads();
    // SYMV: warp per row
    double local = 0.0;
    for (int64_t i = m0 + warp; i < n; i += nwarps) {
      const double* row = a + i * n;
      double acc = 0.0;
      for (int64_t j = m0 + lane; j < n; j += 32) acc = fma(row[j], vs[j], acc);
      acc = warp_sum(acc) * t;
      if (lane == 0) {
        ps[i] = acc;
        local = fma(acc, vs[i], local);
      }
    }
    if (lane == 0) red[warp] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
      double ptv = 0.0;
      for (int w = 0; w < nwarps; ++w) ptv += red[w];
      sh[0] = 0.5 * t * ptv;
    }
    __syncthreads();
    const double alpha = sh[0];
    for (int64_t i = m0 + threadIdx.x; i < n; i += blockDim.x) ps[i] = ps[i] - alpha * vs[i];
    __syncthreads();
    for (int64_t i = m0 + warp; i < n; i += nwarps) {
      double* row = a + i * n;
      const double vi = vs[i], wi = ps[i];
      for (int64_t j = m0 + lane; j < n; j += 32) row[j] -= vi * ps[j] + wi * vs[j];
    }
    __syncthreads();
  }
}

__global__ void tail_kernel(const double* __restrict__ a, int64_t n, double* __restrict__ d,
                            double* __restrict__ e) {
  if (threadIdx.x == 0) {
    d[n - 2] = a[(n - 2) * n + (n - 2)];
    d[n - 1] = a[(n - 1) * n + (n - 1)];
    e[n - 2] = a[(n - 1) * n + (n - 2)];
  }
}

// number of eigenvalues of T strictly less than x (Sturm sequence, dstebz)
__device__ int sturm_less(const double* __restrict__ d, const double* __restrict__ e2, int64_t n,
                          double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0.0) ++cnt;
  for (int64_t i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// e2 = e^2, bounds (Gershgorin), pivmin
__global__ void prep_kernel(const double* __restrict__ d, const double* __restrict__ e, int64_t n,
                            double* __restrict__ e2, double* __restrict__ bounds) {
  __shared__ double lo_s[256], hi_s[256], em_s[256];
  double lo = INFINITY, hi = -INFINITY, em = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double el = (i > 0) ? fabs(e[i - 1]) : 0.0;
    const double er = (i < n - 1) ? fabs(e[i]) : 0.0;
    lo = fmin(lo, d[i] - el - er);
    hi = fmax(hi, d[i] + el + er);
    if (i < n - 1) {
      e2[i] = e[i] * e[i];
      em = fmax(em, e[i] * e[i]);
    }
  }
  lo_s[threadIdx.x] = lo;
  hi_s[threadIdx.x] = hi;
  em_s[threadIdx.x] = em;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < (int)blockDim.x; ++t) {
      lo = fmin(lo, lo_s[t]);
      hi = fmax(hi, hi_s[t]);
      em = fmax(em, em_s[t]);
    }
    const double tnorm = fmax(fabs(lo), fabs(hi));
    bounds[0] = lo - 4.0 * 2.2e-16 * tnorm - 1e-300;
    bounds[1] = hi + 4.0 * 2.2e-16 * tnorm + 1e-300;
    bounds[2] = fmax(2.2e-308, 2.2e-308 * em);  // pivmin (dstebz: safmin * max e^2)
    bounds[3] = tnorm;
  }
}

// w[c] = (c+1)-th largest eigenvalue, c in [c_begin, nvec): multisection,
// one warp per eigenvalue, 32 Sturm counts per round (interval shrinks 33x a
// round).  With limit != null only c <= *limit are computed (the rest = 0).
__global__ void __launch_bounds__(256)
    bisect_kernel(const double* __restrict__ d, const double* __restrict__ e2, int64_t n,
                  int64_t c_begin, int64_t nvec, const double* __restrict__ bounds,
                  const int64_t* __restrict__ limit, double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t c = c_begin + blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c >= nvec) return;
  if (limit != nullptr && c > *limit) {
    if (lane == 0) w[c] = 0.0;
    return;
  }
  const int target = static_cast<int>(n - 1 - c);  // eigenvalue index in ascending order
  double lo = bounds[0], hi = bounds[1];
  const double pivmin = bounds[2];
  for (int round = 0; round < 40; ++round) {
    if (hi - lo <= 2.0 * 2.2e-16 * fmax(fabs(lo), fabs(hi)) + pivmin) break;
    const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    const bool le = sturm_less(d, e2, n, x, pivmin) <= target;   // lambda_target >= x
    const unsigned mask = __ballot_sync(0xffffffffu, le);
    // points are increasing in lane; le is true for a prefix of lanes
    const int cnt = __popc(mask);
    const double nlo = (cnt > 0) ? lo + (hi - lo) * (double)cnt / 33.0 : lo;
    const double nhi = (cnt < 32) ? lo + (hi - lo) * (double)(cnt + 1) / 33.0 : hi;
    if (!(nlo < nhi) || (nlo == lo && nhi == hi)) break;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) w[c] = 0.5 * (lo + hi);
}

// number of eigenvalues strictly above tau * |w0| (Sturm count), into *count
__global__ void count_above_kernel(const double* __restrict__ d, const double* __restrict__ e2,
                                   int64_t n, const double* __restrict__ bounds,
                                   const double* __restrict__ w, double tau,
                                   int64_t* __restrict__ count) {
  if (threadIdx.x != 0) return;
  if (tau < 0.0) {
    *count = n;
    return;
  }
  const double x = tau * fabs(w[0]);
  // eigenvalues > x  ==  n - #(<= x) ; use #(< x) as a slight over-count (safe)
  *count = n - sturm_less(d, e2, n, x, bounds[2]);
}

// Cluster codes: start[c] = 1 opens a cluster (c == 0 or gap w[c-1] - w[c]
// > 1e-3 ||T||, dstein's rule); 2 opens a tight sub-cluster inside one
// (gap > TIGHT_GAP ||T||); 0 continues the current sub-cluster; -1 = no
// vector (eigenvalue at or below tau * |w0|).  Inverse iteration runs one
// warp per tight sub-cluster (MGS inside it, as dstein does for the whole
// cluster): a vector of a sub-cluster separated by more than TIGHT_GAP ||T||
// is accurate to ~eps / TIGHT_GAP on its own, so only the orthogonality
// across sub-clusters is left, restored by cluster_orth_kernel.  This keeps
// the sequential MGS chains short on smoothly decaying spectra (C3 mode 1:
// one 1e-3 cluster of ~50 eigenvalues).
constexpr double TIGHT_GAP = 1e-6;

__global__ void cluster_kernel(const double* __restrict__ w, int64_t nvec,
                               const double* __restrict__ bounds, double tau,
                               int* __restrict__ start) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nvec) return;
  if (c > 0 && !(w[c] > tau * fabs(w[0]))) {
    start[c] = -1;
    return;
  }
  if (c == 0) {
    start[c] = 1;
    return;
  }
  const double gap = w[c - 1] - w[c];
  start[c] = gap > 1e-3 * bounds[3] ? 1 : (gap > TIGHT_GAP * bounds[3] ? 2 : 0);
}

// Orthonormalise each 1e-3 cluster that holds more than one tight
// sub-cluster: classical Gram-Schmidt with one reorthogonalisation (CGS2)
// over its vectors in order, one CTA per cluster.  The vectors are already
// orthogonal to ~eps / TIGHT_GAP, so this only polishes them.
__global__ void __launch_bounds__(1024)
    cluster_orth_kernel(int64_t n, int64_t nvec, const int* __restrict__ start,
                        double* __restrict__ y) {
  extern __shared__ __align__(16) double dots[];
  __shared__ double red[32];
  const int64_t c0 = blockIdx.x;
  if (c0 >= nvec || start[c0] != 1) return;
  int64_t c1 = c0 + 1;
  bool multi = false;
  while (c1 < nvec && (start[c1] == 0 || start[c1] == 2)) {
    multi |= start[c1] == 2;
    ++c1;
  }
  if (!multi) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t c = c0 + 1; c < c1; ++c) {
    double* yc = y + c * n;
    const int64_t k = c - c0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int64_t o = warp; o < k; o += nw) {
        const double* yo = y + (c0 + o) * n;
        double s = 0.0;
        for (int64_t i = lane; i < n; i += 32) s = fma(yo[i], yc[i], s);
        s = warp_sum(s);
        if (lane == 0) dots[o] = s;
      }
      __syncthreads();
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double acc = yc[i];
        for (int64_t o = 0; o < k; ++o) acc = fma(-dots[o], y[(c0 + o) * n + i], acc);
        yc[i] = acc;
      }
      __syncthreads();
    }
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(yc[i], yc[i], s);
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w];
    const double inv = (t > 0.0) ? 1.0 / sqrt(t) : 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) yc[i] *= inv;
    __syncthreads();
  }
}

// Inverse iteration: one warp per tight sub-cluster (a warp whose first
// vector does not open one exits).  Y is stored vector-major: y[c * n + i].
__global__ void __launch_bounds__(32)
    invit_kernel(const double* __restrict__ d, const double* __restrict__ e, int64_t n,
                 int64_t nvec, const double* __restrict__ wv, const int* __restrict__ start,
                 const double* __restrict__ bounds, double* __restrict__ y,
                 double* __restrict__ scratch) {
  const int64_t c0 = blockIdx.x;
  if (c0 >= nvec) return;
  if (start[c0] == -1) {
    for (int64_t i = threadIdx.x; i < n; i += 32) y[c0 * n + i] = 0.0;
    return;
  }
  if (!start[c0]) return;
  int64_t c1 = c0 + 1;
  while (c1 < nvec && start[c1] == 0) ++c1;
  const int lane = threadIdx.x;
  // LU of T - lambda I with partial pivoting: rows i store (u0 diag, u1, u2 super) and
  // multiplier l, piv flag
  double* u0 = scratch + c0 * 5 * n;
  double* u1 = u0 + n;
  double* u2 = u1 + n;
  double* lm = u2 + n;
  double* pv = lm + n;
  const double tnorm = bounds[3];
  const double eps = 2.2e-16;
  double prev_lambda = 0.0;
  for (int64_t c = c0; c < c1; ++c) {
    double lambda = wv[c];
    // dstein: separate coincident eigenvalues in a cluster slightly
    if (c > c0 && lambda >= prev_lambda - 10.0 * eps * tnorm) lambda = prev_lambda - 10.0 * eps * tnorm;
    prev_lambda = lambda;
    double* yc = y + c * n;
    if (lane == 0) {
      // factor T - lambda I = P L U (U: diagonal u0, superdiagonals u1, u2)
      double al = d[0] - lambda, be = (n > 1) ? e[0] : 0.0;
      for (int64_t i = 0; i < n - 1; ++i) {
        const double sub = e[i];
        const double dn = d[i + 1] - lambda;
        const double en = (i + 1 < n - 1) ? e[i + 1] : 0.0;
        if (fabs(al) >= fabs(sub)) {
          const double piv = (al == 0.0) ? eps * tnorm + 1e-300 : al;
          const double l = sub / piv;
          u0[i] = piv;
          u1[i] = be;
          u2[i] = 0.0;
          lm[i] = l;
          pv[i] = 0.0;
          al = dn - l * be;
          be = en;
        } else {
          const double l = al / sub;
          u0[i] = sub;
          u1[i] = dn;
          u2[i] = en;
          lm[i] = l;
          pv[i] = 1.0;
          al = be - l * dn;
          be = -l * en;
        }
      }
      const double a0 = al;
      u0[n - 1] = (a0 == 0.0) ? eps * tnorm + 1e-300 : a0;
      u1[n - 1] = 0.0;
      u2[n - 1] = 0.0;
      // deterministic start vector
      for (int64_t i = 0; i < n; ++i) {
        uint64_t h = (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull ^ (uint64_t)(c + 7) * 0xBF58476D1CE4E5B9ull;
        h ^= h >> 31;
        yc[i] = 1.0 + 0.5 * ((double)(h & 0xFFFFF) / 1048576.0 - 0.5);
      }
    }
    __syncwarp();
    for (int iter = 0; iter < 3; ++iter) {
      if (lane == 0) {
        // forward: apply row interchanges and multipliers
        for (int64_t i = 0; i < n - 1; ++i) {
          if (pv[i] != 0.0) {
            const double t = yc[i];
            yc[i] = yc[i + 1];
            yc[i + 1] = t;
          }
          yc[i + 1] -= lm[i] * yc[i];
        }
        // back substitution with U (diag u0, super u1, super-super u2)
        yc[n - 1] = yc[n - 1] / u0[n - 1];
        if (n > 1) yc[n - 2] = (yc[n - 2] - u1[n - 2] * yc[n - 1]) / u0[n - 2];
        for (int64_t i = n - 3; i >= 0; --i)
          yc[i] = (yc[i] - u1[i] * yc[i + 1] - u2[i] * yc[i + 2]) / u0[i];
      }
      __syncwarp();
      // MGS against earlier members of the cluster, then normalise
      for (int64_t o = c0; o < c; ++o) {
        const double* yo = y + o * n;
        double s = 0.0;
        for (int64_t i = lane; i < n; i += 32) s = fma(yo[i], yc[i], s);
        s = warp_sum(s);
        for (int64_t i = lane; i < n; i += 32) yc[i] -= s * yo[i];
        __syncwarp();
      }
      double s = 0.0;
      for (int64_t i = lane; i < n; i += 32) s = fma(yc[i], yc[i], s);
      s = warp_sum(s);
      const double inv = (s > 0.0) ? 1.0 / sqrt(s) : 0.0;
      for (int64_t i = lane; i < n; i += 32) yc[i] *= inv;
      __syncwarp();
    }
  }
}

// V = Q Y: apply reflectors k = n-3 .. 0; a CTA stages 8 vectors in shared
// memory (one warp each) so the reflector sweep runs out of smem, the
// reflector rows (shared by the 8 warps) come through L1.
__global__ void __launch_bounds__(256)
    backtransform_kernel(const double* __restrict__ vref, const double* __restrict__ tau,
                         int64_t n, int64_t nvec, const int* __restrict__ start,
                         double* __restrict__ y) {
  extern __shared__ __align__(16) double ysm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = blockIdx.x * 8 + warp;
  const bool live = c < nvec && start[c] != -1;
  double* yc = ysm + warp * n;
  if (live)
    for (int64_t i = lane; i < n; i += 32) yc[i] = y[c * n + i];
  __syncwarp();
  if (live) {
    for (int64_t k = n - 3; k >= 0; --k) {
      const double t = tau[k];
      if (t == 0.0) continue;
      const double* v = vref + k * n;
      double s = 0.0;
      for (int64_t i = k + 1 + lane; i < n; i += 32) s = fma(__ldg(v + i), yc[i], s);
      s = warp_sum(s) * t;
      for (int64_t i = k + 1 + lane; i < n; i += 32) yc[i] -= s * __ldg(v + i);
      __syncwarp();
    }
    for (int64_t i = lane; i < n; i += 32) y[c * n + i] = yc[i];
  }
}

// sign rule + row-major output vout (n x nvec)
__global__ void __launch_bounds__(256)
    sign_out_kernel(const double* __restrict__ y, int64_t n, int64_t nvec,
                    double* __restrict__ vout) {
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  for (int64_t c = blockIdx.x; c < nvec; c += gridDim.x) {
    const double* yc = y + c * n;
    double best = -1.0;
    int64_t bidx = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double x = fabs(yc[i]);
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
    const double sgn = (yc[bi[0]] < 0.0) ? -1.0 : 1.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) vout[i * nvec + c] = sgn * yc[i];
    __syncthreads();
  }
}

struct XPlan {
  int64_t off_a, off_v, off_d, off_e, off_e2, off_tau, off_p, off_part, off_bounds, off_start,
      off_y, off_scr, off_ppart, off_cnt, total;
  int parts;
};

XPlan xplan(int64_t n, int64_t nvec) {
  XPlan p;
  p.parts = 148 * 4;
  int64_t o = 0;
  auto take = [&](int64_t k) {
    int64_t at = o;
    o += (k + 1) / 2 * 2;
    return at;
  };
  p.off_a = take(n * n);
  p.off_v = take(n * n);
  p.off_d = take(n);
  p.off_e = take(n);
  p.off_e2 = take(n);
  p.off_tau = take(n);
  p.off_p = take(n);
  p.off_part = take(p.parts);
  p.off_bounds = take(4);
  p.off_start = take(nvec);  // ints fit in doubles
  p.off_y = take(nvec * n);
  p.off_scr = take(nvec * 5 * n);
  p.off_ppart = take(n * ((n + 255) / 256));
  p.off_cnt = take(2);
  p.total = o;
  return p;
}

}  // namespace

extern "C" int64_t bt_syevx_ws_bytes(int64_t n, int64_t nvec) { return xplan(n, nvec).total * 8; }

extern "C" int bt_syevx_f64(const double* a, int64_t n, int64_t nvec, double vec_tau, double* w,
                            double* v, void* wsv, int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_syevx_f64");
  BT_REQUIRE(n >= 3 && nvec >= 1 && nvec <= n, BT_E_SHAPE, "syevx: need n >= 3, 1 <= nvec <= n");
  BT_REQUIRE(n <= 3200, BT_E_SHAPE, "syevx: n = %lld above the shared-memory limit 3200",
             (long long)n);
  XPlan p = xplan(n, nvec);
  BT_REQUIRE(ws_bytes >= p.total * 8, BT_E_VALUE, "syevx: workspace too small");
  cudaStream_t st = bt_stream(stream);
  double* ws = static_cast<double*>(wsv);
  double* A = ws + p.off_a;
  double* V = ws + p.off_v;
  double* d = ws + p.off_d;
  double* e = ws + p.off_e;
  double* e2 = ws + p.off_e2;
  double* tau = ws + p.off_tau;
  double* pp = ws + p.off_p;
  double* part = ws + p.off_part;
  double* bounds = ws + p.off_bounds;
  int* start = reinterpret_cast<int*>(ws + p.off_start);
  double* y = ws + p.off_y;
  double* scr = ws + p.off_scr;
  BT_CUDA_CHECK(cudaMemcpyAsync(A, a, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
  const bool dbg = getenv("BT_EIG_DEBUG") != nullptr;
  cudaEvent_t ev[6];
  if (dbg)
    for (auto& x : ev) cudaEventCreate(&x);
  if (dbg) cudaEventRecord(ev[0], st);
  if (n <= 160) {
    const size_t sm = sizeof(double) * 2 * n;
    BT_CUDA_CHECK(cudaFuncSetAttribute(tridiag_cta_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm)));
    tridiag_cta_kernel<<<1, 1024, sm, st>>>(A, n, d, e, tau, V);
    BT_LAUNCH_CHECK();
  } else {
    int dev = 0, per_sm = 0;
    BT_CUDA_CHECK(cudaGetDevice(&dev));
    BT_CUDA_CHECK(cudaFuncSetAttribute(tridiag_coop_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sizeof(double) * 2 * n)));
    BT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tridiag_coop_kernel, 1024,
                                                                sizeof(double) * 2 * n));
    // small problems are grid-barrier bound (fewer CTAs), large ones latency
    // bound on the L2-resident SYMV/update (more warps in flight)
    const int grid = std::min(bt_num_sms() * std::max(per_sm, 1), bt_num_sms());
    double* ppart = ws + p.off_ppart;
    void* args[] = {&A, (void*)&n, &d, &e, &tau, &V, &ppart, &part};
    const size_t sm = sizeof(double) * 2 * n;
    BT_CUDA_CHECK(cudaFuncSetAttribute(tridiag_coop_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(std::max<size_t>(sm, 1))));
    BT_CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)tridiag_coop_kernel, dim3(grid),
                                              dim3(1024), args, sm, st));
    BT_LAUNCH_CHECK();
  }
  if (dbg) cudaEventRecord(ev[1], st);
  tail_kernel<<<1, 32, 0, st>>>(A, n, d, e);
  BT_LAUNCH_CHECK();
  prep_kernel<<<1, 256, 0, st>>>(d, e, n, e2, bounds);
  BT_LAUNCH_CHECK();
  // largest eigenvalue first, then only those above vec_tau * w0 (+1 for the count)
  int64_t* cnt = reinterpret_cast<int64_t*>(ws + p.off_cnt);
  bisect_kernel<<<1, 32, 0, st>>>(d, e2, n, 0, 1, bounds, nullptr, w);
  BT_LAUNCH_CHECK();
  count_above_kernel<<<1, 32, 0, st>>>(d, e2, n, bounds, w, vec_tau, cnt);
  BT_LAUNCH_CHECK();
  if (nvec > 1) {
    bisect_kernel<<<static_cast<unsigned>(bt_cdiv(nvec - 1, 8)), 256, 0, st>>>(d, e2, n, 1, nvec,
                                                                                bounds, cnt, w);
    BT_LAUNCH_CHECK();
  }
  if (dbg) cudaEventRecord(ev[2], st);
  cluster_kernel<<<static_cast<unsigned>(bt_cdiv(nvec, 256)), 256, 0, st>>>(w, nvec, bounds, vec_tau,
                                                                          start);
  BT_LAUNCH_CHECK();
  invit_kernel<<<static_cast<unsigned>(nvec), 32, 0, st>>>(d, e, n, nvec, w, start, bounds, y, scr);
  BT_LAUNCH_CHECK();
  {
    const size_t sm = sizeof(double) * static_cast<size_t>(nvec);
    if (sm > 48 * 1024)
      BT_CUDA_CHECK(cudaFuncSetAttribute(cluster_orth_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sm)));
    cluster_orth_kernel<<<static_cast<unsigned>(nvec), 1024, sm, st>>>(n, nvec, start, y);
    BT_LAUNCH_CHECK();
  }
  if (dbg) cudaEventRecord(ev[3], st);
  {
    const size_t sm = sizeof(double) * 8 * n;
    BT_CUDA_CHECK(cudaFuncSetAttribute(backtransform_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm)));
    backtransform_kernel<<<static_cast<unsigned>(bt_cdiv(nvec, 8)), 256, sm, st>>>(V, tau, n, nvec,
                                                                                 start, y);
  }
  BT_LAUNCH_CHECK();
  if (dbg) cudaEventRecord(ev[4], st);
  sign_out_kernel<<<static_cast<unsigned>(std::min<int64_t>(nvec, 4096)), 256, 0, st>>>(y, n, nvec, v);
  BT_LAUNCH_CHECK();
  if (dbg) {
    cudaEventRecord(ev[5], st);
    cudaEventSynchronize(ev[5]);
    float t[5];
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    fprintf(stderr, "[syevx n=%lld nvec=%lld] tridiag %.3f bisect %.3f invit %.3f back %.3f out %.3f ms\n",
            (long long)n, (long long)nvec, t[0], t[1], t[2], t[3], t[4]);
    for (auto& x : ev) cudaEventDestroy(x);
  }
  return BT_OK;
}
