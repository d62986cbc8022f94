// Cyclic (round-robin parallel) two-sided Jacobi on a symmetric matrix held
// in shared memory: the on-chip eigensolver behind the CP pinv (numpy
// pinv, decomp.py:387) and the subproblems of the block-Jacobi syevd.
#pragma once

#include "bt_common.cuh"

// sweeps of the last jacobi_warp_t call (diagnostics: bt_debug_jacobi_sweeps)
static __device__ int g_jacobi_sweeps;

// Circle-method round-robin pair k of round rnd for n (even) players
// (0 <= rnd, k < n - 1: conditional subtractions instead of integer modulo).
static __device__ __forceinline__ void rr_pair(int n, int rnd, int k, int& p, int& q) {
  const int m = n - 1;
  if (k == 0) {
    p = rnd;
    q = m;
  } else {
    p = rnd + k;
    if (p >= m) p -= m;
    q = rnd - k + m;
    if (q >= m) q -= m;
  }
  if (p > q) {
    int t = p;
    p = q;
    q = t;
  }
}

// Rotation (c, s) annihilating a_pq, from approximate reciprocal / rsqrt
// refined by two Newton steps each (~1 ulp; c^2 + s^2 = 1 to working
// precision) -- a shorter dependent chain than IEEE div + sqrt, which sets
// the latency of every Jacobi round.
static __device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
static __device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}
static __device__ __forceinline__ void jacobi_rotation(double app, double aqq, double apq,
                                                       double& c, double& s) {
  const double theta = (aqq - app) * rcp_nr(2.0 * apq);
  const double at = fabs(theta);
  double t;
  if (at > 1e150) {
    t = 0.5 * rcp_nr(theta);
  } else {
    const double q2 = fma(theta, theta, 1.0);
    const double root = q2 * rsqrt_nr(q2);
    t = rcp_nr(at + root);
    if (theta < 0.0) t = -t;
  }
  c = rsqrt_nr(fma(t, t, 1.0));
  s = t * c;
}

// Cyclic round-robin Jacobi on a symmetric (n x n, ld) smem matrix,
// accumulating the eigenvectors in qv; one parameter phase and ONE update
// phase per round.  The update applies both rotations
// of a round to disjoint 2x2 blocks (pair k1 rows x pair k2 columns: new
// block = L1 B L2^T), so rows and columns need no separate passes, and the
// eigenvector accumulator's column pairs are updated in the same phase.
// Rotate iff |a_pq| > abs_tol and |a_pq| > rel_tol sqrt(|a_pp a_qq|).
// Works for any blockDim (multiple of 32); callers use 1024 threads.
static __device__ __noinline__ int jacobi_fast(double* a, double* qv, int n, int ld, double* cs,
                                               double* sn, int* pp, int* qq, int max_sweeps,
                                               double abs_tol, double rel_tol) {
  __shared__ int rotated;
  const int nt = blockDim.x;
  const int half = n / 2;
  int any = 0;
  for (int idx = threadIdx.x; idx < n * n; idx += nt) {
    const int r = idx / n, c = idx - r * n;
    qv[r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      for (int k = threadIdx.x; k < half; k += nt) {
        int p, q;
        rr_pair(n, rnd, k, p, q);
        const double apq = a[p * ld + q];
        const double app = a[p * ld + p], aqq = a[q * ld + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && fabs(apq) > abs_tol && fabs(apq) > rel_tol * sqrt(fabs(app) * fabs(aqq))) {
          jacobi_rotation(app, aqq, apq, c, s);
          rotated = 1;
        }
        cs[k] = c;
        sn[k] = s;
        pp[k] = p;
        qq[k] = q;
      }
      __syncthreads();
      // 2-D thread map (lane -> k2 / row, warp -> k1 / pair): no divisions
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = nt >> 5;
      for (int k1 = wid; k1 < half; k1 += nw) {
        const double s1 = sn[k1], c1 = cs[k1];
        const int p1 = pp[k1], q1 = qq[k1];
        for (int k2 = lane; k2 < half; k2 += 32) {
          const double s2 = sn[k2];
          if (s1 == 0.0 && s2 == 0.0) continue;
          const double c2 = cs[k2];
          const int p2 = pp[k2], q2 = qq[k2];
          const double x11 = a[p1 * ld + p2], x12 = a[p1 * ld + q2];
          const double x21 = a[q1 * ld + p2], x22 = a[q1 * ld + q2];
          const double y11 = c1 * x11 - s1 * x21, y12 = c1 * x12 - s1 * x22;
          const double y21 = s1 * x11 + c1 * x21, y22 = s1 * x12 + c1 * x22;
          a[p1 * ld + p2] = c2 * y11 - s2 * y12;
          a[q1 * ld + q2] = s2 * y21 + c2 * y22;
          a[p1 * ld + q2] = (k1 == k2) ? 0.0 : s2 * y11 + c2 * y12;
          a[q1 * ld + p2] = (k1 == k2) ? 0.0 : c2 * y21 - s2 * y22;
        }
        if (s1 == 0.0) continue;
        for (int i = lane; i < n; i += 32) {
          const double x = qv[i * ld + p1], y = qv[i * ld + q1];
          qv[i * ld + p1] = c1 * x - s1 * y;
          qv[i * ld + q1] = s1 * x + c1 * y;
        }
      }
      __syncthreads();
    }
    const int r = rotated;
    __syncthreads();
    if (!r) break;
    any = 1;
  }
  return any;
}

// jacobi_warp with the size known at compile time: every lane's 2x2 blocks
// and eigenvector entries are fixed across rounds, so their (k1, k2) / (k, i)
// coordinates are computed once instead of by integer division every round.
// Same operations per element as jacobi_warp (identical results).
template <int N>
static __device__ __noinline__ int jacobi_warp_t(double* a, double* qv, int ld, double* cs,
                                                 double* sn, int* pp, int* qq, int max_sweeps,
                                                 double abs_tol, double rel_tol) {
  static_assert(N % 2 == 0 && N <= 64, "jacobi_warp_t: even N <= 64");
  constexpr int HALF = N / 2;
  constexpr int NB = (HALF * HALF + 31) / 32;
  constexpr int NQ = (HALF * N + 31) / 32;
  if (threadIdx.x >= 32) return 0;
  const int lane = threadIdx.x;
  int b1[NB], b2[NB], qk[NQ], qi[NQ];
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int e = lane + 32 * u;
    b1[u] = e < HALF * HALF ? e / HALF : -1;
    b2[u] = e < HALF * HALF ? e % HALF : 0;
  }
#pragma unroll
  for (int u = 0; u < NQ; ++u) {
    const int e = lane + 32 * u;
    qk[u] = e < HALF * N ? e / N : -1;
    qi[u] = e < HALF * N ? e % N : 0;
  }
  int any = 0;
  for (int idx = lane; idx < N * N; idx += 32) {
    const int r = idx / N, c = idx - r * N;
    qv[r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncwarp();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int rnd = 0; rnd < N - 1; ++rnd) {
      if (lane < HALF) {
        int p, q;
        rr_pair(N, rnd, lane, p, q);
        const double apq = a[p * ld + q];
        const double app = a[p * ld + p], aqq = a[q * ld + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && fabs(apq) > abs_tol && fabs(apq) > rel_tol * sqrt(fabs(app) * fabs(aqq))) {
          jacobi_rotation(app, aqq, apq, c, s);
          rotated = 1;
        }
        cs[lane] = c;
        sn[lane] = s;
        pp[lane] = p;
        qq[lane] = q;
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int k1 = b1[u], k2 = b2[u];
        if (k1 < 0) continue;
        const double s1 = sn[k1], s2 = sn[k2];
        if (s1 == 0.0 && s2 == 0.0) continue;
        const double c1 = cs[k1], c2 = cs[k2];
        const int p1 = pp[k1], q1 = qq[k1], p2 = pp[k2], q2 = qq[k2];
        const double x11 = a[p1 * ld + p2], x12 = a[p1 * ld + q2];
        const double x21 = a[q1 * ld + p2], x22 = a[q1 * ld + q2];
        const double y11 = c1 * x11 - s1 * x21, y12 = c1 * x12 - s1 * x22;
        const double y21 = s1 * x11 + c1 * x21, y22 = s1 * x12 + c1 * x22;
        a[p1 * ld + p2] = c2 * y11 - s2 * y12;
        a[q1 * ld + q2] = s2 * y21 + c2 * y22;
        a[p1 * ld + q2] = (k1 == k2) ? 0.0 : s2 * y11 + c2 * y12;
        a[q1 * ld + p2] = (k1 == k2) ? 0.0 : c2 * y21 - s2 * y22;
      }
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        const int k = qk[u], i = qi[u];
        if (k < 0) continue;
        const double s = sn[k];
        if (s == 0.0) continue;
        const double c = cs[k];
        const int p = pp[k], q = qq[k];
        const double x = qv[i * ld + p], y = qv[i * ld + q];
        qv[i * ld + p] = c * x - s * y;
        qv[i * ld + q] = s * x + c * y;
      }
      __syncwarp();
    }
    if (!__any_sync(0xffffffffu, rotated)) {
      if (lane == 0) g_jacobi_sweeps = sweep;
      break;
    }
    any = 1;
    if (lane == 0) g_jacobi_sweeps = sweep + 1;
  }
  return any;
}

// Warp-synchronous variant for n <= 32 (the CP pinv at R <= 32): executed by
// warp 0 alone, __syncwarp instead of CTA barriers (a round costs a few
// hundred cycles instead of two CTA-wide barriers).  Same rotation rule and
// update as jacobi_fast.  Other warps must not touch a / qv until the caller's
// next __syncthreads.
static __device__ __noinline__ int jacobi_warp(double* a, double* qv, int n, int ld, double* cs,
                                               double* sn, int* pp, int* qq, int max_sweeps,
                                               double abs_tol, double rel_tol) {
  if (threadIdx.x >= 32) return 0;
  const int lane = threadIdx.x;
  const int half = n / 2;
  int any = 0;
  for (int idx = lane; idx < n * n; idx += 32) {
    const int r = idx / n, c = idx - r * n;
    qv[r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncwarp();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      if (lane < half) {
        int p, q;
        rr_pair(n, rnd, lane, p, q);
        const double apq = a[p * ld + q];
        const double app = a[p * ld + p], aqq = a[q * ld + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && fabs(apq) > abs_tol && fabs(apq) > rel_tol * sqrt(fabs(app) * fabs(aqq))) {
          jacobi_rotation(app, aqq, apq, c, s);
          rotated = 1;
        }
        cs[lane] = c;
        sn[lane] = s;
        pp[lane] = p;
        qq[lane] = q;
      }
      __syncwarp();
      for (int e = lane; e < half * half; e += 32) {
        const int k1 = e / half, k2 = e - k1 * half;
        const double s1 = sn[k1], s2 = sn[k2];
        if (s1 == 0.0 && s2 == 0.0) continue;
        const double c1 = cs[k1], c2 = cs[k2];
        const int p1 = pp[k1], q1 = qq[k1], p2 = pp[k2], q2 = qq[k2];
        const double x11 = a[p1 * ld + p2], x12 = a[p1 * ld + q2];
        const double x21 = a[q1 * ld + p2], x22 = a[q1 * ld + q2];
        const double y11 = c1 * x11 - s1 * x21, y12 = c1 * x12 - s1 * x22;
        const double y21 = s1 * x11 + c1 * x21, y22 = s1 * x12 + c1 * x22;
        a[p1 * ld + p2] = c2 * y11 - s2 * y12;
        a[q1 * ld + q2] = s2 * y21 + c2 * y22;
        a[p1 * ld + q2] = (k1 == k2) ? 0.0 : s2 * y11 + c2 * y12;
        a[q1 * ld + p2] = (k1 == k2) ? 0.0 : c2 * y21 - s2 * y22;
      }
      for (int e = lane; e < half * n; e += 32) {
        const int k = e / n, i = e - k * n;
        const double s = sn[k];
        if (s == 0.0) continue;
        const double c = cs[k];
        const int p = pp[k], q = qq[k];
        const double x = qv[i * ld + p], y = qv[i * ld + q];
        qv[i * ld + p] = c * x - s * y;
        qv[i * ld + q] = s * x + c * y;
      }
      __syncwarp();
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
    any = 1;
  }
  return any;
}
