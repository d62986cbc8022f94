// Cyclic (round-robin parallel) two-sided Jacobi on a symmetric matrix held
// in shared memory: the on-chip eigensolver behind the CP pinv (numpy
// pinv, decomp.py:387) and the subproblems of the block-Jacobi syevd.
#pragma once

#include "bt_common.cuh"

// Circle-method round-robin pair k of round rnd for n (even) players.
static __device__ __forceinline__ void rr_pair(int n, int rnd, int k, int& p, int& q) {
  const int m = n - 1;
  if (k == 0) {
    p = rnd % m;
    q = m;
  } else {
    p = (rnd + k) % m;
    q = (rnd - k + m) % m;
  }
  if (p > q) {
    int t = p;
    p = q;
    q = t;
  }
}

// In-place cyclic Jacobi on a (n x n, ld) smem matrix a, accumulating q (n x n).
// Threads of the CTA cooperate; returns with a diagonalised.
static __device__ __noinline__ int jacobi_smem(double* a, double* qv, int n, int ld, double* cs,
                                        double* sn, int* pp, int* qq, int max_sweeps,
                                        double abs_tol) {
  __shared__ int rotated;
  int any = 0;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x)
    qv[(idx / n) * ld + idx % n] = (idx / n == idx % n) ? 1.0 : 0.0;
  __syncthreads();
  const int half = n / 2;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      for (int k = threadIdx.x; k < half; k += blockDim.x) {
        int p, q;
        rr_pair(n, rnd, k, p, q);
        const double apq = a[p * ld + q];
        const double app = a[p * ld + p], aqq = a[q * ld + q];
        double c = 1.0, s = 0.0;
        // rotate unless a_pq is negligible relative to the diagonal pair
        if (apq != 0.0 && fabs(apq) > abs_tol &&
            fabs(apq) > 1e-18 * sqrt(fabs(app) * fabs(aqq))) {
          const double theta = (aqq - app) / (2.0 * apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
          rotated = 1;
        }
        cs[k] = c;
        sn[k] = s;
        pp[k] = p;
        qq[k] = q;
      }
      __syncthreads();
      // rows p, q
      for (int idx = threadIdx.x; idx < half * n; idx += blockDim.x) {
        const int k = idx / n, j = idx % n;
        const double c = cs[k], s = sn[k];
        if (s == 0.0) continue;
        const int p = pp[k], q = qq[k];
        const double x = a[p * ld + j], y = a[q * ld + j];
        a[p * ld + j] = c * x - s * y;
        a[q * ld + j] = s * x + c * y;
      }
      __syncthreads();
      // columns p, q of a and of the eigenvector accumulator
      for (int idx = threadIdx.x; idx < half * n; idx += blockDim.x) {
        const int k = idx / n, i = idx % n;
        const double c = cs[k], s = sn[k];
        if (s == 0.0) continue;
        const int p = pp[k], q = qq[k];
        double x = a[i * ld + p], y = a[i * ld + q];
        a[i * ld + p] = c * x - s * y;
        a[i * ld + q] = s * x + c * y;
        x = qv[i * ld + p];
        y = qv[i * ld + q];
        qv[i * ld + p] = c * x - s * y;
        qv[i * ld + q] = s * x + c * y;
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

