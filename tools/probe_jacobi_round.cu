// Per-phase cycles of one round of the one-CTA two-sided Jacobi (jacobi.cuh jacobi_fast's
// loop body, timed by thread 0 with clock64) on a random symmetric n x n matrix.
#ifndef VARIANT
#define VARIANT 0
#endif
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2105_01170_b200/csrc/jacobi.cuh"

__global__ void __launch_bounds__(1024) probe(const double* a_in, int n, int sweeps, long long* clk, double* out) {
  extern __shared__ __align__(16) double sm[];
  const int ld = n + 1;
  double* a = sm;
  double* qv = a + n * ld;
  double* cs = qv + n * ld;
  double* sn = cs + n / 2;
  int* pp = reinterpret_cast<int*>(sn + n / 2);
  int* qq = pp + n / 2;
  const int nt = blockDim.x, half = n / 2;
  for (int idx = threadIdx.x; idx < n * n; idx += nt) {
    const int r = idx / n, c = idx - r * n;
    a[r * ld + c] = a_in[idx];
    qv[r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  long long t_p1 = 0, t_b1 = 0, t_p2 = 0, t_b2 = 0;
  int nrot = 0;
  for (int sweep = 0; sweep < sweeps; ++sweep) {
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      long long t0 = clock64();
      for (int k = threadIdx.x; k < half; k += nt) {
        int p, q;
        rr_pair(n, rnd, k, p, q);
        const double apq = a[p * ld + q];
        const double app = a[p * ld + p], aqq = a[q * ld + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && fabs(apq) > 1e-300 && fabs(apq) > 1e-15 * sqrt(fabs(app) * fabs(aqq))) {
          jacobi_rotation(app, aqq, apq, c, s);
          nrot++;
        }
        cs[k] = c; sn[k] = s; pp[k] = p; qq[k] = q;
      }
      long long t1 = clock64();
      __syncthreads();
      long long t2 = clock64();
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = nt >> 5;
#if VARIANT == 0
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
#elif VARIANT == 2
      // the warp map of VARIANT 0 (warp -> pair k1, lane -> pair k2 / row i),
      // but every operand of the warp's blocks is gathered before the first
      // store, then every eigenvector pair: the tasks of a round touch
      // disjoint entries, so their shared-memory latencies overlap
      {
        constexpr int NK = 2, NI = 3;   // half <= 64 = NK * 32 warps / lanes, n <= 96
        double c1[NK], s1[NK], c2[NK], s2[NK];
        int p1[NK], q1[NK], p2[NK], q2[NK];
#pragma unroll
        for (int u = 0; u < NK; ++u) {
          const int k1 = wid + u * nw, k2 = lane + u * 32;
          const bool v1 = k1 < half, v2 = k2 < half;
          c1[u] = v1 ? cs[k1] : 1.0; s1[u] = v1 ? sn[k1] : 0.0;
          p1[u] = v1 ? pp[k1] : 0;   q1[u] = v1 ? qq[k1] : 0;
          c2[u] = v2 ? cs[k2] : 1.0; s2[u] = v2 ? sn[k2] : 0.0;
          p2[u] = v2 ? pp[k2] : 0;   q2[u] = v2 ? qq[k2] : 0;
        }
        double x11[NK][NK], x12[NK][NK], x21[NK][NK], x22[NK][NK];
#pragma unroll
        for (int u = 0; u < NK; ++u)
#pragma unroll
          for (int w = 0; w < NK; ++w) {
            x11[u][w] = a[p1[u] * ld + p2[w]]; x12[u][w] = a[p1[u] * ld + q2[w]];
            x21[u][w] = a[q1[u] * ld + p2[w]]; x22[u][w] = a[q1[u] * ld + q2[w]];
          }
#pragma unroll
        for (int u = 0; u < NK; ++u)
#pragma unroll
          for (int w = 0; w < NK; ++w) {
            const int k1 = wid + u * nw, k2 = lane + w * 32;
            if (k1 >= half || k2 >= half || (s1[u] == 0.0 && s2[w] == 0.0)) continue;
            const double y11 = c1[u] * x11[u][w] - s1[u] * x21[u][w], y12 = c1[u] * x12[u][w] - s1[u] * x22[u][w];
            const double y21 = s1[u] * x11[u][w] + c1[u] * x21[u][w], y22 = s1[u] * x12[u][w] + c1[u] * x22[u][w];
            a[p1[u] * ld + p2[w]] = c2[w] * y11 - s2[w] * y12;
            a[q1[u] * ld + q2[w]] = s2[w] * y21 + c2[w] * y22;
            a[p1[u] * ld + q2[w]] = (k1 == k2) ? 0.0 : s2[w] * y11 + c2[w] * y12;
            a[q1[u] * ld + p2[w]] = (k1 == k2) ? 0.0 : c2[w] * y21 - s2[w] * y22;
          }
        double qx[NK][NI], qy[NK][NI];
#pragma unroll
        for (int u = 0; u < NK; ++u)
#pragma unroll
          for (int w = 0; w < NI; ++w) {
            const int i = lane + w * 32;
            const bool ok = i < n;
            qx[u][w] = ok ? qv[i * ld + p1[u]] : 0.0;
            qy[u][w] = ok ? qv[i * ld + q1[u]] : 0.0;
          }
#pragma unroll
        for (int u = 0; u < NK; ++u)
#pragma unroll
          for (int w = 0; w < NI; ++w) {
            const int k1 = wid + u * nw, i = lane + w * 32;
            if (k1 >= half || i >= n || s1[u] == 0.0) continue;
            qv[i * ld + p1[u]] = c1[u] * qx[u][w] - s1[u] * qy[u][w];
            qv[i * ld + q1[u]] = s1[u] * qx[u][w] + c1[u] * qy[u][w];
          }
      }
#endif
      long long t3 = clock64();
      __syncthreads();
      long long t4 = clock64();
      t_p1 += t1 - t0; t_b1 += t2 - t1; t_p2 += t3 - t2; t_b2 += t4 - t3;
    }
  }
  if (threadIdx.x == 0) { clk[0] = t_p1; clk[1] = t_b1; clk[2] = t_p2; clk[3] = t_b2; clk[4] = nrot; }
  if (threadIdx.x == 32 * 5) { clk[8] = t_p1; clk[9] = t_b1; clk[10] = t_p2; clk[11] = t_b2; }
  for (int i = threadIdx.x; i < n; i += nt) out[i] = a[i * ld + i];
}

int main() {
  for (int n : {32, 48, 96}) {
    std::vector<double> h(n * n);
    srand(1);
    for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) h[i * n + j] = h[j * n + i] = rand() / (double)RAND_MAX - 0.5;
    double *d, *out; long long* clk;
    cudaMalloc(&d, n * n * 8); cudaMalloc(&out, n * 8); cudaMallocManaged(&clk, 128);
    cudaMemcpy(d, h.data(), n * n * 8, cudaMemcpyHostToDevice);
    size_t smem = (2 * n * (n + 1) + n) * 8 + n * 4 + 64;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int sweeps = 3;
    for (int rep = 0; rep < 2; ++rep) { probe<<<1, 1024, smem>>>(d, n, sweeps, clk, out); cudaDeviceSynchronize(); }
    const double rounds = sweeps * (n - 1.0);
    printf("n %d (%d sweeps, all pairs active): thread 0 per round: params %.0f  wait1 %.0f  update %.0f  wait2 %.0f cycles; warp 5: params %.0f wait1 %.0f update %.0f wait2 %.0f; rotations by thread 0: %lld  err %s",
           n, sweeps, clk[0] / rounds, clk[1] / rounds, clk[2] / rounds, clk[3] / rounds, clk[8] / rounds,
           clk[9] / rounds, clk[10] / rounds, clk[11] / rounds, clk[4], cudaGetErrorString(cudaGetLastError()));
    { std::vector<double> ho(n); cudaMemcpy(ho.data(), out, n * 8, cudaMemcpyDeviceToHost); unsigned long long h = 0; for (int i = 0; i < n; ++i) { unsigned long long b; memcpy(&b, &ho[i], 8); h = h * 1315423911ull + b; } printf("  diag checksum %016llx\n", h); }
  }
  return 0;
}
