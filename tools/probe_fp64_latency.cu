// Dependent-issue latency of DFMA / DMUL / DADD / SHFL+DADD / LDS chains on one warp
// and the cost of a 16- / 32-warp __syncthreads (cycles, clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[64];
  double x = x0, y = 1.000000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 << (i % 5));
  long long t4 = clock64();
  sm[threadIdx.x & 63] = x;
  __syncthreads();
  int idx = threadIdx.x & 31;
  for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = (int)(v * 0.0) + ((idx + 1) & 31); x += v; }
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 3.0);
  long long t7 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 3.0);
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7;
  }
  out[threadIdx.x] = x;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8 * 1024); cudaMallocManaged(&cyc, 64);
  const int n = 4096;
  const char* names[8] = {"DFMA", "DMUL", "DADD", "SHFL+DADD", "LDS+dep", "__syncthreads", "IEEE div", "IEEE sqrt"};
  for (int threads : {32, 512, 1024}) {
    lat<<<1, threads>>>(out, cyc, 1.0, n); cudaDeviceSynchronize();
    lat<<<1, threads>>>(out, cyc, 1.0, n); cudaDeviceSynchronize();
    printf("threads %d:", threads);
    for (int k = 0; k < 8; ++k) printf(" %s %.1f", names[k], (double)cyc[k] / n);
    printf(" cycles/op\n");
  }
  return 0;
}
