// K3: weighted-tensor builders for the BASELINE configs.
//
//   hankel   : apps.py:193-201   t[a,k,b] = sqrt(eta_k) h_k[a,b]          (bit-exact)
//   gneiting : psd.py:172-174 + the C3 kernel: t[i,k,j] = sqrt(eta_k) C_k[i,j]
//   psf      : multilevel.py:296-297 generalised to an image grid != K  (bit-exact)
//   cp_model : C5, [[A0,B0,C0]] + noise * Philox4x32-10 Box-Muller normals,
//              index addressable so CPU slabs regenerate the same entries.
// All are single-pass HBM writers (plus one DMMA GEMM for the CP model).
#include <algorithm>

#include "gemm.cuh"

namespace {

__global__ void hankel_kernel(const double* __restrict__ params, int64_t p, int64_t dout,
                              int64_t din, const int64_t* __restrict__ eta,
                              double* __restrict__ t) {
  const int64_t total = dout * p * din;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx % din;
    const int64_t k = (idx / din) % p;
    const int64_t a = idx / (din * p);
    t[idx] = params[(k * dout + a) * din + b] * sqrt(static_cast<double>(eta[k]));
  }
}

// one CTA row-slab: t[i, k, :] for fixed (i, k)
__global__ void __launch_bounds__(256)
    gneiting_kernel(const double* __restrict__ pts, int64_t npts, int64_t lags, double lag_scale,
                    const int64_t* __restrict__ eta, double* __restrict__ t) {
  const int64_t rows = npts * lags;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t i = row / lags, k = row % lags;
    const double u = static_cast<double>(k) / lag_scale;
    const double up1 = u + 1.0;
    const double p4 = pow(up1, 0.25);
    const double w = sqrt(static_cast<double>(eta[k]));
    const double xi = pts[2 * i], yi = pts[2 * i + 1];
    double* out = t + row * npts;
    for (int64_t j = threadIdx.x; j < npts; j += blockDim.x) {
      const double dx = xi - pts[2 * j], dy = yi - pts[2 * j + 1];
      const double h = sqrt(dx * dx + dy * dy);
      st_stream(out + j, (exp(-10.0 * h / p4) / up1) * w);
    }
  }
}

__global__ void psf_kernel(const double* __restrict__ psf, int64_t k, int64_t grid,
                           double* __restrict__ x) {
  const int64_t total = k * k * k;
  const int64_t h = (k - 1) / 2;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i3 = idx % k, i2 = (idx / k) % k, i1 = idx / (k * k);
    const int64_t e1 = grid - (i1 > h ? i1 - h : h - i1);
    const int64_t e2 = grid - (i2 > h ? i2 - h : h - i2);
    const int64_t e3 = grid - (i3 > h ? i3 - h : h - i3);
    const double w = sqrt(static_cast<double>(e1 * e2 * e3));
    x[idx] = w * psf[(i3 * k + i2) * k + i1];
  }
}

// Philox4x32-10; counter (lo, hi, 0, 0), key (key, 0)
__device__ __forceinline__ void philox(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                      uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
    c1 = static_cast<uint32_t>(p1);
    c3 = static_cast<uint32_t>(p0);
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__device__ __forceinline__ double philox_normal(uint64_t idx, uint64_t key) {
  uint32_t c0 = static_cast<uint32_t>(idx), c1 = static_cast<uint32_t>(idx >> 32), c2 = 0, c3 = 0;
  philox(c0, c1, c2, c3, static_cast<uint32_t>(key), 0u);
  const double u1 = (static_cast<double>(c0) + 1.0) * 0x1p-32;
  const double u2 = (static_cast<double>(c1) + 0.5) * 0x1p-32;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

// X_i[j][k] = sum_r B0[j][r] (C0[k][r] A0[i][r]) + noise(lin)
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS)
    cp_model_kernel(BtGemmArgs g, int64_t i0, int64_t J, int64_t KK, int64_t Kfull, int64_t k0,
                    double noise, uint64_t key, double* __restrict__ x) {
  extern __shared__ __align__(16) double smem_dyn[];
  const int64_t tm = blockIdx.x, tn = blockIdx.y, b = blockIdx.z;
  const int64_t m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;
  const int64_t KT = (g.Kin + Cfg::BK - 1) / Cfg::BK;
  double acc[Cfg::FM][Cfg::FN][2];
  bt_gemm_mainloop<Cfg>(g, b, m0, n0, 0, KT, acc, smem_dyn);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WM) * Cfg::TM;
  const int wn0 = (warp / Cfg::WM) * Cfg::TN;
  const int64_t i = i0 + b;
  double* xi = x + b * J * KK;
#pragma unroll
  for (int fi = 0; fi < Cfg::FM; ++fi) {
    const int64_t j = m0 + wm0 + fi * 8 + gq;
    if (j >= J) continue;
#pragma unroll
    for (int fj = 0; fj < Cfg::FN; ++fj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t k = n0 + wn0 + fj * 8 + 2 * tq + h;
        if (k >= KK) continue;
        const uint64_t lin = static_cast<uint64_t>((i * J + j) * Kfull + k0 + k);
        double v = acc[fi][fj][h];
        if (noise != 0.0) v += noise * philox_normal(lin, key);
        xi[j * KK + k] = v;
      }
  }
}

template <int V>
using ModelCfg = GemmCfg<128, 64, 16, 4, 2, 3, true, true, V>;

int grid1d(int64_t n) { return static_cast<int>(std::min<int64_t>(bt_cdiv(n, 256), 8192)); }

}  // namespace

extern "C" int bt_build_hankel_f64(const double* params, int64_t p, int64_t d_out, int64_t d_in,
                                   const int64_t* eta, double* t, void* stream) {
  BT_NVTX("bt_build_hankel_f64");
  BT_REQUIRE(p >= 1 && d_out >= 1 && d_in >= 1, BT_E_SHAPE, "hankel: empty input");
  hankel_kernel<<<grid1d(p * d_out * d_in), 256, 0, bt_stream(stream)>>>(params, p, d_out, d_in,
                                                                         eta, t);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

extern "C" int bt_build_gneiting_f64(const double* points, int64_t npts, int64_t lags,
                                     double lag_scale, const int64_t* eta, double* t,
                                     void* stream) {
  BT_NVTX("bt_build_gneiting_f64");
  BT_REQUIRE(npts >= 1 && lags >= 1 && lag_scale > 0, BT_E_SHAPE, "gneiting: bad extents");
  const int grid = static_cast<int>(std::min<int64_t>(npts * lags, 148 * 32));
  gneiting_kernel<<<grid, 256, 0, bt_stream(stream)>>>(points, npts, lags, lag_scale, eta, t);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

extern "C" int bt_build_psf_f64(const double* psf, int64_t k, int64_t grid, double* x,
                                void* stream) {
  BT_NVTX("bt_build_psf_f64");
  BT_REQUIRE(k >= 1 && (k % 2) == 1, BT_E_SHAPE, "psf extent K must be odd");
  BT_REQUIRE(grid >= (k + 1) / 2, BT_E_SHAPE, "psf: image grid smaller than the kernel radius");
  psf_kernel<<<grid1d(k * k * k), 256, 0, bt_stream(stream)>>>(psf, k, grid, x);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

template <int V>
static int run_model(const double* a0, const double* b0, const double* c0, int64_t I, int64_t J,
                     int64_t K, int64_t R, int64_t k0, int64_t k1, double noise, uint64_t key,
                     double* x, cudaStream_t st) {
  using Cfg = ModelCfg<V>;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(cp_model_kernel<Cfg>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES));
    attr = true;
  }
  const int64_t kk = k1 - k0;
  // X_i = (B0 diag(A0[i])) C0^T : A operand B0 scaled along r by A0[i]
  BtGemmArgs g{};
  g.M = J;
  g.N = kk;
  g.Kin = R;
  g.Kout = 1;
  g.A = BtOperand{b0, R, 0, 1, 0};
  g.B = BtOperand{c0 + k0 * R, R, 0, 1, 0};
  g.ascale = a0;
  g.s_ascale_b = R;
  g.alpha = 1.0;
  for (int64_t i0 = 0; i0 < I; i0 += 65535) {
    const int64_t ni = std::min<int64_t>(65535, I - i0);
    BtGemmArgs gi = g;
    gi.ascale = a0 + i0 * R;
    dim3 grid(static_cast<unsigned>(bt_cdiv(J, Cfg::BM)), static_cast<unsigned>(bt_cdiv(kk, Cfg::BN)),
              static_cast<unsigned>(ni));
    cp_model_kernel<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(gi, i0, J, kk, K, k0, noise,
                                                                      key, x + i0 * J * kk);
    BT_LAUNCH_CHECK();
  }
  return BT_OK;
}

extern "C" int bt_build_cp_model_f64(const double* a0, const double* b0, const double* c0,
                                     int64_t I, int64_t J, int64_t K, int64_t R, int64_t k0,
                                     int64_t k1, double noise, uint64_t key, double* x, void* ws,
                                     int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_build_cp_model_f64");
  BT_REQUIRE(I >= 1 && J >= 1 && K >= 1 && R >= 1 && 0 <= k0 && k0 < k1 && k1 <= K, BT_E_SHAPE,
             "cp_model: bad extents");
  (void)ws;
  (void)ws_bytes;
  cudaStream_t st = bt_stream(stream);
  if (R % 2 == 0) return run_model<2>(a0, b0, c0, I, J, K, R, k0, k1, noise, key, x, st);
  return run_model<1>(a0, b0, c0, I, J, K, R, k0, k1, noise, key, x, st);
}

// out[i] = Philox4x32-10 / Box-Muller normal of index i under `key`: the
// deterministic Gaussian blocks of the eigensolver (subspace starts,
// orthonormal completion), generated on the device.
__global__ void bt_fill_normal_kernel(double* __restrict__ out, int64_t n, uint64_t key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = philox_normal(static_cast<uint64_t>(i), key);
}

extern "C" int bt_fill_normal_f64(double* out, int64_t n, uint64_t key, void* stream) {
  if (n <= 0) return BT_OK;
  const int64_t blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
  bt_fill_normal_kernel<<<static_cast<int>(blocks), 256, 0, bt_stream(stream)>>>(out, n, key);
  BT_LAUNCH_CHECK();
  return BT_OK;
}
