// bt200 -- CP-ALS for small ranks (R <= 16) on tensors larger than one SM
// (C4: 255^3, R = 16; decomp.py:344-410).
//
// The general path (cp.cu) is built for R = 64 tiles and spends, at C4's
// size, most of a sweep in launch gaps, split-K reductions and a separate
// explicit-residual pass.  This path runs a sweep as TWO passes over X:
//
//   pass 1  P = X x3 C (I*J x 16, stays in L2) AND the explicit residual
//           ||X - [[A lam, B, C]]||^2 of the factors the previous sweep
//           left, both on DMMA from the same registers: an 8x8 block of X
//           is held as the m8n8k4 A operand with the reduction index
//           permuted (k = 2t + s) so that the same registers are also that
//           block in the accumulator layout, where the model tile
//           (A_i o B_j lam) C^T is subtracted from it;
//           modes 1 and 2 are contractions of P (read from L2);
//   pass 2  the mode-3 MTTKRP, X^T (A o B) on DMMA, row chunks sized so
//           that every SM holds two resident CTAs; chunk partials summed
//           in a fixed order.
//
// Each factor update is ONE one-CTA kernel (F = M pinv(V), Gram, column
// norms, normalised factor; the mode-3 update also lambda, A lam and the
// Gram-identity fit); the R x R pseudo-inverses run on a side stream and
// overlap the passes.  The whole sweep is one CUDA graph.  The fit of sweep
// t is the residual computed by pass 1 of sweep t + 1 (one extra pass 1
// after the last sweep), so "auto" and "explicit" both report the
// reference's explicit fit (decomp.py:395-396); "gram" the Gram identity.
// No floating-point atomics: tiles are handed out by an integer ticket and
// every partial is stored per tile / per chunk and summed in a fixed order.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "bt_common.cuh"

// cp.cu: pinv of g0 o g1 (R <= 16), one warp
int bt_cp_pinv_small(const double* g0, const double* g1, int R, double* vp, double* state,
                     cudaStream_t st);

namespace {

constexpr int NP = 16;    // padded rank
constexpr int LDX = 20;   // C copy read as C[k0 + g][4 s + t]: conflict free for ld == 4 (mod 16)
constexpr int LDP = 18;   // C copy read as C[k0 + 2 t + s][g]: conflict free for 2 ld == 4 (mod 16)
constexpr int UB = 8;     // 8x8 X blocks per register buffer (two buffers: 8-16 loads in flight per lane)

__device__ __forceinline__ double ldg_nc(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// ---------------------------------------------------------------------------
// pass 1: P = X x3 C and (RESID) per-tile sums of (X - Xhat)^2
// ---------------------------------------------------------------------------
template <bool RESID>
__global__ void __launch_bounds__(256, 2)
    mid_pass1_kernel(const double* __restrict__ X, int64_t IJ, int J, int K, int R,
                     const double* __restrict__ W, const double* __restrict__ Bf,
                     const double* __restrict__ Cf, double* __restrict__ P,
                     double* __restrict__ res_part, unsigned* __restrict__ ticket) {
  extern __shared__ __align__(16) double sm[];
  const int Kp = (K + 7) / 8 * 8;
  double* cx = sm;
  double* cp = sm + (int64_t)Kp * LDX;
  // loads batched 8 deep: one global round trip per batch, not per element
  for (int base = threadIdx.x; base < Kp * NP; base += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * blockDim.x;
      const int k = idx / NP, r = idx % NP;
      v[u] = (idx < Kp * NP && k < K && r < R) ? __ldg(Cf + (int64_t)k * R + r) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * blockDim.x;
      if (idx < Kp * NP) {
        const int k = idx / NP, r = idx % NP;
        cx[k * LDX + r] = v[u];
        cp[k * LDP + r] = v[u];
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t ntiles = (IJ + 7) / 8;
  const int nkb = Kp / 8;
  const bool wide = R > 8;
  // the ticket of the NEXT tile is drawn while the current one is processed
  // (a global atomic round trip per tile otherwise)
  unsigned tk = 0;
  if (lane == 0) tk = atomicAdd(ticket, 1u);
  for (;;) {
    const int64_t tile = __shfl_sync(0xffffffffu, tk, 0);
    if (tile >= ntiles) break;
    if (lane == 0) tk = atomicAdd(ticket, 1u);
    const int64_t row = tile * 8 + gq;
    const bool valid = row < IJ;
    const double* xr = X + (valid ? row : 0) * K;
    double p00 = 0.0, p01 = 0.0, p10 = 0.0, p11 = 0.0, res = 0.0;
    double xc[UB][2], xn[UB][2];
    auto load = [&](double (&dst)[UB][2], int kb0) {
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int kk = (kb0 + u) * 8 + 2 * tq;
        dst[u][0] = (valid && kk < K) ? __ldg(xr + kk) : 0.0;
        dst[u][1] = (valid && kk + 1 < K) ? __ldg(xr + kk + 1) : 0.0;
      }
    };
    load(xc, 0);
    double wa[4] = {0.0, 0.0, 0.0, 0.0};
    if (RESID && valid) {
      const int64_t i = row / J;
      const int j = static_cast<int>(row - i * J);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int r = 4 * s + tq;
        if (r < R) wa[s] = __ldg(W + i * NP + r) * __ldg(Bf + (int64_t)j * R + r);
      }
    }
    auto compute = [&](const double (&xv)[UB][2], int kb0) {
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (kb0 + u < nkb) {
          const int kbase = (kb0 + u) * 8;
          const double* c0 = cp + (kbase + 2 * tq) * LDP + gq;
          dmma884(p00, p01, xv[u][0], c0[0]);
          dmma884(p00, p01, xv[u][1], c0[LDP]);
          if (wide) {
            dmma884(p10, p11, xv[u][0], c0[8]);
            dmma884(p10, p11, xv[u][1], c0[LDP + 8]);
          }
          if (RESID) {
            const double* c1 = cx + (kbase + gq) * LDX + tq;
            double d0 = 0.0, d1 = 0.0;
            dmma884(d0, d1, wa[0], c1[0]);
            dmma884(d0, d1, wa[1], c1[4]);
            if (wide) {
              dmma884(d0, d1, wa[2], c1[8]);
              dmma884(d0, d1, wa[3], c1[12]);
            }
            const double e0 = xv[u][0] - d0, e1 = xv[u][1] - d1;
            res = fma(e0, e0, res);
            res = fma(e1, e1, res);
          }
        }
      }
    };
    // ping-pong register buffers: UB blocks (2 UB loads per lane) always in flight
    for (int kb0 = 0; kb0 < nkb; kb0 += 2 * UB) {
      if (kb0 + UB < nkb) load(xn, kb0 + UB);
      compute(xc, kb0);
      if (kb0 + 2 * UB < nkb) load(xc, kb0 + 2 * UB);
      if (kb0 + UB < nkb) compute(xn, kb0 + UB);
    }
    if (valid) {
      double* pr = P + row * NP;
      *reinterpret_cast<double2*>(pr + 2 * tq) = make_double2(p00, p01);
      *reinterpret_cast<double2*>(pr + 8 + 2 * tq) = make_double2(p10, p11);
    }
    if (RESID) {
      res = warp_sum(res);
      if (lane == 0) res_part[tile] = res;
    }
  }
}

// ---------------------------------------------------------------------------
// out[a][r] = sum_b src[(a sa + b sb) NP + r] * (F ? F[b][r] : 1), fixed order
// (mode 1 / mode 2 from P; the chunk sum of the mode-3 partials)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    mid_contract_kernel(const double* __restrict__ src, int64_t sa, int64_t sb, int nb,
                        const double* __restrict__ F, int R, double* __restrict__ out) {
  __shared__ double red[16][NP];
  const int r = threadIdx.x & 15, bc = threadIdx.x >> 4;
  const int64_t a = blockIdx.x;
  const double* s = src + a * sa * NP + r;
  double acc = 0.0;
  // loads batched 8 deep (independent), sums in the fixed b order
  if (F != nullptr) {
    if (r < R) {
      int b = bc;
      for (; b + 7 * 16 < nb; b += 8 * 16) {
        double v[8], f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u] = s[(int64_t)(b + 16 * u) * sb * NP];
          f[u] = F[(int64_t)(b + 16 * u) * R + r];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(v[u], f[u], acc);
      }
      for (; b < nb; b += 16) acc = fma(s[(int64_t)b * sb * NP], F[(int64_t)b * R + r], acc);
    }
  } else {
    int b = bc;
    for (; b + 7 * 16 < nb; b += 8 * 16) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = s[(int64_t)(b + 16 * u) * sb * NP];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; b < nb; b += 16) acc += s[(int64_t)b * sb * NP];
  }
  red[bc][r] = acc;
  __syncthreads();
  if (threadIdx.x < NP) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) t += red[q][threadIdx.x];
    out[a * NP + threadIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// pass 2: mode-3 MTTKRP partials, part[chunk][k][r] = sum over the chunk's
// (i, j) rows of X[ij][k] A[i][r] B[j][r]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 2)
    mid_mode3_kernel(const double* __restrict__ X, int64_t IJ, int J, int K, int R,
                     const double* __restrict__ Af, const double* __restrict__ Bf, int rpc,
                     double* __restrict__ part) {
  extern __shared__ __align__(16) double sm[];
  double* wb = sm;   // rpc4 x LDX; reused for the row-half partials (4 x 32 x 33)
  const int rpc4 = (rpc + 7) / 8 * 8;
  const int64_t rbeg = (int64_t)blockIdx.x * rpc;
  const int64_t rend = rbeg + rpc < IJ ? rbeg + rpc : IJ;
  for (int base = threadIdx.x; base < rpc4 * NP; base += 8 * blockDim.x) {
    double va[8], vb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * blockDim.x;
      const int rr = idx / NP, r = idx % NP;
      const int64_t row = rbeg + rr;
      va[u] = vb[u] = 0.0;
      if (idx < rpc4 * NP && row < rend && r < R) {
        const int64_t i = row / J;
        const int64_t j = row - i * J;
        va[u] = __ldg(Af + i * R + r);
        vb[u] = __ldg(Bf + j * R + r);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = base + u * blockDim.x;
      if (idx < rpc4 * NP) wb[(idx / NP) * LDX + idx % NP] = va[u] * vb[u];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int kg = warp & 3, rh = warp >> 2;
  const int k0 = blockIdx.y * 256 + kg * 64;
  const bool active = k0 < K;
  const bool wide = R > 8;
  double acc[8][2][2];
#pragma unroll
  for (int m = 0; m < 8; ++m) acc[m][0][0] = acc[m][0][1] = acc[m][1][0] = acc[m][1][1] = 0.0;
  if (active) {
    const int nsteps = rpc4 / 4;   // even
    double xc[8], xn[8];
    auto load = [&](double (&dst)[8], int st) {
      const int64_t row = rbeg + st * 4 + tq;
      const bool valid = row < rend;
      const double* xr = X + (valid ? row : 0) * K + k0 + gq;
#pragma unroll
      for (int m = 0; m < 8; ++m) dst[m] = (valid && k0 + 8 * m + gq < K) ? ldg_nc(xr + 8 * m) : 0.0;
    };
    auto compute = [&](const double (&xv)[8], int st) {
      const double* w0 = wb + (st * 4 + tq) * LDX + gq;
      const double b0 = w0[0], b1 = w0[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        dmma884(acc[m][0][0], acc[m][0][1], xv[m], b0);
        if (wide) dmma884(acc[m][1][0], acc[m][1][1], xv[m], b1);
      }
    };
    load(xc, rh);
    for (int st = rh; st < nsteps; st += 4) {
      if (st + 2 < nsteps) load(xn, st + 2);
      compute(xc, st);
      if (st + 4 < nsteps) load(xc, st + 4);
      if (st + 2 < nsteps) compute(xn, st + 2);
    }
  }
  __syncthreads();
  double* hp = sm + (kg * 32 + lane) * 33;
  if (active && rh == 1) {
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      hp[m * 4 + 0] = acc[m][0][0];
      hp[m * 4 + 1] = acc[m][0][1];
      hp[m * 4 + 2] = acc[m][1][0];
      hp[m * 4 + 3] = acc[m][1][1];
    }
  }
  __syncthreads();
  if (active && rh == 0) {
    double* out = part + (int64_t)blockIdx.x * K * NP;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int k = k0 + 8 * m + gq;
      if (k < K) {
        double* o = out + (int64_t)k * NP;
        *reinterpret_cast<double2*>(o + 2 * tq) =
            make_double2(acc[m][0][0] + hp[m * 4 + 0], acc[m][0][1] + hp[m * 4 + 1]);
        *reinterpret_cast<double2*>(o + 8 + 2 * tq) =
            make_double2(acc[m][1][0] + hp[m * 4 + 2], acc[m][1][1] + hp[m * 4 + 3]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// factor update (one CTA): F_un = M Vp, Gram, column norms (0 -> 1),
// normalised factor and Gram; the mode-3 update also sets lambda, W = A lam
// and the Gram-identity fit (decomp.py:386-393)
// ---------------------------------------------------------------------------
struct MidFit {
  const double* g0;     // normalised Grams of the other two modes
  const double* g1;
  const double* a;      // I x R (mode-1 factor) -> W
  double* w;            // I x NP
  double* lam;          // R
  double* fit_hist;
  const int* iter;
  double x2;
  int I;
  int gram_fit;         // write the Gram-identity fit into fit_hist[*iter]
  unsigned* ticket;     // pass-1 tile ticket, reset here (a memset node costs a ~4 us gap)
};

__device__ long long g_mid_clk[12];  // phase clocks of the last solve (diagnostics)

// F_un = M Vp and the Gram F_un^T F_un both on DMMA: the scalar version was
// bound by its shared-memory loads (two 8-byte LDS per DFMA, 12 us per
// update).  Fragment reads are conflict free at leading dimension 20.
constexpr int LDF = 20;
constexpr int GW = 16;   // warps forming Gram partials

__global__ void __launch_bounds__(1024)
    mid_solve_kernel(const double* __restrict__ M, const double* __restrict__ Vp, int rows, int R,
                     double* __restrict__ F, double* __restrict__ G, int mode3, MidFit fit) {
  extern __shared__ __align__(16) double sm[];
  const int rows8 = (rows + 7) / 8 * 8;
  double* fs = sm;                                // rows8 x LDF
  double* ms = sm + (int64_t)rows8 * LDF;         // rows8 x LDF
  __shared__ double vs[NP * LDF], gw[GW][NP * NP], gun[NP * NP], nrm[NP], red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  int ck = 0;
#define MID_CLK() do { if (tid == 0) g_mid_clk[ck] = clock64(); ++ck; } while (0)
  MID_CLK();
  for (int e = tid; e < NP * NP; e += blockDim.x) {
    const int q = e / NP, c = e % NP;
    vs[q * LDF + c] = (q < R && c < R) ? Vp[q * R + c] : 0.0;
  }
  for (int e = tid; e < rows8 * NP; e += blockDim.x)
    ms[(e / NP) * LDF + e % NP] = e < rows * NP ? M[e] : 0.0;
  __syncthreads();
  MID_CLK();
  for (int mt = warp; mt * 8 < rows; mt += 32) {
    const double* mr = ms + (mt * 8 + gq) * LDF + tq;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4) {
      const double av = mr[4 * s4];
      const double* vr = vs + (4 * s4 + tq) * LDF + gq;
      dmma884(c00, c01, av, vr[0]);
      dmma884(c10, c11, av, vr[8]);
    }
    double* fr = fs + (mt * 8 + gq) * LDF;
    fr[2 * tq] = c00;
    fr[2 * tq + 1] = c01;
    fr[8 + 2 * tq] = c10;
    fr[9 + 2 * tq] = c11;
  }
  __syncthreads();
  MID_CLK();
  if (warp < GW) {
    double g00a = 0.0, g00b = 0.0, g01a = 0.0, g01b = 0.0, g10a = 0.0, g10b = 0.0, g11a = 0.0, g11b = 0.0;
    for (int ks = warp; ks * 4 < rows8; ks += GW) {
      const double* fr = fs + (ks * 4 + tq) * LDF + gq;
      const double a0 = fr[0], a1 = fr[8];
      dmma884(g00a, g00b, a0, a0);
      dmma884(g01a, g01b, a0, a1);
      dmma884(g10a, g10b, a1, a0);
      dmma884(g11a, g11b, a1, a1);
    }
    double* o = gw[warp];
    o[gq * NP + 2 * tq] = g00a;
    o[gq * NP + 2 * tq + 1] = g00b;
    o[gq * NP + 8 + 2 * tq] = g01a;
    o[gq * NP + 9 + 2 * tq] = g01b;
    o[(8 + gq) * NP + 2 * tq] = g10a;
    o[(8 + gq) * NP + 2 * tq + 1] = g10b;
    o[(8 + gq) * NP + 8 + 2 * tq] = g11a;
    o[(8 + gq) * NP + 9 + 2 * tq] = g11b;
  }
  double inner = 0.0;
  if (mode3) {
    double s = 0.0;
    for (int e = tid; e < rows * NP; e += blockDim.x) {
      const int row = e / NP, c = e % NP;
      s = fma(fs[row * LDF + c], ms[row * LDF + c], s);   // padded columns are zero
    }
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
  }
  __syncthreads();
  MID_CLK();
  if (tid < NP * NP) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < GW; ++w) t += gw[w][tid];
    gun[tid] = t;
  }
  if (mode3 && tid < 32) {
    const double t = warp_sum(red[tid]);
    if (tid == 0) red[0] = t;
  }
  __syncthreads();
  MID_CLK();
  inner = red[0];
  if (tid < NP) {
    double v = sqrt(gun[tid * NP + tid]);
    if (v == 0.0 || tid >= R) v = 1.0;
    nrm[tid] = v;
  }
  __syncthreads();
  MID_CLK();
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int a = e / R, b = e % R;
    G[e] = gun[a * NP + b] / (nrm[a] * nrm[b]);
  }
  for (int e = tid; e < rows * R; e += blockDim.x) {
    const int row = e / R, c = e % R;
    F[e] = fs[row * LDF + c] / nrm[c];
  }
  MID_CLK();
  if (!mode3) return;
  for (int r = tid; r < R; r += blockDim.x) fit.lam[r] = nrm[r];
  if (tid == 0) *fit.ticket = 0u;
  for (int e = tid; e < fit.I * NP; e += blockDim.x) {
    const int i = e / NP, r = e % NP;
    fit.w[e] = r < R ? fit.a[(int64_t)i * R + r] * nrm[r] : 0.0;
  }
  __syncthreads();
  // ||Xhat||^2 = lam^T (G0 o G1 o G2) lam ; <X, Xhat> = sum(C_un o M3)
  double s = 0.0;
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int a = e / R, b = e % R;
    s += nrm[a] * nrm[b] * fit.g0[e] * fit.g1[e] * (gun[a * NP + b] / (nrm[a] * nrm[b]));
  }
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (tid < 32 && fit.gram_fit) {
    const double xh2 = warp_sum(red[tid]);
    if (tid == 0) {
      const double res2 = fmax(fit.x2 - 2.0 * inner + xh2, 0.0);
      fit.fit_hist[*fit.iter] = 1.0 - sqrt(res2 / fit.x2);
    }
  }
#undef MID_CLK
}

// sum of the per-tile residual partials (fixed order), explicit fit, sweep counter
__global__ void __launch_bounds__(1024)
    mid_fit_kernel(const double* __restrict__ res_part, int64_t n, double x2,
                   double* __restrict__ fit_hist, int* __restrict__ iter, int explicit_fit,
                   int* __restrict__ have) {
  __shared__ double red[1024];
  // lagged use (first node of the sweep graph, fit of the PREVIOUS sweep): the
  // first replay has no residual yet
  if (have != nullptr) {
    const int h = *have;
    __syncthreads();
    if (h == 0) {
      if (threadIdx.x == 0) *have = 1;
      return;
    }
  }
  if (explicit_fit) {
    double s = 0.0;
    int64_t k = threadIdx.x;
    for (; k + 7 * 1024 < n; k += 8 * 1024) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = res_part[k + 1024 * u];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; k < n; k += 1024) s += res_part[k];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    if (explicit_fit) fit_hist[*iter] = 1.0 - sqrt(red[0]) / sqrt(x2);
    *iter += 1;
  }
}

__global__ void __launch_bounds__(1024)
    mid_gram_kernel(const double* __restrict__ f, int rows, int R, double* __restrict__ g) {
  extern __shared__ __align__(16) double sm[];   // rows x 17
  __shared__ double part[4][NP * NP];
  for (int e = threadIdx.x; e < rows * R; e += blockDim.x) sm[(e / R) * 17 + e % R] = f[e];
  __syncthreads();
  const int e = threadIdx.x & 255, q = threadIdx.x >> 8;
  const int a = e / NP, b = e % NP;
  double s = 0.0;
  if (a < R && b < R)
    for (int r = q; r < rows; r += 4) s = fma(sm[r * 17 + a], sm[r * 17 + b], s);
  part[q][e] = s;
  __syncthreads();
  if (threadIdx.x < NP * NP && a < R && b < R)
    g[a * R + b] = (part[0][e] + part[1][e]) + (part[2][e] + part[3][e]);
}

// KruskalRep.x = A lam (the first R columns of W)
__global__ void mid_out_kernel(const double* __restrict__ w, int I, int R, double* __restrict__ a) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < I * R; e += gridDim.x * blockDim.x)
    a[e] = w[(e / R) * NP + e % R];
}

struct MidBuf {
  double *P, *part, *M, *res_part, *G[3], *vp[3], *W, *fit_hist;
  int* iter;
  unsigned* ticket;
};

}  // namespace

extern "C" int bt_debug_mid_clocks(long long* out12) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out12, g_mid_clk, sizeof(long long) * 12);
}

namespace {

// The sweep graph of the last call, kept for the next one: a repeated call on
// the same buffers (same X, factor, lambda and scratch addresses, shape, fit
// mode and ||X||) replays it instead of capturing and instantiating again
// (~0.4 ms of host time per call at C4).  Every pointer and scalar baked into
// the graph's kernel arguments is part of the key; the streams and events
// used for capturing live for the process.
struct MidGraphKey {
  const void *x, *a, *b, *c, *lam, *ws;
  int64_t I, J, K, ws_elems;
  int R, explicit_fit, dev, lagged;
  double x2;
  bool operator==(const MidGraphKey& o) const {
    return x == o.x && a == o.a && b == o.b && c == o.c && lam == o.lam && ws == o.ws && I == o.I &&
           J == o.J && K == o.K && ws_elems == o.ws_elems && R == o.R &&
           explicit_fit == o.explicit_fit && dev == o.dev && lagged == o.lagged && x2 == o.x2;
  }
};
struct MidGraphCache {
  std::mutex mu;
  bool valid = false;
  MidGraphKey key{};
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t side = nullptr, cs = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int stream_dev = -1;
  void drop() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    gexec = nullptr;
    graph = nullptr;
    valid = false;
  }
};
MidGraphCache g_mid_cache;

}  // namespace

// Returns 1 when it ran (outputs written, *rc set), 0 when the problem is not eligible.
int bt_cp_mid_try(const bt_cp_problem* pb, double* a, double* b, double* c, double* lam,
                  int max_iters, double tol, int fit_mode, double* fit_history, int* n_iters,
                  int* converged, cudaStream_t st, int* rc) {
  // read per call: the parity tests switch paths in-process
  const bool off = getenv("BT_CP_MID") && getenv("BT_CP_MID")[0] == '0';
  *rc = BT_OK;
  const int64_t I = pb->I, J = pb->J, K = pb->K;
  const int R = static_cast<int>(pb->R);
  if (off || pb->R > NP || R < 1 || I < 1 || J < 1 || K < 1 || I > 576 || J > 576 || K > 512 ||
      I * J < 4096 || pb->norm_x <= 0.0 || max_iters < 1)
    return 0;
  const int64_t IJ = I * J;
  const int nsm = bt_num_sms();
  const int Kp = static_cast<int>((K + 7) / 8 * 8);
  const size_t smem1 = sizeof(double) * Kp * (LDX + LDP);
  const int kspans = static_cast<int>(bt_cdiv(K, 256));
  // row chunks of pass 2: two resident CTAs per SM over all k spans
  // (one CTA slot short of two per SM: the two-CTA register footprint fills an
  // SM, and the one-warp pinv on the side stream needs a slot to overlap)
  const int64_t want_chunks = std::max<int64_t>(1, (2 * nsm - 1) / kspans);
  int rpc = static_cast<int>(bt_cdiv(bt_cdiv(IJ, want_chunks), 8) * 8);
  rpc = std::max(rpc, 64);
  const int64_t nchunks = bt_cdiv(IJ, rpc);
  const size_t smem3 = sizeof(double) * std::max<size_t>((size_t)rpc * LDX, 4 * 32 * 33);
  const int64_t maxrows = std::max(I, std::max(J, K));
  const size_t smem_solve = sizeof(double) * ((maxrows + 7) / 8 * 8) * LDF * 2;
  if (smem1 > 100 * 1024 || smem3 > 100 * 1024 || smem_solve > 184 * 1024 /* + ~38 KB static in mid_solve_kernel */) return 0;
  const int64_t ntiles = bt_cdiv(IJ, 8);
  const bool explicit_fit = fit_mode != 2;

  auto fail = [&](const char* what, cudaError_t e) {
    bt_set_error("cp_als (small-rank path): %s: %s", what, cudaGetErrorString(e));
    *rc = BT_E_CUDA;
    return 1;
  };
  // workspace (doubles)
  int64_t o = 0;
  auto take = [&](int64_t n) {
    const int64_t at = o;
    o += (n + 1) / 2 * 2;
    return at;
  };
  const int64_t oP = take(IJ * NP), oPart = take(nchunks * K * NP), oM = take(maxrows * NP),
                oRes = take(ntiles), oG = take(3 * NP * NP), oVp = take(3 * NP * NP),
                oW = take(I * NP), oHist = take(max_iters + 2), oInt = take(4), oPst = take(4);
  double* ws = nullptr;
  bt_keep_async_pool();
  cudaError_t e = cudaMallocAsync(&ws, sizeof(double) * o, st);
  if (e != cudaSuccess) return fail("workspace", e);
  MidBuf B;
  B.P = ws + oP;
  B.part = ws + oPart;
  B.M = ws + oM;
  B.res_part = ws + oRes;
  for (int k = 0; k < 3; ++k) {
    B.G[k] = ws + oG + k * NP * NP;
    B.vp[k] = ws + oVp + k * NP * NP;
  }
  B.W = ws + oW;
  B.fit_hist = ws + oHist;
  double* pst = ws + oPst;   // per-mode pinv path memory
  B.iter = reinterpret_cast<int*>(ws + oInt);
  B.ticket = reinterpret_cast<unsigned*>(ws + oInt) + 2;

  MidGraphCache& gc = g_mid_cache;
  std::lock_guard<std::mutex> lock(gc.mu);
  int dev = 0;
  cudaGetDevice(&dev);
  // an error path drops the cached graph (it may be half built) and frees the scratch
  auto cleanup = [&]() {
    gc.drop();
    cudaFreeAsync(ws, st);
  };
#define MID_CHECK(x, what)          \
  do {                              \
    cudaError_t e_ = (x);           \
    if (e_ != cudaSuccess) {        \
      cleanup();                    \
      return fail(what, e_);        \
    }                               \
  } while (0)
#define MID_LAUNCH(what)            \
  do {                              \
    bt_count_launch();              \
    MID_CHECK(cudaGetLastError(), what); \
  } while (0)

  MID_CHECK(cudaFuncSetAttribute(mid_pass1_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem1), "pass1 attr");
  MID_CHECK(cudaFuncSetAttribute(mid_pass1_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem1), "pass1 attr");
  MID_CHECK(cudaFuncSetAttribute(mid_mode3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem3), "mode3 attr");
  MID_CHECK(cudaFuncSetAttribute(mid_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_solve), "solve attr");
  MID_CHECK(cudaFuncSetAttribute(mid_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(double) * maxrows * 17)), "gram attr");
  if (gc.stream_dev != dev) {
    gc.drop();
    gc.side = gc.cs = nullptr;       // streams of another device are left to the driver
    gc.ev_fork = gc.ev_join = nullptr;
    MID_CHECK(cudaStreamCreateWithFlags(&gc.side, cudaStreamNonBlocking), "side stream");
    MID_CHECK(cudaStreamCreateWithFlags(&gc.cs, cudaStreamNonBlocking), "capture stream");
    MID_CHECK(cudaEventCreateWithFlags(&gc.ev_fork, cudaEventDisableTiming), "event");
    MID_CHECK(cudaEventCreateWithFlags(&gc.ev_join, cudaEventDisableTiming), "event");
    gc.stream_dev = dev;
  }
  cudaStream_t side = gc.side, cs = gc.cs;
  cudaEvent_t ev_fork = gc.ev_fork, ev_join = gc.ev_join;

  const double x2 = pb->norm_x * pb->norm_x;
  const int grid1 = 2 * nsm - 1;   // one slot left for the concurrent pinv warp
  double* F[3] = {a, b, c};
  const int rows[3] = {(int)I, (int)J, (int)K};

  // head of sweep 1: Grams of the initial factors, pinv for mode 1, P = X x3 C
  MID_CHECK(cudaMemsetAsync(B.iter, 0, 64, st), "memset");
  for (int k = 0; k < 3; ++k) {
    mid_gram_kernel<<<1, 1024, sizeof(double) * rows[k] * 17, st>>>(F[k], rows[k], R, B.G[k]);
    MID_LAUNCH("gram");
  }
  if ((*rc = bt_cp_pinv_small(B.G[1], B.G[2], R, B.vp[0], pst, st)) != BT_OK) {
    cleanup();
    return 1;
  }
  mid_pass1_kernel<false><<<grid1, 256, smem1, st>>>(pb->x, IJ, (int)J, (int)K, R, nullptr, b, c,
                                                     B.P, B.res_part, B.ticket);
  MID_LAUNCH("pass1");

  // the sweep graph: tail of sweep t (three updates) + head of sweep t + 1;
  // replayed from the cache when every baked-in argument is unchanged
  // tol == 0: the fit kernel of a sweep runs as a side branch at the START of
  // the next replay, beside the mode-1 contraction, instead of closing its own
  // replay alone (5 us + a launch gap per sweep); one stand-alone fit follows
  // the last replay.  tol > 0 needs each sweep's fit before the next starts.
  const bool lagged = !(tol > 0.0);
  int* have = B.iter + 1;
  const MidGraphKey key{pb->x, a, b, c, lam, ws, I, J, K, o, R, explicit_fit ? 1 : 0, dev,
                        lagged ? 1 : 0, x2};
  if (!(gc.valid && gc.key == key)) {
  gc.drop();
  MID_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
  int cap_rc = BT_OK;
  cudaError_t cap_e = cudaSuccess;
  auto note = [&]() {
    bt_count_launch();
    const cudaError_t le = cudaGetLastError();
    if (cap_e == cudaSuccess && le != cudaSuccess) cap_e = le;
  };
  auto fork_pinv = [&](int g0, int g1, int dst) {
    if (cap_e == cudaSuccess) cap_e = cudaEventRecord(ev_fork, cs);
    if (cap_e == cudaSuccess) cap_e = cudaStreamWaitEvent(side, ev_fork, 0);
    if (cap_rc == BT_OK) cap_rc = bt_cp_pinv_small(B.G[g0], B.G[g1], R, B.vp[dst], pst + dst, side);
    if (cap_e == cudaSuccess) cap_e = cudaEventRecord(ev_join, side);
  };
  auto join = [&]() {
    if (cap_e == cudaSuccess) cap_e = cudaStreamWaitEvent(cs, ev_join, 0);
  };
  MidFit nofit{};
  if (lagged) {
    if (cap_e == cudaSuccess) cap_e = cudaEventRecord(ev_fork, cs);
    if (cap_e == cudaSuccess) cap_e = cudaStreamWaitEvent(side, ev_fork, 0);
    mid_fit_kernel<<<1, 1024, 0, side>>>(B.res_part, ntiles, x2, B.fit_hist, B.iter,
                                         explicit_fit ? 1 : 0, have);
    note();
    // joined with the mode-2 pinv (same side stream, in order) before pass 1 rewrites the partials
  }
  // mode 1 (its pinv was forked by the previous sweep / the head above)
  mid_contract_kernel<<<(unsigned)I, 256, 0, cs>>>(B.P, J, 1, (int)J, b, R, B.M);
  note();
  mid_solve_kernel<<<1, 1024, smem_solve, cs>>>(B.M, B.vp[0], (int)I, R, a, B.G[0], 0, nofit);
  note();
  // mode 2
  fork_pinv(0, 2, 1);
  mid_contract_kernel<<<(unsigned)J, 256, 0, cs>>>(B.P, 1, J, (int)I, a, R, B.M);
  note();
  join();
  mid_solve_kernel<<<1, 1024, smem_solve, cs>>>(B.M, B.vp[1], (int)J, R, b, B.G[1], 0, nofit);
  note();
  // mode 3
  fork_pinv(0, 1, 2);
  mid_mode3_kernel<<<dim3((unsigned)nchunks, (unsigned)kspans), 256, smem3, cs>>>(
      pb->x, IJ, (int)J, (int)K, R, a, b, rpc, B.part);
  note();
  mid_contract_kernel<<<(unsigned)K, 256, 0, cs>>>(B.part, 1, K, (int)nchunks, nullptr, R, B.M);
  note();
  join();
  MidFit fit{B.G[0], B.G[1], a, B.W, lam, B.fit_hist, B.iter, x2, (int)I, explicit_fit ? 0 : 1, B.ticket};
  mid_solve_kernel<<<1, 1024, smem_solve, cs>>>(B.M, B.vp[2], (int)K, R, c, B.G[2], 1, fit);
  note();
  // head of the next sweep: pinv for mode 1, P and this sweep's residual
  fork_pinv(1, 2, 0);
  if (explicit_fit)
    mid_pass1_kernel<true><<<grid1, 256, smem1, cs>>>(pb->x, IJ, (int)J, (int)K, R, B.W, b, c, B.P,
                                                      B.res_part, B.ticket);
  else
    mid_pass1_kernel<false><<<grid1, 256, smem1, cs>>>(pb->x, IJ, (int)J, (int)K, R, nullptr, b, c,
                                                       B.P, B.res_part, B.ticket);
  note();
  if (!lagged) {
    mid_fit_kernel<<<1, 1024, 0, cs>>>(B.res_part, ntiles, x2, B.fit_hist, B.iter, explicit_fit ? 1 : 0,
                                       nullptr);
    note();
  }
  join();
  const cudaError_t end_e = cudaStreamEndCapture(cs, &gc.graph);
  if (cap_rc != BT_OK || cap_e != cudaSuccess || end_e != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    if (cap_rc != BT_OK) {
      *rc = cap_rc;
      return 1;
    }
    return fail("sweep graph capture", cap_e != cudaSuccess ? cap_e : end_e);
  }
  MID_CHECK(cudaGraphInstantiate(&gc.gexec, gc.graph, 0), "graph instantiate");
  gc.key = key;
  gc.valid = true;
  }

  int it = 0, conv = 0;
  double prev = -INFINITY;
  for (it = 1; it <= max_iters; ++it) {
    MID_CHECK(cudaGraphLaunch(gc.gexec, st), "graph launch");
    if (tol > 0.0) {
      double fitv = 0.0;
      MID_CHECK(cudaMemcpyAsync(&fitv, B.fit_hist + (it - 1), sizeof(double), cudaMemcpyDeviceToHost, st),
                "fit read");
      MID_CHECK(cudaStreamSynchronize(st), "sync");
      if (std::fabs(fitv - prev) < tol) {
        conv = 1;
        break;
      }
      prev = fitv;
    }
  }
  if (it > max_iters) it = max_iters;
  if (lagged) {
    mid_fit_kernel<<<1, 1024, 0, st>>>(B.res_part, ntiles, x2, B.fit_hist, B.iter, explicit_fit ? 1 : 0,
                                       have);
    MID_LAUNCH("fit");
  }
  mid_out_kernel<<<(unsigned)std::min<int64_t>(bt_cdiv(I * R, 256), 1024), 256, 0, st>>>(B.W, (int)I, R, a);
  MID_LAUNCH("output");
  if (fit_history)
    MID_CHECK(cudaMemcpyAsync(fit_history, B.fit_hist, sizeof(double) * it, cudaMemcpyDeviceToHost, st),
              "history read");
  MID_CHECK(cudaStreamSynchronize(st), "sync");
  *n_iters = it;
  *converged = conv;
  cudaFreeAsync(ws, st);   // the cached graph is only replayed if the next call gets this block again
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail("sync", e);
#undef MID_CHECK
#undef MID_LAUNCH
  return 1;
}
