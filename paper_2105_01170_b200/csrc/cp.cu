// K4-K6: CP-ALS (decomp.py:344-410) device resident.
//
// Per sweep the reference builds three Khatri-Rao matrices and multiplies
// three unfolding copies (decomp.py:373, 385-387), then reconstructs the
// whole tensor for the fit (decomp.py:395-396).  Here, over ONE C-order
// layout of X (no unfoldings):
//   P      = X x_3 C                    (DMMA GEMM, IJ x K x R; dimension tree)
//   M1     = sum_j P[i,j,:] * B[j,:]    (fused epilogue of the P kernel)
//   M2     = sum_i P[i,j,:] * A[i,:]    (HBM stream over P, new A)
//   M3     = X_(3) (B kr A)             (DMMA GEMM, Khatri-Rao generated on the
//                                         fly as a per-i column scale of B)
// and after each MTTKRP the R x R solve of decomp.py:386-393 runs on chip:
// pinv(G_a o G_b) by a cyclic Jacobi eigensolver in one CTA (numpy's pinv
// cutoff 1e-15 * max|eig|), F = M pinv(V), column norms, lambda, Grams.
// The fit uses the Gram identity ||X||^2 - 2<X,Xhat> + ||Xhat||^2 (exact
// algebra, no extra pass) and switches to an explicit fused residual pass
// (DMMA reconstruction tile - X tile) when the identity would lose digits.
// Every reduction is a fixed-order tree: results are bit-reproducible.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cmath>
#include <vector>

#include <cooperative_groups.h>

#include "gemm.cuh"
#include "jacobi.cuh"
#include "tma.cuh"

int bt_gemm_run(BtGemmArgs g, int64_t batch, cudaStream_t st, int want_splits, int64_t ws_elems);
int bt_gemm_at_tma(const double* a, int64_t lda, int64_t sAb, const double* b, int64_t ldb, double* c,
                   int64_t ldc, int64_t sCb, int64_t M, int64_t N, int64_t Kdim, int64_t batch,
                   cudaStream_t st);
// BT_GEMM_TMA=0: the Q-tree GEMMs on the cp.async engine (A/B runs)
static bool use_at_tma() {
  static const int v = [] {
    const char* e = getenv("BT_GEMM_TMA");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v != 0;
}
extern "C" const char* bt_last_error(void);
int64_t bt_gemm_ws_elems(BtGemmArgs g, int64_t batch);

namespace {

constexpr int PINV_MAX_R = 96;

// ---------------------------------------------------------------------------
// P = X x_3 C with the mode-1 MTTKRP reduction fused into the epilogue
// ---------------------------------------------------------------------------

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS)
    tree_p_kernel(BtGemmArgs g, const double* __restrict__ Bf, int64_t R, double* __restrict__ m1part,
                  int64_t jtiles, int store_p) {
  extern __shared__ __align__(16) double smem_dyn[];
  __shared__ double red[Cfg::WM][Cfg::BN];
  const int64_t tm = blockIdx.x;  // j-tile
  const int64_t tn = blockIdx.y;  // r-tile
  const int64_t i = blockIdx.z;   // batch = mode-1 index
  const int64_t m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;
  const int64_t KT = (g.Kin + Cfg::BK - 1) / Cfg::BK;
  double acc[Cfg::FM][Cfg::FN][2];
  bt_gemm_mainloop<Cfg>(g, i, m0, n0, 0, KT, acc, smem_dyn);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wmi = warp % Cfg::WM;
  const int wm0 = wmi * Cfg::TM;
  const int wn0 = (warp / Cfg::WM) * Cfg::TN;
  double* Pb = g.C + i * g.sCb;
  double colsum[Cfg::FN][2];
#pragma unroll
  for (int j = 0; j < Cfg::FN; ++j) colsum[j][0] = colsum[j][1] = 0.0;
#pragma unroll
  for (int fi = 0; fi < Cfg::FM; ++fi) {
    const int64_t jrow = m0 + wm0 + fi * 8 + gq;
    const bool rv = jrow < g.M;
#pragma unroll
    for (int fj = 0; fj < Cfg::FN; ++fj) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = n0 + wn0 + fj * 8 + 2 * tq + h;
        if (rv && r < g.N) {
          const double v = acc[fi][fj][h];
          if (store_p) Pb[jrow * g.sCm + r] = v;
          colsum[fj][h] = fma(v, __ldg(Bf + jrow * R + r), colsum[fj][h]);
        }
      }
    }
  }
  // reduce over the 8 row-groups of the warp (lane bits 2..4)
#pragma unroll
  for (int fj = 0; fj < Cfg::FN; ++fj)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double v = colsum[fj][h];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      colsum[fj][h] = v;
    }
  if (gq == 0) {
#pragma unroll
    for (int fj = 0; fj < Cfg::FN; ++fj)
#pragma unroll
      for (int h = 0; h < 2; ++h) red[wmi][wn0 + fj * 8 + 2 * tq + h] = colsum[fj][h];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < Cfg::BN; c += Cfg::THREADS) {
    const int64_t r = n0 + c;
    if (r >= g.N) continue;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < Cfg::WM; ++w) s += red[w][c];
    m1part[(i * jtiles + tm) * R + r] = s;
  }
}

// Warp-specialised variant of the tree kernel: Cfg::THREADS consumer threads
// (the DMMA warps) plus one producer warp that streams the X / C tiles with
// cp.async into the STAGES ring; full / empty mbarriers replace the per-stage
// CTA barrier, and the consumers carry no copy-address state (fewer
// registers, no cp.async issue between their DMMAs).  Same math, same
// epilogue, same summation order as tree_p_kernel.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS + 32, 2)
    tree_p_ws_kernel(BtGemmArgs g, const double* __restrict__ Bf, int64_t R,
                     double* __restrict__ m1part, int64_t jtiles, int store_p) {
  static_assert(Cfg::A_KCONTIG && !Cfg::B_KCONTIG, "tree layout: X rows K-contiguous, C N-contiguous");
  extern __shared__ __align__(16) double smem_dyn[];
  __shared__ double red[Cfg::WM][Cfg::BN];
  __shared__ __align__(8) uint64_t full[Cfg::STAGES], empty[Cfg::STAGES];
  const int64_t tm = blockIdx.x, tn = blockIdx.y, i = blockIdx.z;
  const int64_t m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;
  const int64_t KT = (g.Kin + Cfg::BK - 1) / Cfg::BK;
  double* As = smem_dyn;
  double* Bs = smem_dyn + Cfg::STAGES * Cfg::A_STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CW = Cfg::THREADS / 32;  // consumer warps
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], CW);
    }
  }
  __syncthreads();
  if (warp == CW) {
    // ---------------- producer warp ----------------
    const double* a_tile = g.A.ptr + i * g.A.s_b + m0 * g.A.s_mn;
    const double* b_tile = g.B.ptr + n0;
    const int64_t m_left = g.M - m0, n_left = g.N - n0;
    constexpr int V = Cfg::VEC;
    constexpr int ACH = Cfg::BK / V;            // chunks per A row
    constexpr int ATOT = Cfg::BM * ACH;
    constexpr int BCH = Cfg::BN / V;            // chunks per B row (k)
    constexpr int BTOT = Cfg::BK * BCH;
    for (int64_t kt = 0; kt < KT; ++kt) {
      const int s = static_cast<int>(kt % Cfg::STAGES);
      if (kt >= Cfg::STAGES) mbar_wait(&empty[s], static_cast<unsigned>(((kt / Cfg::STAGES) - 1) & 1));
      const int64_t k0 = kt * Cfg::BK;
      const int64_t k_left = g.Kin - k0;
      double* as = As + s * Cfg::A_STAGE;
      double* bs = Bs + s * Cfg::B_STAGE;
      for (int c = lane; c < ATOT; c += 32) {
        const int r = c / ACH, cc = (c % ACH) * V;
        int64_t valid = (r < m_left) ? (k_left - cc) : 0;
        valid = valid < 0 ? 0 : (valid > V ? V : valid);
        const double* src = valid > 0 ? a_tile + r * g.A.s_mn + k0 + cc : g.A.ptr;
        if (V == 2)
          cp_async16(as + r * Cfg::LDA + cc, src, static_cast<int>(valid * 8));
        else
          cp_async8(as + r * Cfg::LDA + cc, src, static_cast<int>(valid * 8));
      }
      for (int c = lane; c < BTOT; c += 32) {
        const int r = c / BCH, cc = (c % BCH) * V;
        int64_t valid = (r < k_left) ? (n_left - cc) : 0;
        valid = valid < 0 ? 0 : (valid > V ? V : valid);
        const double* src = valid > 0 ? b_tile + (k0 + r) * g.B.s_ki + cc : g.B.ptr;
        if (V == 2)
          cp_async16(bs + r * Cfg::LDB + cc, src, static_cast<int>(valid * 8));
        else
          cp_async8(bs + r * Cfg::LDB + cc, src, static_cast<int>(valid * 8));
      }
      mbar_cp_async_arrive(&full[s]);
    }
    return;
  }
  // ---------------- consumer warps ----------------
  const int gq = lane >> 2, tq = lane & 3;
  const int wmi = warp % Cfg::WM;
  const int wm0 = wmi * Cfg::TM;
  const int wn0 = (warp / Cfg::WM) * Cfg::TN;
  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int a = 0; a < Cfg::FM; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  constexpr int KSTEPS = Cfg::BK / 4;
  double afr[2][Cfg::FM], bfr[2][Cfg::FN];
  for (int64_t kt = 0; kt < KT; ++kt) {
    const int s = static_cast<int>(kt % Cfg::STAGES);
    mbar_wait(&full[s], static_cast<unsigned>((kt / Cfg::STAGES) & 1));
    const double* as = As + s * Cfg::A_STAGE;
    const double* bs = Bs + s * Cfg::B_STAGE;
    auto load_frags = [&](int buf, int kk) {
#pragma unroll
      for (int a = 0; a < Cfg::FM; ++a) afr[buf][a] = as[(wm0 + a * 8 + gq) * Cfg::LDA + kk + tq];
#pragma unroll
      for (int b = 0; b < Cfg::FN; ++b) bfr[buf][b] = bs[(kk + tq) * Cfg::LDB + wn0 + b * 8 + gq];
    };
    load_frags(0, 0);
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      if (ks + 1 < KSTEPS) load_frags((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int a = 0; a < Cfg::FM; ++a)
#pragma unroll
        for (int b = 0; b < Cfg::FN; ++b)
          dmma884(acc[a][b][0], acc[a][b][1], afr[ks & 1][a], bfr[ks & 1][b]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  // epilogue (as tree_p_kernel; consumer-only named barrier)
  double* Pb = g.C + i * g.sCb;
  double colsum[Cfg::FN][2];
#pragma unroll
  for (int j = 0; j < Cfg::FN; ++j) colsum[j][0] = colsum[j][1] = 0.0;
#pragma unroll
  for (int fi = 0; fi < Cfg::FM; ++fi) {
    const int64_t jrow = m0 + wm0 + fi * 8 + gq;
    const bool rv = jrow < g.M;
#pragma unroll
    for (int fj = 0; fj < Cfg::FN; ++fj) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = n0 + wn0 + fj * 8 + 2 * tq + h;
        if (rv && r < g.N) {
          const double v = acc[fi][fj][h];
          if (store_p) Pb[jrow * g.sCm + r] = v;
          colsum[fj][h] = fma(v, __ldg(Bf + jrow * R + r), colsum[fj][h]);
        }
      }
    }
  }
#pragma unroll
  for (int fj = 0; fj < Cfg::FN; ++fj)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double v = colsum[fj][h];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      colsum[fj][h] = v;
    }
  if (gq == 0) {
#pragma unroll
    for (int fj = 0; fj < Cfg::FN; ++fj)
#pragma unroll
      for (int h = 0; h < 2; ++h) red[wmi][wn0 + fj * 8 + 2 * tq + h] = colsum[fj][h];
  }
  asm volatile("bar.sync 1, %0;" ::"n"(Cfg::THREADS));
  for (int c = threadIdx.x; c < Cfg::BN; c += Cfg::THREADS) {
    const int64_t r = n0 + c;
    if (r >= g.N) continue;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < Cfg::WM; ++w) sum += red[w][c];
    m1part[(i * jtiles + tm) * R + r] = sum;
  }
}

// TMA tree kernel.  Both operand tiles arrive by cp.async.bulk.tensor into
// dense 128-byte-swizzled stage buffers (16-byte chunk c of a 128-byte row r
// lands at chunk c ^ (r & 7)): the X tile (128 rows j x 16 k, K-contiguous)
// as one box, the C tile (16 k x 64 r) as four 16 x 16 boxes.  With no
// padding, 4 stages of 24 KB fit twice per SM.  There is no producer warp:
// each of the 4 DMMA warps counts itself out of a stage on a shared counter
// and the LAST one to leave re-arms the stage's mbarrier and issues its
// refill (k-tile kt + STAGES), so the CTA is 128 threads and the register
// budget (255) holds the 64x32 warp tile without spills.
// Fragment k assignment: a 64-bit LDS is served per half-warp (lanes gq in
// 4h..4h+3, tq 0..3 -> 16 x 8 B = one pass over the 32 banks), so the 4
// k values a k-step gives the tq lanes must spread over distinct 8-byte
// slots for BOTH operands: A wants distinct (bit 0, bit 3) of k (chunk group
// and half under the row XOR), B wants distinct (bit 1, bit 2) of k (the XOR
// with k & 7).  k = {0, 3, 12, 15} ^ d with d = {0, 1, 4, 5} per k-step
// satisfies both and covers the 16 k of a stage.  The products per output
// are the same; they are added in this fixed order (bit-reproducible).
template <int STAGES_, int MINB_>
struct TreeTmaT {
  static constexpr int BM = 128, BN = 64, BK = 16, STAGES = STAGES_, MINB = MINB_;
  static constexpr int WM = 2, WN = 2, THREADS = WM * WN * 32;
  static constexpr int TM = BM / WM, TN = BN / WN, FM = TM / 8, FN = TN / 8;
  static constexpr int A_STAGE = BM * BK;  // doubles
  static constexpr int B_STAGE = BK * BN;
  static constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;  // + alignment slack
};
using TreeTma = TreeTmaT<4, 2>;

__device__ __forceinline__ void tree_tma_issue(const CUtensorMap* xmap, const CUtensorMap* cmap,
                                               double* as, double* bs, uint64_t* bar, int k0, int m0,
                                               int n0, int i, uint64_t pol_x, uint64_t pol_c) {
  mbar_arrive_expect_tx(bar, TreeTma::STAGE_BYTES);
  tma_load_3d(as, xmap, bar, k0, m0, i, pol_x);
#pragma unroll
  for (int q = 0; q < TreeTma::BN / 16; ++q)
    tma_load_2d(bs + q * 16 * TreeTma::BK, cmap, bar, n0 + 16 * q, k0, pol_c);
}

// REDUCE = false: the plain product (store_p ignored, P always stored, no
// mode-1 reduction): the last-mode tensor-times-matrix of tucker.cu
template <class T, bool REDUCE = true>
__global__ void __launch_bounds__(T::THREADS, T::MINB)
    tree_p_tma_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap cmap,
                      BtGemmArgs g, const double* __restrict__ Bf, int64_t R,
                      double* __restrict__ m1part, int64_t jtiles, int store_p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[T::WM][T::BN];
  __shared__ __align__(8) uint64_t full[T::STAGES];
  __shared__ int left_cnt[T::STAGES];
  const int tm = blockIdx.x, tn = blockIdx.y, i = blockIdx.z;
  const int m0 = tm * T::BM, n0 = tn * T::BN;
  const int KT = static_cast<int>((g.Kin + T::BK - 1) / T::BK);
  // offset from smem_raw (not an integer round trip) so the fragment reads
  // stay LDS instead of generic loads
  double* As = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  double* Bs = As + T::STAGES * T::A_STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol_x = l2_policy_evict_first();
  const uint64_t pol_c = l2_policy_evict_last();
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&xmap);
    tma_prefetch_desc(&cmap);
    for (int s = 0; s < T::STAGES; ++s) {
      mbar_init(&full[s], 1);
      left_cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < T::STAGES && s < KT; ++s)
      tree_tma_issue(&xmap, &cmap, As + s * T::A_STAGE, Bs + s * T::B_STAGE, &full[s], s * T::BK, m0,
                     n0, i, pol_x, pol_c);
  }
  __syncthreads();
  const int gq = lane >> 2, tq = lane & 3;
  const int wmi = warp % T::WM;
  const int wm0 = wmi * T::TM;
  const int wn0 = (warp / T::WM) * T::TN;
  double acc[T::FM][T::FN][2];
#pragma unroll
  for (int a = 0; a < T::FM; ++a)
#pragma unroll
    for (int b = 0; b < T::FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  constexpr int KSTEPS = T::BK / 4;
  const int kq = 3 * (tq & 1) + 12 * (tq >> 1);   // {0, 3, 12, 15}
  const int g2 = gq >> 1, g1 = gq & 1;
  double afr[2][T::FM], bfr[2][T::FN];
  auto load_frags = [&](int buf, const double* as, const double* bs, int ks) {
    const int k = kq ^ ((ks & 1) + 4 * (ks >> 1));     // ^ {0, 1, 4, 5}
    const int acol = 2 * ((k >> 1) ^ gq) + (k & 1);
#pragma unroll
    for (int a = 0; a < T::FM; ++a) afr[buf][a] = as[(wm0 + a * 8 + gq) * T::BK + acol];
    const int x = k & 7;
#pragma unroll
    for (int b = 0; b < T::FN; ++b) {
      const int q = (wn0 >> 4) + (b >> 1);
      const int chunk = (4 * (b & 1) + g2) ^ x;
      bfr[buf][b] = bs[q * 16 * T::BK + k * 16 + 2 * chunk + g1];
    }
  };
  // fragments are software-pipelined across stages: the last k-step of
  // stage s issues its DMMAs after the first fragments of stage s + 1 are in
  // flight, and stage s is released (refilled) as soon as its last
  // fragments sit in registers
  if (KT > 0) {
    mbar_wait(&full[0], 0u);
    load_frags(0, As, Bs, 0);
  }
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % T::STAGES;
    const double* as = As + s * T::A_STAGE;
    const double* bs = Bs + s * T::B_STAGE;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      if (ks + 1 < KSTEPS) {
        load_frags((ks + 1) & 1, as, bs, ks + 1);
      } else {
        // leave stage s; the last warp out refills it with k-tile kt + STAGES
        __syncwarp();
        if (lane == 0) {
          int old;
          asm volatile("atom.release.cta.shared::cta.add.s32 %0, [%1], 1;"
                       : "=r"(old)
                       : "r"(smem_u32(&left_cnt[s]))
                       : "memory");
          if (old == T::WM * T::WN - 1) {
            asm volatile("fence.acq_rel.cta;" ::: "memory");
            left_cnt[s] = 0;
            const int nk = kt + T::STAGES;
            if (nk < KT) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              tree_tma_issue(&xmap, &cmap, As + s * T::A_STAGE, Bs + s * T::B_STAGE, &full[s],
                             nk * T::BK, m0, n0, i, pol_x, pol_c);
            }
          }
        }
        if (kt + 1 < KT) {
          const int s1 = (kt + 1) % T::STAGES;
          mbar_wait(&full[s1], static_cast<unsigned>(((kt + 1) / T::STAGES) & 1));
          load_frags(0, As + s1 * T::A_STAGE, Bs + s1 * T::B_STAGE, 0);
        }
      }
#pragma unroll
      for (int a = 0; a < T::FM; ++a)
#pragma unroll
        for (int b = 0; b < T::FN; ++b) dmma884(acc[a][b][0], acc[a][b][1], afr[ks & 1][a], bfr[ks & 1][b]);
    }
  }
  // epilogue (tree_p_ws_kernel's)
  double* Pb = g.C + i * g.sCb;
  double colsum[T::FN][2];
#pragma unroll
  for (int j = 0; j < T::FN; ++j) colsum[j][0] = colsum[j][1] = 0.0;
#pragma unroll
  for (int fi = 0; fi < T::FM; ++fi) {
    const int64_t jrow = m0 + wm0 + fi * 8 + gq;
    const bool rv = jrow < g.M;
#pragma unroll
    for (int fj = 0; fj < T::FN; ++fj) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = n0 + wn0 + fj * 8 + 2 * tq + h;
        if (rv && r < g.N) {
          const double v = acc[fi][fj][h];
          if (!REDUCE || store_p) Pb[jrow * g.sCm + r] = v;
          if (REDUCE) colsum[fj][h] = fma(v, __ldg(Bf + jrow * R + r), colsum[fj][h]);
        }
      }
    }
  }
  if (!REDUCE) return;
#pragma unroll
  for (int fj = 0; fj < T::FN; ++fj)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double v = colsum[fj][h];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      colsum[fj][h] = v;
    }
  if (gq == 0) {
#pragma unroll
    for (int fj = 0; fj < T::FN; ++fj)
#pragma unroll
      for (int h = 0; h < 2; ++h) red[wmi][wn0 + fj * 8 + 2 * tq + h] = colsum[fj][h];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < T::BN; c += T::THREADS) {
    const int64_t r = n0 + c;
    if (r >= g.N) continue;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < T::WM; ++w) sum += red[w][c];
    m1part[(i * jtiles + tm) * R + r] = sum;
  }
}

// ---------------------------------------------------------------------------
// M2 partials from P: m2part[s][j][r] = sum_{i in chunk s} P[i][j][r] A[i][r]
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256)
    mode2_from_p_kernel(const double* __restrict__ P, const double* __restrict__ A, int64_t I,
                        int64_t JR, int64_t R, int64_t chunk, double* __restrict__ m2part) {
  const int64_t s = blockIdx.y;
  const int64_t i0 = s * chunk, i1 = min(I, i0 + chunk);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < JR;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % R;
    double acc0 = 0.0, acc1 = 0.0;
    int64_t i = i0;
    for (; i + 1 < i1; i += 2) {
      acc0 = fma(ld_stream(P + i * JR + e), __ldg(A + i * R + r), acc0);
      acc1 = fma(ld_stream(P + (i + 1) * JR + e), __ldg(A + (i + 1) * R + r), acc1);
    }
    if (i < i1) acc0 = fma(ld_stream(P + i * JR + e), __ldg(A + i * R + r), acc0);
    m2part[s * JR + e] = acc0 + acc1;
  }
}

// Q-tree mode 2: m2[j][r] = sum_k Q[j][k][r] C[k][r], one CTA per j; G
// k-groups of R threads sum k = g, g + G, ... in order, then the groups are
// added in a fixed order (bit-reproducible)
__global__ void __launch_bounds__(256)
    mode2_from_q_kernel(const double* __restrict__ Q, const double* __restrict__ C, int64_t K,
                        int R, double* __restrict__ m2) {
  __shared__ double part[256];
  const int64_t j = blockIdx.x;
  const double* q = Q + j * K * R;
  const int groups = R <= 256 ? 256 / R : 1;
  for (int r0 = 0; r0 < R; r0 += 256) {
    const int g = R <= 256 ? threadIdx.x / R : 0;
    const int r = R <= 256 ? threadIdx.x % R : r0 + threadIdx.x;
    const bool act = (R <= 256) ? (g < groups) : (r < R);
    double acc0 = 0.0, acc1 = 0.0;
    if (act) {
      int64_t k = g;
      for (; k + groups < K; k += 2 * groups) {
        acc0 = fma(ld_stream(q + k * R + r), __ldg(C + k * R + r), acc0);
        acc1 = fma(ld_stream(q + (k + groups) * R + r), __ldg(C + (k + groups) * R + r), acc1);
      }
      if (k < K) acc0 = fma(ld_stream(q + k * R + r), __ldg(C + k * R + r), acc0);
    }
    part[threadIdx.x] = acc0 + acc1;
    __syncthreads();
    if (R <= 256) {
      if (threadIdx.x < R) {
        double v = 0.0;
        for (int gg = 0; gg < groups; ++gg) v += part[gg * R + threadIdx.x];
        m2[j * R + threadIdx.x] = v;
      }
      break;
    }
    if (r < R) m2[j * R + r] = part[threadIdx.x];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// on-chip symmetric Jacobi: pinv of an R x R symmetric matrix
// ---------------------------------------------------------------------------

__device__ void pinv_from_eig(const double* a, const double* qv, int R, int ld, double* out) {
  __shared__ double wmax;
  __shared__ double inv[PINV_MAX_R + 1];
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < R; ++i) m = fmax(m, fabs(a[i * ld + i]));
    wmax = m;
  }
  __syncthreads();
  const double cut = 1e-15 * wmax;  // numpy pinv: rcond 1e-15 times the largest singular value
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const double w = a[i * ld + i];
    inv[i] = (fabs(w) > cut) ? 1.0 / w : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
    const int r = idx / R, c = idx % R;
    double s = 0.0;
    for (int k = 0; k < R; ++k) s = fma(qv[r * ld + k] * inv[k], qv[c * ld + k], s);
    out[idx] = s;
  }
}

template <int NP>
__device__ __forceinline__ void load_v(const double* __restrict__ g0, const double* __restrict__ g1,
                                       int R, double* a, double& ss) {
  constexpr int LD = NP + 1;
  ss = 0.0;
  for (int idx = threadIdx.x; idx < NP * NP; idx += blockDim.x) {
    const int r = idx / NP, c = idx % NP;
    double v = 0.0;
    if (r < R && c < R) v = g1 ? g0[r * R + c] * g1[r * R + c] : g0[r * R + c];
    a[r * LD + c] = v;
    ss = fma(v, v, ss);
  }
}

// Vp = pinv(V), V = G0 o G1 (SPD Gram-Hadamard product, R <= NP).
// Fast path: V^-1 = L^-T L^-1 from a Cholesky factorisation in shared memory
// (R steps), accepted when the exact 1-norm condition number
// ||V||_1 ||V^-1||_1 <= 1e12 -- there numpy's pinv (decomp.py:387, cutoff
// 1e-15 sigma_max) is the inverse and both agree to ~cond * eps.  Otherwise
// (or on a non-positive pivot) the eigen path: cyclic Jacobi + the pinv cutoff.
// The whole CTA computes vp (global or shared); smf: 3 NP (NP+1) doubles of
// shared scratch.  Used by pinv_fast_kernel and by the fused small CP-ALS.
template <int NP>
__device__ void pinv_block(const double* __restrict__ g0, const double* __restrict__ g1, int R,
                           double* __restrict__ vp, double* smf) {
  constexpr int LD = NP + 1;
  constexpr int HALF = NP / 2;
  double* a = smf;
  double* q = a + NP * LD;
  double* x = q + NP * LD;
  __shared__ double cs[HALF], sn[HALF];
  __shared__ int pp[HALF], qq[HALF];
  __shared__ double fro_red[32];
  __shared__ int chol_ok;
  __shared__ double vnorm1, inorm1;
  const int tid = threadIdx.x;
  double ss;
  load_v<NP>(g0, g1, R, a, ss);
  if (tid == 0) chol_ok = 1;
  __syncthreads();
  // ||V||_1 (column sums in parallel) and the working copy of the lower triangle
  if (tid < 32) {
    double m = 0.0;
    for (int c = tid; c < R; c += 32) {
      double c1 = 0.0;
      for (int r = 0; r < R; ++r) c1 += fabs(a[r * LD + c]);
      m = fmax(m, c1);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tid == 0) vnorm1 = m;
  }
  for (int idx = tid; idx < R * R; idx += blockDim.x) {
    const int r = idx / R, c = idx % R;
    q[r * LD + c] = a[r * LD + c];
  }
  __syncthreads();
  // Cholesky, one barrier per step: the trailing update uses the unscaled
  // pivot column (q[i][k] q[j][k] / d) and L's column k goes to x, so no
  // value read in the phase is written in it
  const int tx = tid & 31, ty = tid >> 5, ny = blockDim.x >> 5;
  for (int k = 0; k < R; ++k) {
    const double d = q[k * LD + k];
    if (!(d > 0.0)) {
      chol_ok = 0;  // every thread sees the same d: uniform exit
      break;
    }
    const double rs = 1.0 / sqrt(d), rd = rs * rs;
    for (int i = k + ty; i < R; i += ny) {
      const double qik = q[i * LD + k];
      if (tx == 0) x[i * LD + k] = qik * rs;
      for (int j = k + 1 + tx; j <= i; j += 32) q[i * LD + j] -= qik * q[j * LD + k] * rd;
    }
    __syncthreads();
  }
  __syncthreads();
  if (chol_ok && tid == 0) {
    // kappa_2(V) >= (max l_kk / min l_kk)^2 and kappa_1 >= kappa_2 / R: a
    // diagonal ratio beyond R * 1e12 fails the test below for sure, so the
    // inverse is not formed (ill-conditioned V goes straight to the eigen path)
    double lo = INFINITY, hi = 0.0;
    for (int k = 0; k < R; ++k) {
      const double l = x[k * LD + k];
      lo = fmin(lo, l);
      hi = fmax(hi, l);
    }
    if ((hi / lo) * (hi / lo) > 1e12 * R) chol_ok = 0;
  }
  __syncthreads();
  if (chol_ok) {
    // Y = L^-1 by right-looking substitution on the identity, one barrier
    // per step (row k's division is applied one step late, when no thread
    // reads it any more); Y overwrites q
    for (int idx = tid; idx < R * R; idx += blockDim.x) {
      const int r = idx / R, c = idx % R;
      q[r * LD + c] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int k = 0; k < R; ++k) {
      const double rk = 1.0 / x[k * LD + k];
      if (k > 0 && ty == 0) {
        const double rp = 1.0 / x[(k - 1) * LD + (k - 1)];
        for (int j = tx; j < R; j += 32) q[(k - 1) * LD + j] *= rp;
      }
      for (int i = k + 1 + ty; i < R; i += ny) {
        const double f = x[i * LD + k] * rk;
        for (int j = tx; j < R; j += 32) q[i * LD + j] -= f * q[k * LD + j];
      }
      __syncthreads();
    }
    {
      const double rl = 1.0 / x[(R - 1) * LD + (R - 1)];
      for (int j = tid; j < R; j += blockDim.x) q[(R - 1) * LD + j] *= rl;
    }
    __syncthreads();
    // V^-1 = Y^T Y into a (V is reloaded if the eigen path is needed)
    for (int idx = tid; idx < R * R; idx += blockDim.x) {
      const int r = idx / R, c = idx % R;
      const int k0 = r > c ? r : c;
      double v = 0.0;
      for (int k = k0; k < R; ++k) v = fma(q[k * LD + r], q[k * LD + c], v);
      a[r * LD + c] = v;
    }
    __syncthreads();
    if (tid < 32) {
      double m = 0.0;
      for (int c = tid; c < R; c += 32) {
        double c1 = 0.0;
        for (int r = 0; r < R; ++r) c1 += fabs(a[r * LD + c]);
        m = fmax(m, c1);
      }
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (tid == 0) inorm1 = m;
    }
    __syncthreads();
    if (vnorm1 * inorm1 <= 1e12) {
      for (int idx = tid; idx < R * R; idx += blockDim.x)
        vp[idx] = a[(idx / R) * LD + idx % R];
      return;
    }
    load_v<NP>(g0, g1, R, a, ss);
    __syncthreads();
  }
  // eigen path.  Absolute floor 1e-15 ||V||_F: off-diagonals below it are
  // rounding noise (the reference's SVD-based pinv resolves V only to
  // ~eps ||V|| as well)
  ss = warp_sum(ss);
  if ((tid & 31) == 0) fro_red[tid >> 5] = ss;
  __syncthreads();
  double fro2 = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) fro2 += fro_red[w];
  if constexpr (NP <= 32)
    jacobi_warp_t<NP>(a, q, LD, cs, sn, pp, qq, 40, 1e-15 * sqrt(fro2), 1e-15);
  else
    jacobi_fast(a, q, NP, LD, cs, sn, pp, qq, 40, 1e-15 * sqrt(fro2), 1e-15);
  __syncthreads();
  pinv_from_eig(a, q, R, LD, vp);
}

// Vp = pinv(V), V = G0 o G1, R <= NP <= 32, by one-sided (Hestenes) Jacobi
// held in the registers of ONE warp: lane (c + NP h) owns rows
// [h ROWS, (h+1) ROWS) of column c of W (= V J, starts at V) and of the
// accumulated rotation J (starts at I).  A round pairs the columns by the
// circle method (partner of c in round r: (2r - c) mod (NP - 1), with NP - 1
// meeting r); the two lanes of a pair swap their halves by shuffles, form
// ||w_p||^2, ||w_q||^2, w_p . w_q (row halves added in a fixed order, so both
// lanes get the same bits), and apply the same rotation -- no shared memory,
// no barrier, no data-dependent register index.  The rotation is the
// one-sided one (it orthogonalises W = V J, i.e. diagonalises J^T V^2 J, whose
// eigenvectors are V's); the stopping rule and the pinv are the two-sided
// eigen path's: rotate while |(J^T V J)_pq| > 1e-15 ||V||_F, then
// pinv(V) = sum_{|lambda_k| > 1e-15 max|lambda|} J_k J_k^T / lambda_k with
// lambda_k = (J^T V J)_kk (numpy's rcond cutoff, decomp.py:387).

// In-place Gauss-Jordan inverse of V = g0 o g1 (SPD: no pivoting needed) by
// one warp, the matrix spread over the lanes' registers (NP = 8: lane holds
// 2 entries of a row, NP = 16: 8).  One step per column: the pivot row and
// the lane's own column-k entry arrive by shuffles, one refined reciprocal,
// one fused update -- ~170 cycles of dependent latency per step where the
// Cholesky route (factor, triangular inverse, Y^T Y through shared memory)
// took ~6k cycles at NP = 8.  Accepted when every pivot is positive,
// max / min pivot <= 1e14 R and ||V||_1 ||V^-1||_1 <= 1e14: numpy's pinv
// (rcond 1e-15) is the plain inverse up to kappa_2 = 1e15, and both are
// accurate to ~kappa eps there; beyond, the eigen path decides the cutoff.
template <int NP>
__device__ __forceinline__ bool spd_inv_gj(const double* __restrict__ g0,
                                           const double* __restrict__ g1, int R,
                                           double* __restrict__ vp) {
  static_assert(NP == 8 || NP == 16, "NP in {8, 16}");
  constexpr int EPL = NP * NP / 32;   // entries per lane
  constexpr int LPR = NP / EPL;       // lanes per row
  const int lane = threadIdx.x & 31;
  const int i = lane / LPR, sub = lane % LPR, jb = sub * EPL;
  double a[EPL];
  double rs = 0.0;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const int j = jb + e;
    double v = (i == j) ? 1.0 : 0.0;
    if (i < R && j < R) {
      v = g1 ? g0[i * R + j] * g1[i * R + j] : g0[i * R + j];
      rs += fabs(v);
    }
    a[e] = v;
  }
  auto row_max = [&](double v) {   // sum over the row's lanes, then max over rows
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  };
  const double vn1 = row_max(rs);
  bool ok = true;
  double lo = INFINITY, hi = 0.0;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int ck = k / EPL, ek = k % EPL;
    const double f = __shfl_sync(0xffffffffu, a[ek], i * LPR + ck);
    const double p = __shfl_sync(0xffffffffu, a[ek], k * LPR + ck);
    double prow[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) prow[e] = __shfl_sync(0xffffffffu, a[e], k * LPR + sub);
    ok = ok && (p > 0.0);
    lo = fmin(lo, p);
    hi = fmax(hi, p);
    const double ip = rcp_nr(fmax(p, 1e-300));
    const double fi = -f * ip;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const bool colk = (jb + e == k);
      if (i == k)
        a[e] = colk ? ip : a[e] * ip;
      else
        a[e] = colk ? fi : fma(fi, prow[e], a[e]);
    }
  }
  if (!ok || hi > 1e14 * R * lo) return false;   // warp-uniform
  double is = 0.0;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const int j = jb + e;
    if (i < R && j < R) {
      vp[i * R + j] = a[e];
      is += fabs(a[e]);
    }
  }
  const double in1 = row_max(is);
  __syncwarp();
  return vn1 * in1 <= 1e14;
}


__device__ long long g_pinv1s_dbg[2];  // sweeps, cycles of the last call (diagnostics)
__device__ long long g_pinv1s_log[512];  // (sweeps << 40 | cycles) per call, ring (diagnostics)
__device__ unsigned g_pinv1s_n;

// One-warp pinv of V = g0 o g1 (R <= NP).  jstore / warm are kept for the
// launch signature (the warm start from the previous sweep's rotation was
// dropped: ALS changes C4's V too much between sweeps for it to help).
template <int NP>
__global__ void __launch_bounds__(32) pinv_jacobi1_kernel(const double* __restrict__ g0,
                                                          const double* __restrict__ g1, int R,
                                                          double* __restrict__ vp,
                                                          double* __restrict__ jstore, int warm) {
  static_assert(NP == 8 || NP == 16 || NP == 32, "NP in {8, 16, 32}");
  constexpr int HALVES = 32 / NP, ROWS = NP / HALVES;
  __shared__ double js[NP][NP + 1], ws[NP][NP + 1], isg[NP];
  const int lane = threadIdx.x;
  const int col = lane % NP, half = lane / NP, r0 = half * ROWS;
  double w[ROWS];
  // ---- well-conditioned V: in-register Gauss-Jordan inverse (spd_inv_gj),
  // accepted on pinv_block's test (kappa_1 <= 1e12, where numpy's pinv is
  // the inverse to ~kappa eps)
  {
    const bool ok = spd_inv_gj<NP == 32 ? 16 : NP>(g0, g1, R, vp);
    if (ok) return;
    __syncwarp();
  }
  // ---- ill-conditioned / singular V.  Stage 1: Cholesky with diagonal
  // pivoting in shared memory, V = L L^T with L's columns in pivot order
  // (rows stay in V's order: no permutation to undo), stopped at the first
  // pivot below NP eps max(diag V) -- the Schur complement is rounding noise
  // of V from there on.  Stage 2: one-sided Jacobi on the COLUMNS of L
  // (L W = U Sigma, so V = U Sigma^2 U^T): L^T L is far closer to diagonal
  // than V, the columns carry their own scale (a pair is rotated while
  // |w_p . w_q| > 1e-15 |w_p| |w_q|, no absolute floor needed) and no
  // eigenvector accumulator is kept -- 5-6 sweeps where Jacobi on V itself
  // took 10-14 (C4's mode-3 normal matrices, cond ~1e18) and each round
  // moves half the data.  pinv = sum over sigma_k^2 > 1e-15 max sigma^2 of
  // w_k w_k^T / sigma_k^4 (numpy's rcond on the eigenvalues sigma^2).
  (void)warm;
  (void)jstore;
  double d0 = 0.0;
  for (int idx = lane; idx < NP * NP; idx += 32) {
    const int r = idx / NP, c = idx % NP;
    double v = 0.0;
    if (r < R && c < R) v = g1 ? g0[r * R + c] * g1[r * R + c] : g0[r * R + c];
    ws[r][c] = v;
    js[r][c] = 0.0;
    if (r == c) d0 = fmax(d0, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
  __syncwarp();
  const double piv_floor = NP * 2.220446049250313e-16 * d0;
  unsigned done = 0u;
  int rank = 0;
  double dmin = d0;
  for (int k = 0; k < R; ++k) {
    double dv = (lane < NP && !((done >> lane) & 1u)) ? ws[lane][lane] : -1.0;
    int di = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, dv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, di, o);
      if (ov > dv || (ov == dv && oi < di)) {
        dv = ov;
        di = oi;
      }
    }
    if (!(dv > piv_floor)) break;
    ++rank;
    dmin = dv;
    const double inv = rsqrt_nr(dv), piv = dv * inv;
    if (lane < NP) {
      double l = 0.0;
      if (lane == di) l = piv;
      else if (!((done >> lane) & 1u)) l = ws[lane][di] * inv;
      js[lane][k] = l;
    }
    done |= 1u << di;
    __syncwarp();
    for (int idx = lane; idx < NP * NP; idx += 32) {
      const int r = idx / NP, c = idx % NP;
      if (!((done >> r) & 1u) && !((done >> c) & 1u)) ws[r][c] = fma(-js[r][k], js[c][k], ws[r][c]);
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < ROWS; ++i) w[i] = js[r0 + i][col];
  __syncwarp();
  // sum over the HALVES row blocks of a column in a fixed order (block 0
  // first), identical in every lane holding that column
  auto colsum = [&](double v) {
#pragma unroll
    for (int o = NP; o < 32; o <<= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v, o);
      v = (lane & o) ? (u + v) : (v + u);
    }
    return v;
  };
  const long long t_start = clock64();
  int sweeps_done = 0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    int big = 0;
    sweeps_done = sweep + 1;
    for (int rnd = 0; rnd < NP - 1; ++rnd) {
      int partner;
      if (col == NP - 1) {
        partner = rnd;
      } else if (col == rnd) {
        partner = NP - 1;
      } else {
        partner = 2 * rnd - col;
        if (partner < 0) partner += NP - 1;
        if (partner >= NP - 1) partner -= NP - 1;
      }
      const int src = partner + half * NP;
      double pw[ROWS];
#pragma unroll
      for (int i = 0; i < ROWS; ++i) pw[i] = __shfl_sync(0xffffffffu, w[i], src);
      const bool lo = col < partner;
      double a = 0.0, b = 0.0, g = 0.0, a1 = 0.0, b1 = 0.0, g1s = 0.0;
#pragma unroll
      for (int i = 0; i < ROWS; i += 2) {
        const double wp = lo ? w[i] : pw[i], wq = lo ? pw[i] : w[i];
        a = fma(wp, wp, a);
        b = fma(wq, wq, b);
        g = fma(wp, wq, g);
        if (i + 1 < ROWS) {
          const double wp1 = lo ? w[i + 1] : pw[i + 1], wq1 = lo ? pw[i + 1] : w[i + 1];
          a1 = fma(wp1, wp1, a1);
          b1 = fma(wq1, wq1, b1);
          g1s = fma(wp1, wq1, g1s);
        }
      }
      a = colsum(a + a1);
      b = colsum(b + b1);
      g = colsum(g + g1s);
      const double g2 = g * g, ab = a * b;
      if (g2 > 1e-30 * ab) {
        // tan of the rotation angle from tan(2 phi) = 2g / (b - a):
        // t = sgn(d) h / (|d| + sqrt(d^2 + h^2)), d = b - a, h = 2g, with
        // once-refined rsqrt / rcp (an angle good to ~1e-13 keeps the
        // quadratic convergence); c = 1/sqrt(1 + t^2) to full precision and
        // s = t c, so the rotation is orthogonal to rounding whatever t is
        const double d = b - a, h = 2.0 * g;
        const double r2 = fma(d, d, h * h);
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
        y = y * fma(-0.5 * r2 * y, y, 1.5);
        const double den = fma(r2, y, fabs(d));
        double q;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(den));
        q = fma(q, fma(-den, q, 1.0), q);
        const double t = (d < 0.0 ? -h : h) * q;
        const double c = rsqrt_nr(fma(t, t, 1.0));
        const double s = t * c;
        // a sweep whose rotations all had |cos| <= 1e-8 leaves |cos| ~ 1e-16
        // behind (quadratic convergence): it is the last one
        if (g2 > 1e-16 * ab) big = 1;
#pragma unroll
        for (int i = 0; i < ROWS; ++i) w[i] = lo ? (c * w[i] - s * pw[i]) : (s * pw[i] + c * w[i]);
      }
    }
    if (!__any_sync(0xffffffffu, big)) break;
  }
  if (lane == 0) {
    g_pinv1s_dbg[0] = sweeps_done;
    g_pinv1s_dbg[1] = clock64() - t_start;
    const unsigned slot = atomicAdd(&g_pinv1s_n, 1u);
    // sweeps (8 bits) | rank (8 bits) | -log10(dmin / d0) (8 bits) | cycles (32 bits)
    const long long lg = dmin > 0.0 && d0 > 0.0 ? (long long)fmin(255.0, -log10(dmin / d0)) : 255;
    g_pinv1s_log[slot & 511u] = ((long long)sweeps_done << 56) | ((long long)rank << 48) | (lg << 40) |
                                (g_pinv1s_dbg[1] & 0xffffffffll);
  }
  double lk = 0.0;
#pragma unroll
  for (int i = 0; i < ROWS; ++i) lk = fma(w[i], w[i], lk);
  lk = colsum(lk);   // sigma_k^2 = lambda_k
  double lmax = lk;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  if (half == 0) isg[col] = (lk > 1e-15 * lmax) ? 1.0 / (lk * lk) : 0.0;
#pragma unroll
  for (int i = 0; i < ROWS; ++i) js[r0 + i][col] = w[i];
  __syncwarp();
  for (int idx = lane; idx < R * R; idx += 32) {
    const int r = idx / R, c = idx % R;
    double v = 0.0;
    for (int k = 0; k < NP; ++k) v = fma(js[r][k] * isg[k], js[c][k], v);
    vp[idx] = v;
  }
}

template <int NP>
__global__ void __launch_bounds__(1024) pinv_fast_kernel(const double* __restrict__ g0,
                                                         const double* __restrict__ g1, int R,
                                                         double* __restrict__ vp) {
  extern __shared__ __align__(16) double smf[];
  pinv_block<NP>(g0, g1, R, vp, smf);
}


// ---------------------------------------------------------------------------
// Fused small CP-ALS (C1-sized tensors): every sweep of decomp.py:376-401 in
// ONE launch of one CTA -- factors, P = X x3 C, MTTKRPs, Grams and the pinv
// (pinv_block) live in shared memory, X streams from L2.  Same arithmetic as
// the phase kernels (dimension tree for modes 1/2, Cholesky-first pinv, Gram-
// identity fit with the explicit-residual switch, fixed-order sums); used
// when the whole problem fits one SM (the multi-kernel sweep is launch-bound
// there: ~25 kernels of a few microseconds each).
// ---------------------------------------------------------------------------

constexpr int SMALL_RS = 16;  // register row of R values
__device__ long long g_small_clk[16];  // phase clocks of sweep 1 (tools/prof_c1_small.py)

struct SmallLayout {
  int64_t a, b, c, p, m, g, vp, gbuf, nrm, smf, red, total;
};

__host__ __device__ inline SmallLayout small_layout(int64_t I, int64_t J, int64_t K, int64_t R,
                                                    int NP) {
  SmallLayout l{};
  int64_t o = 0;
  auto take = [&](int64_t n) {
    const int64_t at = o;
    o += (n + 1) / 2 * 2;
    return at;
  };
  l.a = take(I * R);
  l.b = take(J * R);
  l.c = take(K * R);
  // P (I J R); reused for the mode-3 chunk partials [chunks][K][16] (16 warps)
  const int64_t mt = (K + 7) / 8;
  const int64_t ch = mt < 15 ? 15 / mt : 1;  // 15 compute warps (warp 0 runs the pinv)
  l.p = take(I * J * R > ch * K * 16 ? I * J * R : ch * K * 16);
  const int64_t mx = I > J ? (I > K ? I : K) : (J > K ? J : K);
  l.m = take(mx * R);
  l.g = take(3 * R * R);
  l.vp = take(R * R);
  l.gbuf = take(R * R + 2);
  l.nrm = take(R);
  l.smf = take(3 * NP * (NP + 1));
  l.red = take(64);
  l.total = o;
  return l;
}

// fixed-order CTA sum (warp shuffles, then warp partials in order); all
// threads return the total
__device__ __forceinline__ double small_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
  return t;
}

// Cholesky-first pinv of V = G0 o G1 (R <= 32) by ONE warp (warp-level
// syncs only): the fast path of pinv_block (V^-1 = L^-T L^-1, accepted when
// ||V||_1 ||V^-1||_1 <= 1e12).  Returns false (warp-uniform) when the caller
// must take pinv_block's eigen path.  a, y: R x (R+1) scratch each.
__device__ bool pinv_warp_chol(const double* __restrict__ g0, const double* __restrict__ g1,
                               int R, double* __restrict__ vp, double* a, double* y) {
  const int lane = threadIdx.x & 31;
  const int ld = R + 1;
  for (int e = lane; e < R * R; e += 32) {
    const int r = e / R, c = e % R;
    a[r * ld + c] = g0[e] * g1[e];
  }
  __syncwarp();
  double cs = 0.0;
  if (lane < R)
    for (int r = 0; r < R; ++r) cs += fabs(a[r * ld + lane]);
  double vn1 = cs;
  for (int o = 16; o > 0; o >>= 1) vn1 = fmax(vn1, __shfl_xor_sync(0xffffffffu, vn1, o));
  // in place: lower triangle -> L; the diagonal's reciprocals go to y's
  // diagonal slots (Newton-refined rsqrt: no IEEE sqrt / division on the
  // critical path -- this warp runs beside 15 DMMA warps)
  for (int k = 0; k < R; ++k) {
    const double d = a[k * ld + k];
    if (!(d > 0.0)) return false;  // same d in every lane
    const double rl = rsqrt_nr(d);
    __syncwarp();
    for (int i = k + 1 + lane; i < R; i += 32) a[i * ld + k] *= rl;
    if (lane == 0) {
      a[k * ld + k] = d * rl;
      y[k * ld + k] = rl;       // 1 / l_kk
    }
    __syncwarp();
    // trailing update, one row per lane (R <= 32: no index division)
    for (int i = k + 1 + lane; i < R; i += 32) {
      const double lik = a[i * ld + k];
      for (int j = k + 1; j <= i; ++j) a[i * ld + j] -= lik * a[j * ld + k];
    }
    __syncwarp();
  }
  // Y = L^-1, one column per lane (reciprocal diagonal from the factorisation)
  __syncwarp();
  if (lane < R) {
    const int c = lane;
    for (int i = 0; i < c; ++i) y[i * ld + c] = 0.0;
    for (int i = c + 1; i < R; ++i) {
      double sacc = 0.0;
      for (int k = c; k < i; ++k) sacc = fma(a[i * ld + k], y[k * ld + c], sacc);
      y[i * ld + c] = -sacc * y[i * ld + i];
    }
  }
  __syncwarp();
  // V^-1 = Y^T Y
  for (int e = lane; e < R * R; e += 32) {
    const int r = e / R, c = e % R;
    const int k0 = r > c ? r : c;
    double v = 0.0;
    for (int k = k0; k < R; ++k) v = fma(y[k * ld + r], y[k * ld + c], v);
    vp[e] = v;
  }
  __syncwarp();
  double ic = 0.0;
  if (lane < R)
    for (int r = 0; r < R; ++r) ic += fabs(vp[r * R + lane]);
  for (int o = 16; o > 0; o >>= 1) ic = fmax(ic, __shfl_xor_sync(0xffffffffu, ic, o));
  return vn1 * ic <= 1e12;
}

template <int NP>
__global__ void __launch_bounds__(512)
    cp_small_kernel(const double* __restrict__ X, int I, int J, int K, int R,
                    double* __restrict__ ga, double* __restrict__ gb, double* __restrict__ gc,
                    double* __restrict__ glam, double x2, int max_iters, double tol, int fit_mode,
                    double* __restrict__ fit_hist, int* __restrict__ out_info) {
  extern __shared__ __align__(16) double sm[];
  const SmallLayout L = small_layout(I, J, K, R, NP);
  double* F[3] = {sm + L.a, sm + L.b, sm + L.c};
  double* P = sm + L.p;
  double* M = sm + L.m;
  double* G[3] = {sm + L.g, sm + L.g + R * R, sm + L.g + 2 * R * R};
  double* Vp = sm + L.vp;
  double* gbuf = sm + L.gbuf;
  double* nrm = sm + L.nrm;
  double* smf = sm + L.smf;
  double* red = sm + L.red;
  __shared__ int stop, pinv_ok;
  __shared__ double fit_s, explicit_s;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t rows[3] = {I, J, K};
  int it = 0;
  for (int e = tid; e < I * R; e += nt) F[0][e] = ga[e];
  for (int e = tid; e < J * R; e += nt) F[1][e] = gb[e];
  for (int e = tid; e < K * R; e += nt) F[2][e] = gc[e];
  if (tid == 0) stop = 0;
  __syncthreads();
  for (int k = 0; k < 3; ++k)
    for (int e = tid; e < R * R; e += nt) {
      const int a = e / R, b = e % R;
      double s = 0.0;
      for (int64_t r = 0; r < rows[k]; ++r) s = fma(F[k][r * R + a], F[k][r * R + b], s);
      G[k][e] = s;
    }
  __syncthreads();
  // one factor update from M (rows x R): pinv, F_un = M Vp, Gram, norms
  // warp 0: Cholesky-first pinv of G_o0 o G_o1 while warps 1.. run the
  // mode's MTTKRP (the Grams it needs are final before that MTTKRP starts)
  auto pinv_w0 = [&](int go0, int go1) {
    if ((tid >> 5) == 0) {
      const long long c0 = clock64();
      const bool ok = R <= 8 ? spd_inv_gj<8>(G[go0], G[go1], R, Vp)
                             : (R <= 16 ? spd_inv_gj<16>(G[go0], G[go1], R, Vp)
                                        : pinv_warp_chol(G[go0], G[go1], R, Vp, smf, smf + R * (R + 1)));
      if (tid == 0) pinv_ok = ok ? 1 : 0;
      if (it == 1 && tid == 0) g_small_clk[9 + go0 + go1] = clock64() - c0;
    }
  };
  auto solve = [&](int k, int go0, int go1, bool last) {
    if (!pinv_ok) {
      pinv_block<NP>(G[go0], G[go1], R, Vp, smf);
      __syncthreads();
    }
    const int64_t nr = rows[k];
    double* f = F[k];
    for (int64_t e = tid; e < nr * R; e += nt) {
      const int64_t row = e / R;
      const int c = static_cast<int>(e % R);
      double s = 0.0;
      for (int q = 0; q < R; ++q) s = fma(M[row * R + q], Vp[q * R + c], s);
      f[e] = s;
    }
    __syncthreads();
    for (int e = tid; e < R * R; e += nt) {
      const int a = e / R, b = e % R;
      double s = 0.0;
      for (int64_t r = 0; r < nr; ++r) s = fma(f[r * R + a], f[r * R + b], s);
      gbuf[e] = s;
    }
    double inner = 0.0;
    if (last) {
      double s = 0.0;
      for (int64_t e = tid; e < nr * R; e += nt) s = fma(f[e], M[e], s);
      inner = small_block_sum(s, red);
    }
    __syncthreads();
    for (int r = tid; r < R; r += nt) {
      double v = sqrt(gbuf[r * R + r]);
      if (v == 0.0) v = 1.0;
      nrm[r] = v;
    }
    __syncthreads();
    for (int e = tid; e < R * R; e += nt) G[k][e] = gbuf[e] / (nrm[e / R] * nrm[e % R]);
    for (int64_t e = tid; e < nr * R; e += nt) f[e] = f[e] / nrm[e % R];
    __syncthreads();
    if (last) {
      double s = 0.0;
      for (int e = tid; e < R * R; e += nt)
        s += nrm[e / R] * nrm[e % R] * G[0][e] * G[1][e] * G[2][e];
      const double xh2 = small_block_sum(s, red);
      if (tid == 0) {
        const double res2 = fmax(x2 - 2.0 * inner + xh2, 0.0);
        const double relres = sqrt(res2 / x2);
        explicit_s = ((fit_mode == 1) || (fit_mode == 0 && relres < 1e-3)) ? 1.0 : 0.0;
        fit_s = 1.0 - relres;
      }
      __syncthreads();
    }
  };
  double prev = -INFINITY;
  int conv = 0;
  for (it = 0; it < max_iters; ++it) {
    if (it == 1 && tid == 0) g_small_clk[0] = clock64();
    // P = X x3 C  (P[ij][r] = sum_k X[ij][k] C[k][r]) on DMMA: warp per
    // 8-row tile of (ij), both 8-wide r tiles, k in steps of 4
    pinv_w0(1, 2);
    if (tid >= 32) {
      const int lane = tid & 31, warp = (tid >> 5) - 1, nw = (nt >> 5) - 1;
      const int gq = lane >> 2, tq = lane & 3;
      const int64_t IJ = (int64_t)I * J;
      for (int64_t m0 = (int64_t)warp * 8; m0 < IJ; m0 += (int64_t)nw * 8) {
        double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
        const int64_t row = m0 + gq;
        const double* xr = X + (row < IJ ? row : 0) * K;
        // 8 X loads in flight per lane (32 k per chunk): the L2 latency is
        // paid once per chunk instead of once per k-step
        constexpr int UK = 8;
        for (int k0 = 0; k0 < K; k0 += 4 * UK) {
          double av[UK];
#pragma unroll
          for (int u = 0; u < UK; ++u) {
            const int kk = k0 + 4 * u + tq;
            av[u] = (row < IJ && kk < K) ? __ldg(xr + kk) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < UK; ++u) {
            const int kk = k0 + 4 * u + tq;
            const double b0 = (kk < K && gq < R) ? F[2][kk * R + gq] : 0.0;
            dmma884(c00, c01, av[u], b0);
            if (R > 8) {
              const double b1 = (kk < K && 8 + gq < R) ? F[2][kk * R + 8 + gq] : 0.0;
              dmma884(c10, c11, av[u], b1);
            }
          }
        }
        if (row < IJ) {
          const int n = 2 * tq;
          if (n < R) P[row * R + n] = c00;
          if (n + 1 < R) P[row * R + n + 1] = c01;
          if (R > 8) {
            if (8 + n < R) P[row * R + 8 + n] = c10;
            if (9 + n < R) P[row * R + 9 + n] = c11;
          }
        }
      }
    }
    __syncthreads();
    if (it == 1 && tid == 0) g_small_clk[1] = clock64();
    // mode 1: M[i][r] = sum_j P[i][j][r] B[j][r]
    if (tid >= 32)
      for (int e = tid - 32; e < I * R; e += nt - 32) {
        const int i = e / R, r = e % R;
        double s = 0.0;
        for (int j = 0; j < J; ++j) s = fma(P[((int64_t)i * J + j) * R + r], F[1][j * R + r], s);
        M[e] = s;
      }
    __syncthreads();
    if (it == 1 && tid == 0) g_small_clk[2] = clock64();
    solve(0, 1, 2, false);
    if (it == 1 && tid == 0) g_small_clk[3] = clock64();
    // mode 2: M[j][r] = sum_i P[i][j][r] A[i][r]  (A just updated)
    pinv_w0(0, 2);
    if (tid >= 32)
      for (int e = tid - 32; e < J * R; e += nt - 32) {
        const int j = e / R, r = e % R;
        double s = 0.0;
        for (int i = 0; i < I; ++i) s = fma(P[((int64_t)i * J + j) * R + r], F[0][i * R + r], s);
        M[e] = s;
      }
    __syncthreads();
    if (it == 1 && tid == 0) g_small_clk[4] = clock64();
    solve(1, 0, 2, false);
    if (it == 1 && tid == 0) g_small_clk[5] = clock64();
    // mode 3: M[k][r] = sum_ij X[ij][k] A[i][r] B[j][r] on DMMA: rows k
    // (8-tiles), cols r, the (ij) reduction split in fixed chunks over the
    // warps, chunk partials summed in order through shared memory
    pinv_w0(0, 1);
    {
      const int lane = tid & 31, warp = (tid >> 5) - 1, nw = (nt >> 5) - 1;
      const int gq = lane >> 2, tq = lane & 3;
      const int64_t IJ = (int64_t)I * J;
      const int mtiles = (K + 7) / 8;
      const int chunks = nw / mtiles > 0 ? nw / mtiles : 1;  // as small_layout (nw = 15)
      const int64_t clen = ((IJ + chunks - 1) / chunks + 3) / 4 * 4;
      double* part = P;  // P is free again: [chunk][k][16] partials
      for (int item = warp; warp >= 0 && item < mtiles * chunks; item += nw) {
        const int mt = item % mtiles, ch = item / mtiles;
        const int kr = mt * 8 + gq;
        double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
        const int64_t s0 = ch * clen, s1 = s0 + clen < IJ ? s0 + clen : IJ;
        int64_t ij = s0 + tq;
        int64_t ii = ij / J, jj = ij - ii * J;
        constexpr int UN = 8;  // X loads in flight per lane
        for (int64_t base = s0; base < s1; base += 4 * UN) {
          double av[UN];
          int iu[UN], ju[UN];
          bool vu[UN];
#pragma unroll
          for (int u = 0; u < UN; ++u) {
            vu[u] = ij < s1;
            av[u] = (vu[u] && kr < K) ? __ldg(X + ij * K + kr) : 0.0;
            iu[u] = static_cast<int>(ii);
            ju[u] = static_cast<int>(jj);
            ij += 4;
            jj += 4;
            while (jj >= J) {
              jj -= J;
              ++ii;
            }
          }
#pragma unroll
          for (int u = 0; u < UN; ++u) {
            double w0 = 0.0, w1 = 0.0;
            if (vu[u]) {
              if (gq < R) w0 = F[0][iu[u] * R + gq] * F[1][ju[u] * R + gq];
              if (8 + gq < R) w1 = F[0][iu[u] * R + 8 + gq] * F[1][ju[u] * R + 8 + gq];
            }
            dmma884(c00, c01, av[u], w0);
            if (R > 8) dmma884(c10, c11, av[u], w1);
          }
        }
        double* pp = part + ((int64_t)ch * K) * 16;
        if (kr < K) {
          pp[kr * 16 + 2 * tq] = c00;
          pp[kr * 16 + 2 * tq + 1] = c01;
          pp[kr * 16 + 8 + 2 * tq] = c10;
          pp[kr * 16 + 9 + 2 * tq] = c11;
        }
      }
      __syncthreads();
      for (int e = tid; e < K * R; e += nt) {
        const int kk = e / R, r = e % R;
        double s = 0.0;
        for (int ch = 0; ch < chunks; ++ch) s += part[((int64_t)ch * K + kk) * 16 + r];
        M[e] = s;
      }
    }
    __syncthreads();
    if (it == 1 && tid == 0) g_small_clk[6] = clock64();
    solve(2, 0, 1, true);   // sets glam-equivalent nrm, fit_s, explicit_s
    if (it == 1 && tid == 0) g_small_clk[7] = clock64();
    if (explicit_s != 0.0) {
      // ||X - [[A lam, B, C]]||^2, one (i, j) row per thread pass
      double loc = 0.0;
      for (int64_t ij = tid; ij < (int64_t)I * J; ij += nt) {
        const int64_t i = ij / J, j = ij % J;
        double wb[SMALL_RS];
#pragma unroll
        for (int r = 0; r < SMALL_RS; ++r)
          wb[r] = (r < R) ? F[0][i * R + r] * nrm[r] * F[1][j * R + r] : 0.0;
        const double* xr = X + ij * K;
        for (int kk = 0; kk < K; ++kk) {
          double xh = 0.0;
#pragma unroll
          for (int r = 0; r < SMALL_RS; ++r)
            if (r < R) xh = fma(wb[r], F[2][kk * R + r], xh);
          const double d = __ldg(xr + kk) - xh;
          loc = fma(d, d, loc);
        }
      }
      const double res2 = small_block_sum(loc, red);
      if (tid == 0) fit_s = 1.0 - sqrt(res2) / sqrt(x2);
    }
    __syncthreads();
    if (it == 1 && tid == 0) g_small_clk[8] = clock64();
    if (tid == 0) {
      const double fit = fit_s;
      fit_hist[it] = fit;
      if (tol > 0.0 && fabs(fit - prev) < tol) stop = 1;
      prev = fit;
    }
    __syncthreads();
    if (stop) {
      conv = 1;
      ++it;
      break;
    }
  }
  if (it > max_iters) it = max_iters;
  // outputs: x = F0 * lam (KruskalRep.x), normalised F1, F2, lam
  for (int e = tid; e < I * R; e += nt) ga[e] = F[0][e] * nrm[e % R];
  for (int e = tid; e < J * R; e += nt) gb[e] = F[1][e];
  for (int e = tid; e < K * R; e += nt) gc[e] = F[2][e];
  for (int r = tid; r < R; r += nt) glam[r] = nrm[r];
  if (tid == 0) {
    out_info[0] = it;
    out_info[1] = conv;
  }
}

#include "cp_cluster.cuh"

// ---------------------------------------------------------------------------
// solve: F_un = (sum_s Mpart[s]) @ Vp ; per-CTA Gram + <F_un, M> partials
// ---------------------------------------------------------------------------

constexpr int SOLVE_ROWS = 32;  // rows of F per CTA

__global__ void __launch_bounds__(256)
    solve_apply_kernel(const double* __restrict__ mpart, int64_t nparts, int64_t part_stride,
                       int64_t row_stride, const double* __restrict__ vp, int64_t rows, int R, double* __restrict__ f,
                       double* __restrict__ gram_part, double* __restrict__ inner_part) {
  extern __shared__ __align__(16) double sm[];
  double* ms = sm;                     // SOLVE_ROWS x R  (reduced M rows)
  double* fs = ms + SOLVE_ROWS * R;    // SOLVE_ROWS x R  (F_un rows)
  double* vs = fs + SOLVE_ROWS * R;    // R x R
  const int64_t r0 = blockIdx.x * (int64_t)SOLVE_ROWS;
  const int nr = static_cast<int>(rows - r0 < SOLVE_ROWS ? rows - r0 : SOLVE_ROWS);
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) vs[idx] = vp[idx];
  for (int idx = threadIdx.x; idx < SOLVE_ROWS * R; idx += blockDim.x) {
    const int rr = idx / R;
    double s = 0.0;
    if (rr < nr) {
      const double* src = mpart + (r0 + rr) * row_stride + idx % R;
      for (int64_t p = 0; p < nparts; ++p) s += src[p * part_stride];
    }
    ms[idx] = s;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < SOLVE_ROWS * R; idx += blockDim.x) {
    const int rr = idx / R, c = idx % R;
    double s = 0.0;
    for (int k = 0; k < R; ++k) s = fma(ms[rr * R + k], vs[k * R + c], s);
    fs[idx] = s;
    if (rr < nr) f[(r0 + rr) * R + c] = s;
  }
  __syncthreads();
  double* gp = gram_part + blockIdx.x * (int64_t)R * R;
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
    const int a = idx / R, b = idx % R;
    double s = 0.0;
    for (int rr = 0; rr < nr; ++rr) s = fma(fs[rr * R + a], fs[rr * R + b], s);
    gp[idx] = s;
  }
  if (inner_part != nullptr) {
    __shared__ double red[8];
    double s = 0.0;
    for (int idx = threadIdx.x; idx < nr * R; idx += blockDim.x) s = fma(fs[idx], ms[idx], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      inner_part[blockIdx.x] = t;
    }
  }
}

// Device-side state of one CP-ALS run.
struct CpState {
  double* gram[3];     // normalised Grams G_k = F_k^T F_k
  double* vp;          // R x R
  double* norms;       // R
  double* lam;         // R
  double* scal;        // [0] ||X||^2, [1] <X,Xhat>, [2] explicit residual^2, [3] use_explicit
  double* fit_hist;    // max_iters
  int* iter;           // device sweep index, read by kernels launched with it < 0 (graph replay)
};

__global__ void set_iter_kernel(int* iter, int v) {
  if (threadIdx.x == 0) *iter = v;
}
__global__ void advance_iter_kernel(int* iter) {
  if (threadIdx.x == 0) *iter += 1;
}

// Sum the per-CTA Gram partials (and <F_un, M> partials) of one solve into
// gbuf = [G_un (R*R), inner, 0] -- the buffer a mode-3-sharded caller sums
// across ranks before the finish.
__device__ __forceinline__ double warp_ordered_sum(const double* __restrict__ p, int64_t n) {
  double s = 0.0;
  for (int64_t k = threadIdx.x & 31; k < n; k += 32) s += p[k];
  return warp_sum(s);
}

__global__ void __launch_bounds__(256)
    gram_reduce_kernel(const double* __restrict__ gram_part, int64_t nparts, int R,
                       const double* __restrict__ inner_part, double* __restrict__ gbuf) {
  // one thread per Gram entry across the grid (was one CTA for all R*R:
  // 255 us per solve at R = 64, I = 4096); same per-entry summation order
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < R * R;
       idx += gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll 4
    for (int64_t p = 0; p < nparts; ++p) s += gram_part[p * R * R + idx];
    gbuf[idx] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const double inner = inner_part ? warp_ordered_sum(inner_part, nparts) : 0.0;
    if (threadIdx.x == 0) {
      gbuf[R * R] = inner;
      gbuf[R * R + 1] = 0.0;
    }
  }
}

// Column norms (0 -> 1) from the Gram diagonal, normalised Gram; the mode-3
// update also sets lambda, the Gram-identity fit and the explicit decision.
__global__ void __launch_bounds__(256)
    solve_finish_kernel(const double* __restrict__ gbuf, int R, double* __restrict__ norms,
                        double* __restrict__ gram_out, double* __restrict__ lam, CpState st,
                        int it, int fit_mode) {
  if (it < 0) it = *st.iter;
  __shared__ double nrm[PINV_MAX_R];
  __shared__ double red[8];
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    double v = sqrt(gbuf[r * R + r]);
    if (v == 0.0) v = 1.0;
    nrm[r] = v;
    norms[r] = v;
    if (lam) lam[r] = v;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
    const int a = idx / R, b = idx % R;
    gram_out[idx] = gbuf[idx] / (nrm[a] * nrm[b]);
  }
  if (lam == nullptr) return;
  __syncthreads();
  // ||Xhat||^2 = lam^T (G0 o G1 o G2) lam ; <X, Xhat> = sum(C_un o M3)
  double s = 0.0;
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
    const int a = idx / R, b = idx % R;
    s += nrm[a] * nrm[b] * st.gram[0][idx] * st.gram[1][idx] * st.gram[2][idx];
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double xh2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) xh2 += red[w];
    const double inner = gbuf[R * R];
    const double x2 = st.scal[0];
    const double res2 = fmax(x2 - 2.0 * inner + xh2, 0.0);
    const double relres = sqrt(res2 / x2);
    st.scal[1] = inner;
    // identity error ~ c*eps*||X||^2 / (2 res): switch to the explicit
    // residual once the relative residual is small enough to lose digits
    const bool explicit_fit = (fit_mode == 1) || (fit_mode == 0 && relres < 1e-3);
    st.scal[3] = explicit_fit ? 1.0 : 0.0;
    st.fit_hist[it] = 1.0 - relres;
  }
}

__global__ void scale_cols_kernel(double* __restrict__ f, int64_t rows, int R,
                                  const double* __restrict__ norms) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < rows * R;
       idx += (int64_t)gridDim.x * blockDim.x)
    f[idx] = f[idx] / norms[idx % R];
}

__global__ void gram_kernel(const double* __restrict__ f, int64_t rows, int R,
                            double* __restrict__ g) {
  // small: one CTA, fixed order over rows
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) {
    const int a = idx / R, b = idx % R;
    double s = 0.0;
    for (int64_t r = 0; r < rows; ++r) s = fma(f[r * R + a], f[r * R + b], s);
    g[idx] = s;
  }
}

// W = A * lam (row scale for the explicit residual)
__global__ void lam_scale_kernel(const double* a, const double* __restrict__ lam, int64_t rows,
                                 int R, double* w) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < rows * R;
       idx += (int64_t)gridDim.x * blockDim.x)
    w[idx] = a[idx] * lam[idx % R];
}

// ---------------------------------------------------------------------------
// explicit residual ||X - [[lam; A, B, C]]||^2 (decomp.py:395-396, fused)
// Xhat tile (j-rows x k-cols) for fixed i = (B o W_i) C^T on DMMA; epilogue
// subtracts X and accumulates squares.  Persistent grid; exits at once when
// the Gram identity was judged accurate (scal[3] == 0).
// ---------------------------------------------------------------------------

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS)
    residual_kernel(BtGemmArgs g, const double* __restrict__ X, int64_t J, int64_t K,
                    int64_t tiles_total, const double* __restrict__ flag,
                    double* __restrict__ part) {
  extern __shared__ __align__(16) double smem_dyn[];
  __shared__ double red[Cfg::THREADS / 32];
  if (flag != nullptr && *flag == 0.0) {
    if (threadIdx.x == 0) part[blockIdx.x] = 0.0;
    return;
  }
  const int64_t tiles_m = (J + Cfg::BM - 1) / Cfg::BM;
  const int64_t tiles_n = (K + Cfg::BN - 1) / Cfg::BN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WM) * Cfg::TM;
  const int wn0 = (warp / Cfg::WM) * Cfg::TN;
  const int64_t KT = (g.Kin + Cfg::BK - 1) / Cfg::BK;
  double local = 0.0;
  for (int64_t tile = blockIdx.x; tile < tiles_total; tile += gridDim.x) {
    const int64_t i = tile / (tiles_m * tiles_n);
    const int64_t rem = tile % (tiles_m * tiles_n);
    const int64_t tm = rem % tiles_m, tn = rem / tiles_m;
    const int64_t m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;
    double acc[Cfg::FM][Cfg::FN][2];
    __syncthreads();
    bt_gemm_mainloop<Cfg>(g, i, m0, n0, 0, KT, acc, smem_dyn);
    const double* xi = X + i * J * K;
#pragma unroll
    for (int fi = 0; fi < Cfg::FM; ++fi) {
      const int64_t j = m0 + wm0 + fi * 8 + gq;
      if (j >= J) continue;
#pragma unroll
      for (int fj = 0; fj < Cfg::FN; ++fj)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t k = n0 + wn0 + fj * 8 + 2 * tq + h;
          if (k < K) {
            const double d = ld_stream(xi + j * K + k) - acc[fi][fj][h];
            local = fma(d, d, local);
          }
        }
    }
  }
  local = warp_sum(local);
  if (lane == 0) red[warp] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < Cfg::THREADS / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

// Explicit residual for small ranks (R <= RS, e.g. C4's R = 16), where the
// DMMA tile version is latency bound (a K = R reduction per X tile): a warp
// owns a 32-wide k chunk -- C[k, :] in registers -- and streams (i, j) rows
// of X with coalesced loads; Xhat[i][j][k] = sum_r (W[i][r] B[j][r]) C[k][r].
// The row factors W[i] o B[j] of the warp's rows are formed once into
// shared memory (each lane two products per row instead of 2 R loads per
// element) and read back as broadcast double2.  Fixed-order sums
// (deterministic); X read once.
template <int RS>
__global__ void __launch_bounds__(256)
    residual_small_kernel(const double* __restrict__ X, const double* __restrict__ W,
                          const double* __restrict__ Bf, const double* __restrict__ Cf, int64_t I,
                          int64_t J, int64_t K, int R, const double* __restrict__ flag,
                          double* __restrict__ part) {
  constexpr int ROWS = 512 / RS;  // 32 KB of row factors per CTA
  __shared__ __align__(16) double wbs[8][ROWS * RS];
  __shared__ double red[8];
  if (flag != nullptr && *flag == 0.0) {
    if (threadIdx.x == 0) part[blockIdx.x] = 0.0;
    return;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* wb = wbs[wid];
  const int64_t kchunks = (K + 31) / 32;
  const int64_t gw = blockIdx.x * (int64_t)(blockDim.x >> 5) + wid;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  double local = 0.0;
  // warp work item: (k chunk, row group of ROWS (i, j) rows)
  const int64_t rows = I * J;
  const int64_t groups = (rows + ROWS - 1) / ROWS;
  for (int64_t item = gw; item < kchunks * groups; item += nwarps) {
    const int64_t kc = item % kchunks, g = item / kchunks;
    const int64_t k = kc * 32 + lane;
    double c[RS];
#pragma unroll
    for (int r = 0; r < RS; ++r) c[r] = (k < K && r < R) ? __ldg(Cf + k * R + r) : 0.0;
    const int64_t r0 = g * ROWS, r1 = r0 + ROWS < rows ? r0 + ROWS : rows;
    __syncwarp();
    for (int e = lane; e < ROWS * RS; e += 32) {
      const int rr = e / RS, r = e - rr * RS;
      const int64_t row = r0 + rr;
      double v = 0.0;
      if (row < r1 && r < R) {
        const int64_t i = row / J, j = row - i * J;
        v = __ldg(W + i * R + r) * __ldg(Bf + j * R + r);
      }
      wb[e] = v;
    }
    __syncwarp();
    constexpr int UR = 4;  // independent X loads in flight per lane
    for (int64_t row = r0; row < r1; row += UR) {
      double xv[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u)
        xv[u] = (row + u < r1 && k < K) ? ld_stream(X + (row + u) * K + k) : 0.0;
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        if (row + u >= r1) break;
        const double2* w2 = reinterpret_cast<const double2*>(wb + (row + u - r0) * RS);
        double xh = 0.0;
#pragma unroll
        for (int r = 0; r < RS / 2; ++r) {
          const double2 w = w2[r];
          xh = fma(w.x, c[2 * r], xh);
          xh = fma(w.y, c[2 * r + 1], xh);
        }
        if (k < K) {
          const double d = xv[u] - xh;
          local = fma(d, d, local);
        }
      }
    }
  }
  local = warp_sum(local);
  if (lane == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

// Fixed-order warp sum of n partials (lane-strided runs, then a fixed
// shuffle tree): deterministic, and no 1-thread chain of dependent loads.
__global__ void residual_reduce_kernel(const double* __restrict__ part, int n,
                                       double* __restrict__ out) {
  const double s = warp_ordered_sum(part, n);
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void residual_finish_kernel(const double* __restrict__ res2, CpState st, int it) {
  if (it < 0) it = *st.iter;
  if (threadIdx.x != 0) return;
  if (st.scal[3] == 0.0) return;
  st.scal[2] = res2[0];
  st.fit_hist[it] = 1.0 - sqrt(res2[0]) / sqrt(st.scal[0]);
}

// buf[0] = sum of squares partial result copy (init finish helper)
__global__ void copy_scalar_kernel(const double* __restrict__ src, double* __restrict__ dst) {
  if (threadIdx.x == 0) dst[0] = src[0];
}

// ---------------------------------------------------------------------------
// host-side plan
// ---------------------------------------------------------------------------

template <int BN, int VARIANT = 0>
struct TreeCfgSel;
template <int VARIANT>
struct TreeCfgSel<64, VARIANT> {
  // 128x64 tile, 4 warps of 64x32, 3 stages, 2 CTAs/SM (the tuned all-warps
  // variant; profiles/r01_fp64_and_tuning.md lists the configurations tried)
  template <int V>
  using Cfg = GemmCfg<128, 64, 16, 2, 2, 3, true, false, V>;
};
template <int VARIANT>
struct TreeCfgSel<16, VARIANT> {
  template <int V>
  using Cfg = GemmCfg<128, 16, 16, 8, 1, 4, true, false, V>;
};
template <int VARIANT>
struct TreeCfgSel<8, VARIANT> {
  template <int V>
  using Cfg = GemmCfg<128, 8, 16, 8, 1, 4, true, false, V>;
};

int tree_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BT_TREE_CFG");
    // 11 (default): warp-specialised with the X tile by TMA, 4 unpadded
    // swizzled stages (tree_p_tma_kernel); 9: the same with a cp.async
    // producer and 3 padded stages (tree_p_ws_kernel: 72.5 ms on C5); 6:
    // the same tile with all warps loading and computing: 73.5 ms
    v = e ? atoi(e) : 11;
  }
  return v;
}

// residual: rows j, cols k, reduction r (K-contig on both sides)
template <int V>
using ResCfg = GemmCfg<128, 64, 16, 4, 2, 3, true, true, V>;

int tree_bn(int64_t R) { return R <= 8 ? 8 : (R <= 16 ? 16 : 64); }

int tree_bm(int) { return 128; }

struct Plan {
  int64_t I, J, K, R;
  int bn;          // tree-P tile width
  int64_t jtiles;  // tree-P row tiles per i
  int64_t s2;      // i-chunks for mode 2
  int64_t chunk2;
  int64_t solve_parts_max;
  int res_grid;
  // workspace layout (doubles)
  int64_t off_p, off_m1, off_m2, off_m3, off_m3ws, off_gp, off_ip, off_f, off_state, off_res,
      off_w, off_m1d, off_m2d, off_gbuf, off_init, off_res1, total;
  int64_t m3_ws_elems;
  // dimension-tree root.  0: P = X x3 C (I x J x R; modes 1 and 2 from P,
  // mode 3 a full GEMM).  1: Q = X x1 A_new (J x K x R; mode 1 from the tree
  // kernel's fused epilogue with no P store, modes 2 and 3 from Q) -- chosen
  // whenever K <= I (C5, and a rank's mode-3 slab at any GPU count), where P
  // would be I*J*R (8.6 GB at C5 written and re-read every sweep) while Q is
  // J*K*R
  int qtree;
  int64_t s3, chunk3;  // j-chunks of the mode-3 reduction from Q
  // Q tree with a short mode-3 slab (K <= 256, i.e. <= 16 k-tiles per tree
  // tile): mode 1 as T[i] = X[i]^T B (batched over i, the reduction over J
  // is long) then m1[i][r] = sum_k T[i][k][r] C[k][r]
  int m1_via_t;
  int64_t off_t;
  int64_t off_jstore;
};

BtGemmArgs mode3_args(const Plan& pl, const double* X, const double* A, const double* B,
                      double* out) {
  BtGemmArgs g{};
  g.M = pl.K;
  g.N = pl.R;
  g.Kin = pl.J;
  g.Kout = pl.I;
  g.A = BtOperand{X, 1, pl.J * pl.K, pl.K, 0};
  g.B = BtOperand{B, 1, 0, pl.R, 0};
  g.bscale = A;
  g.s_scale_ko = pl.R;
  g.C = out;
  g.sCm = pl.R;
  g.sCn = 1;
  g.alpha = 1.0;
  g.beta = 0.0;
  return g;
}

// Q[(j,k)][r] = sum_i X[i][j][k] A[i][r]  (rows (j,k) M-contiguous in X)
BtGemmArgs qtree_args(const Plan& pl, const double* X, const double* A, double* Q) {
  BtGemmArgs g{};
  g.M = pl.J * pl.K;
  g.N = pl.R;
  g.Kin = pl.I;
  g.Kout = 1;
  g.A = BtOperand{X, 1, 0, pl.J * pl.K, 0};
  g.B = BtOperand{A, 1, 0, pl.R, 0};
  g.C = Q;
  g.sCm = pl.R;
  g.sCn = 1;
  g.alpha = 1.0;
  g.beta = 0.0;
  return g;
}

// T[i][k][r] = sum_j X[i][j][k] B[j][r]: batch i, rows k M-contiguous
BtGemmArgs tslab_args(const Plan& pl, const double* X, const double* B, double* T) {
  BtGemmArgs g{};
  g.M = pl.K;
  g.N = pl.R;
  g.Kin = pl.J;
  g.Kout = 1;
  g.A = BtOperand{X, 1, 0, pl.K, pl.J * pl.K};
  g.B = BtOperand{B, 1, 0, pl.R, 0};
  g.C = T;
  g.sCm = pl.R;
  g.sCn = 1;
  g.sCb = pl.K * pl.R;
  g.alpha = 1.0;
  g.beta = 0.0;
  return g;
}

int cp_tree_variant(int64_t I, int64_t J, int64_t K, int64_t R) {
  static const char* e = getenv("BT_CP_TREE");  // A/B switch (tools/scale_proxy.py)
  if (e && e[0] == 'p') return 0;
  if (e && e[0] == 'q') return 1;
  (void)J;
  // Q (J*K*R) is no larger than P (I*J*R) and the Q GEMM (X rows
  // M-contiguous, no operand scale) beats the mode-3 GEMM with its
  // Khatri-Rao B-scale: C5 sweep 153.4 -> 149.8 ms at K = 1024, 24.1 -> 22.4
  // ms at a rank's K = 128 slab.  R <= 16 keeps the narrow-tile P tree (C4).
  return (R > 16 && K <= I) ? 1 : 0;
}

// variant < 0: the cp_tree_variant rule; the standalone bt_mttkrp_f64
// (one mode, P layout) passes 0
Plan make_plan(const bt_cp_problem* pb, int variant = -1) {
  Plan pl;
  pl.I = pb->I;
  pl.J = pb->J;
  pl.K = pb->K;
  pl.R = pb->R;
  pl.bn = tree_bn(pl.R);
  pl.jtiles = bt_cdiv(pl.J, tree_bm(pl.bn));
  const int64_t JR = pl.J * pl.R;
  // mode 2: enough CTAs along (j, r) x i-chunks to fill the GPU ~4x
  const int64_t blocks_jr = std::max<int64_t>(1, std::min<int64_t>(bt_cdiv(JR, 256), 2048));
  pl.s2 = std::max<int64_t>(1, std::min<int64_t>(pl.I, bt_cdiv(4 * bt_num_sms(), blocks_jr)));
  pl.chunk2 = bt_cdiv(pl.I, pl.s2);
  pl.s2 = bt_cdiv(pl.I, pl.chunk2);
  const int64_t maxrows = std::max(pl.I, std::max(pl.J, pl.K));
  pl.solve_parts_max = bt_cdiv(maxrows, SOLVE_ROWS);
  pl.res_grid = 8 * bt_num_sms();
  pl.qtree = variant < 0 ? cp_tree_variant(pl.I, pl.J, pl.K, pl.R) : variant;
  {
    const int64_t KR = pl.K * pl.R;
    const int64_t blocks_kr = std::max<int64_t>(1, std::min<int64_t>(bt_cdiv(KR, 256), 2048));
    pl.s3 = std::max<int64_t>(1, std::min<int64_t>(pl.J, bt_cdiv(4 * bt_num_sms(), blocks_kr)));
    pl.chunk3 = bt_cdiv(pl.J, pl.s3);
    pl.s3 = bt_cdiv(pl.J, pl.chunk3);
  }
  BtGemmArgs g3 = mode3_args(pl, nullptr, nullptr, nullptr, nullptr);
  pl.m3_ws_elems = bt_gemm_ws_elems(g3, 1);
  if (pl.qtree) pl.m3_ws_elems = bt_gemm_ws_elems(qtree_args(pl, nullptr, nullptr, nullptr), 1);
  pl.m1_via_t = pl.qtree && pl.K <= 256 && pl.I <= 65535;
  const int64_t RR = pl.R * pl.R;
  int64_t o = 0;
  auto take = [&](int64_t n) {
    int64_t at = o;
    o += (n + 1) / 2 * 2;  // keep 16-byte alignment
    return at;
  };
  pl.off_p = take(pl.qtree ? pl.J * pl.K * pl.R : pl.I * pl.J * pl.R);   // P or Q
  pl.off_m1 = take(pl.I * pl.jtiles * pl.R);
  pl.off_t = take(pl.m1_via_t ? pl.I * pl.K * pl.R : 0);
  pl.off_m2 = take(pl.qtree ? pl.s3 * pl.K * pl.R : pl.s2 * JR);
  pl.off_m3 = take(pl.K * pl.R);
  pl.off_m3ws = take(pl.m3_ws_elems);
  pl.off_gp = take(std::max<int64_t>(pl.solve_parts_max, 64) * RR);  // also Gram split-K partials
  pl.off_ip = take(pl.solve_parts_max);
  pl.off_f = take(maxrows * pl.R);
  pl.off_state = take(3 * RR + RR + 2 * pl.R + 8);
  pl.off_res = take(std::max<int64_t>(pl.res_grid, 2048));
  pl.off_w = take(pl.I * pl.R);
  pl.off_m1d = take(pl.I * pl.R);
  pl.off_m2d = take(pl.J * pl.R);
  pl.off_gbuf = take(pl.R * pl.R + 2);
  pl.off_init = take(pl.R * pl.R + 2);
  pl.off_res1 = take(2);
  pl.off_jstore = take(3 * 16 * 16);   // warm-start rotations of the R <= 16 pinv, per mode
  pl.total = o;
  return pl;
}

// warp-specialised tree kernel (BT_TREE_CFG=9): 128x64 tile, 2x2 consumer
// warps + 1 producer warp, 3 stages, 2 CTAs per SM
template <int V>
int launch_tree_ws(const Plan& pl, const double* X, const double* C, const double* B, double* P,
                   double* m1part, int store_p, cudaStream_t st) {
  using Cfg = GemmCfg<128, 64, 16, 2, 2, 3, true, false, V>;
  BtGemmArgs g{};
  g.M = pl.J;
  g.N = pl.R;
  g.Kin = pl.K;
  g.Kout = 1;
  g.A = BtOperand{X, pl.K, 0, 1, pl.J * pl.K};
  g.B = BtOperand{C, 1, 0, pl.R, 0};
  g.C = P;
  g.sCm = pl.R;
  g.sCn = 1;
  g.sCb = pl.J * pl.R;
  g.alpha = 1.0;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(tree_p_ws_kernel<Cfg>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES));
    attr = true;
  }
  BT_REQUIRE(pl.I <= 65535, BT_E_SHAPE, "cp: mode-1 extent %lld exceeds 65535", (long long)pl.I);
  dim3 grid(static_cast<unsigned>(bt_cdiv(pl.J, Cfg::BM)), static_cast<unsigned>(bt_cdiv(pl.R, 64)),
            static_cast<unsigned>(pl.I));
  tree_p_ws_kernel<Cfg><<<grid, Cfg::THREADS + 32, Cfg::SMEM_BYTES, st>>>(g, B, pl.R, m1part,
                                                                          pl.jtiles, store_p);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// TMA tree kernel (default for R > 16 with K even; BT_TREE_CFG=9 keeps the
// cp.async producer of tree_p_ws_kernel for A/B runs)
template <class T>
int launch_tree_tma_t(const Plan& pl, const double* X, const double* C, const double* B, double* P,
                    double* m1part, int store_p, cudaStream_t st) {
  BtGemmArgs g{};
  g.M = pl.J;
  g.N = pl.R;
  g.Kin = pl.K;
  g.Kout = 1;
  g.A = BtOperand{X, pl.K, 0, 1, pl.J * pl.K};
  g.B = BtOperand{C, 1, 0, pl.R, 0};
  g.C = P;
  g.sCm = pl.R;
  g.sCn = 1;
  g.sCb = pl.J * pl.R;
  g.alpha = 1.0;
  CUtensorMap xmap, cmap;
  BT_TRY(bt_tma_map_f64_3d(&xmap, X, pl.K, pl.J, pl.I, pl.K, pl.J * pl.K, T::BK, T::BM, 1));
  BT_TRY(bt_tma_map_f64_2d(&cmap, C, pl.R, pl.K, pl.R, 16, T::BK));
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(tree_p_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       T::SMEM_BYTES));
    attr = true;
  }
  BT_REQUIRE(pl.I <= 65535, BT_E_SHAPE, "cp: mode-1 extent %lld exceeds 65535", (long long)pl.I);
  dim3 grid(static_cast<unsigned>(bt_cdiv(pl.J, T::BM)), static_cast<unsigned>(bt_cdiv(pl.R, T::BN)),
            static_cast<unsigned>(pl.I));
  tree_p_tma_kernel<T><<<grid, T::THREADS, T::SMEM_BYTES, st>>>(xmap, cmap, g, B, pl.R, m1part, pl.jtiles,
                                                            store_p);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// Y (rows x R) = X (rows x K, row-major) U (K x R, row-major) on the TMA tree
// kernel without its reduction epilogue: the tensor-times-matrix over the
// LAST mode (tucker.cu bt_ttm_f64; K and R even for the 16-byte TMA strides)
int ttm_last_tma_impl(const double* x, int64_t rows, int64_t K, const double* u, int64_t R,
                      double* y, cudaStream_t st) {
  using T = TreeTma;
  BtGemmArgs g{};
  g.M = rows;
  g.N = R;
  g.Kin = K;
  g.Kout = 1;
  g.A = BtOperand{x, K, 0, 1, rows * K};
  g.B = BtOperand{u, 1, 0, R, 0};
  g.C = y;
  g.sCm = R;
  g.sCn = 1;
  g.sCb = rows * R;
  g.alpha = 1.0;
  CUtensorMap xmap, cmap;
  BT_TRY(bt_tma_map_f64_3d(&xmap, x, K, rows, 1, K, rows * K, T::BK, T::BM, 1));
  BT_TRY(bt_tma_map_f64_2d(&cmap, u, R, K, R, 16, T::BK));
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(tree_p_tma_kernel<T, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM_BYTES));
    attr = true;
  }
  dim3 grid(static_cast<unsigned>(bt_cdiv(rows, T::BM)), static_cast<unsigned>(bt_cdiv(R, T::BN)), 1);
  tree_p_tma_kernel<T, false><<<grid, T::THREADS, T::SMEM_BYTES, st>>>(xmap, cmap, g, nullptr, R,
                                                                       nullptr, 1, 1);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// (a 3-stage, 3-CTA/SM variant was tried: at the 168-register cap it spills
// ~300 bytes per thread, so the 4-stage, 2-CTA configuration stays)
int launch_tree_tma(const Plan& pl, const double* X, const double* C, const double* B, double* P,
                    double* m1part, int store_p, cudaStream_t st) {
  return launch_tree_tma_t<TreeTma>(pl, X, C, B, P, m1part, store_p, st);
}

template <int BN, int V, int VAR = 0>
int launch_tree(const Plan& pl, const double* X, const double* C, const double* B, double* P,
                double* m1part, int store_p, cudaStream_t st) {
  using Cfg = typename TreeCfgSel<BN, VAR>::template Cfg<V>;
  BtGemmArgs g{};
  g.M = pl.J;
  g.N = pl.R;
  g.Kin = pl.K;
  g.Kout = 1;
  g.A = BtOperand{X, pl.K, 0, 1, pl.J * pl.K};
  g.B = BtOperand{C, 1, 0, pl.R, 0};
  g.C = P;
  g.sCm = pl.R;
  g.sCn = 1;
  g.sCb = pl.J * pl.R;
  g.alpha = 1.0;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(tree_p_kernel<Cfg>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES));
    attr = true;
  }
  BT_REQUIRE(pl.I <= 65535, BT_E_SHAPE, "cp: mode-1 extent %lld exceeds 65535",
             (long long)pl.I);
  dim3 grid(static_cast<unsigned>(bt_cdiv(pl.J, Cfg::BM)), static_cast<unsigned>(bt_cdiv(pl.R, BN)),
            static_cast<unsigned>(pl.I));
  tree_p_kernel<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(g, B, pl.R, m1part, pl.jtiles,
                                                                   store_p);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

int run_tree(const Plan& pl, const double* X, const double* C, const double* B, double* P,
             double* m1part, int store_p, cudaStream_t st) {
  const bool v2 = (pl.K % 2 == 0) && (pl.R % 2 == 0) &&
                  ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(C)) & 15u) == 0;
  switch (pl.bn) {
    case 8:
      return v2 ? launch_tree<8, 2>(pl, X, C, B, P, m1part, store_p, st)
                : launch_tree<8, 1>(pl, X, C, B, P, m1part, store_p, st);
    case 16:
      return v2 ? launch_tree<16, 2>(pl, X, C, B, P, m1part, store_p, st)
                : launch_tree<16, 1>(pl, X, C, B, P, m1part, store_p, st);
    default:
      if (v2) {
        const int tv = tree_variant();
        if (tv == 6) return launch_tree<64, 2>(pl, X, C, B, P, m1part, store_p, st);
        if (tv == 9 || pl.K > INT32_MAX || pl.J > INT32_MAX)
          return launch_tree_ws<2>(pl, X, C, B, P, m1part, store_p, st);
        return launch_tree_tma(pl, X, C, B, P, m1part, store_p, st);
      }
      return launch_tree<64, 1>(pl, X, C, B, P, m1part, store_p, st);
  }
}

int run_mode2(const Plan& pl, const double* P, const double* A, double* m2part, cudaStream_t st) {
  const int64_t JR = pl.J * pl.R;
  const int64_t bx = std::max<int64_t>(1, std::min<int64_t>(bt_cdiv(JR, 256), 2048));
  mode2_from_p_kernel<<<dim3(static_cast<unsigned>(bx), static_cast<unsigned>(pl.s2)), 256, 0,
                        st>>>(P, A, pl.I, JR, pl.R, pl.chunk2, m2part);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

int run_mode3(const Plan& pl, const double* X, const double* A, const double* B, double* out,
              double* ws, cudaStream_t st) {
  BtGemmArgs g = mode3_args(pl, X, A, B, out);
  g.ws = ws;
  return bt_gemm_run(g, 1, st, 0, pl.m3_ws_elems);
}

template <int NP>
int launch_pinv_fast(const double* g0, const double* g1, int R, double* vp, cudaStream_t st) {
  constexpr int SM = 3 * NP * (NP + 1) * 8;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(pinv_fast_kernel<NP>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    attr = true;
  }
  // barrier cost grows with the CTA: small systems take small CTAs
  constexpr int THREADS = NP <= 16 ? 64 : 256;
  pinv_fast_kernel<NP><<<1, THREADS, SM, st>>>(g0, g1, R, vp);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// BT_PINV_1S=0: the shared-memory Cholesky-first / two-sided Jacobi pinv for
// R <= 16 as well (A/B runs)
static bool use_pinv_1s() {
  static const int v = [] {
    const char* e = getenv("BT_PINV_1S");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v != 0;
}

int run_pinv(const double* g0, const double* g1, int R, double* vp, cudaStream_t st,
             double* jstore = nullptr, int warm = 0) {
  if (R <= 16 && use_pinv_1s()) {
    if (R <= 8)
      pinv_jacobi1_kernel<8><<<1, 32, 0, st>>>(g0, g1, R, vp, jstore, warm);
    else
      pinv_jacobi1_kernel<16><<<1, 32, 0, st>>>(g0, g1, R, vp, jstore, warm);
    BT_LAUNCH_CHECK();
    return BT_OK;
  }
  if (R <= 8) return launch_pinv_fast<8>(g0, g1, R, vp, st);
  if (R <= 16) return launch_pinv_fast<16>(g0, g1, R, vp, st);
  if (R <= 32) return launch_pinv_fast<32>(g0, g1, R, vp, st);
  if (R <= 64) return launch_pinv_fast<64>(g0, g1, R, vp, st);
  return launch_pinv_fast<96>(g0, g1, R, vp, st);  // R <= PINV_MAX_R is enforced upstream
}

// Factor update, local half: Vp = pinv(G_o0 o G_o1), F_un = M Vp (M summed
// over nparts partials), gbuf = [F_un^T F_un, <F_un, M>] (summed over CTAs).
int run_solve_rows(const Plan& pl, const CpState& s, double* ws, const double* mpart,
                   int64_t nparts, int64_t part_stride, int64_t row_stride, int64_t rows, int go0,
                   int go1, double* F, bool with_inner, double* gbuf, cudaStream_t st,
                   bool pinv_done = false) {
  const int R = static_cast<int>(pl.R);
  if (!pinv_done) BT_TRY(run_pinv(s.gram[go0], s.gram[go1], R, s.vp, st));
  const int64_t parts = bt_cdiv(rows, SOLVE_ROWS);
  double* gp = ws + pl.off_gp;
  double* ip = ws + pl.off_ip;
  const size_t sm = (size_t)(2 * SOLVE_ROWS * R + R * R) * 8;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(solve_apply_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (2 * SOLVE_ROWS * PINV_MAX_R + PINV_MAX_R * PINV_MAX_R) * 8));
    attr = true;
  }
  if (parts > 0) {
    solve_apply_kernel<<<static_cast<unsigned>(parts), 256, sm, st>>>(
        mpart, nparts, part_stride, row_stride, s.vp, rows, R, F, gp, with_inner ? ip : nullptr);
    BT_LAUNCH_CHECK();
  }
  gram_reduce_kernel<<<static_cast<unsigned>(bt_cdiv(static_cast<int64_t>(R) * R, 256)), 256, 0,
                       st>>>(gp, parts, R, with_inner ? ip : nullptr, gbuf);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// Factor update, finishing half (after a possible cross-rank sum of gbuf).
int run_solve_finish(const Plan& pl, const CpState& s, const double* gbuf, int64_t rows,
                     double* F, int k, bool last_mode, int it, int fit_mode, cudaStream_t st) {
  const int R = static_cast<int>(pl.R);
  solve_finish_kernel<<<1, 256, 0, st>>>(gbuf, R, s.norms, s.gram[k], last_mode ? s.lam : nullptr,
                                         s, it, fit_mode);
  BT_LAUNCH_CHECK();
  const int64_t n = rows * pl.R;
  if (n > 0) {
    scale_cols_kernel<<<static_cast<unsigned>(std::min<int64_t>(bt_cdiv(n, 256), 4096)), 256, 0,
                        st>>>(F, rows, R, s.norms);
    BT_LAUNCH_CHECK();
  }
  return BT_OK;
}

}  // namespace

// tucker.cu: last-mode tensor-times-matrix on the TMA tree kernel (see
// ttm_last_tma_impl); BT_E_VALUE when the operands do not meet TMA's
// 16-byte address / stride rules (the caller takes the engine route)
int bt_ttm_last_tma(const double* x, int64_t rows, int64_t K, const double* u, int64_t R, double* y,
                    cudaStream_t st) {
  if ((K & 1) || (R & 1) || rows < 1 || K < 1 || R < 1 || rows >= ((int64_t)1 << 31) ||
      K >= ((int64_t)1 << 31) || rows * K >= ((int64_t)1 << 36) ||
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(u)) & 15u))
    return BT_E_VALUE;
  return ttm_last_tma_impl(x, rows, K, u, R, y, st);
}

// cp_mid.cu: the R <= 16 one-warp pinv of g0 o g1 (state: one double per mode, zero-initialised)
int bt_cp_pinv_small(const double* g0, const double* g1, int R, double* vp, double* state,
                     cudaStream_t st) {
  return run_pinv(g0, g1, R, vp, st, state, 0);
}

// Explicit residual: Xhat_i = B diag(W_i) C^T with W = A * lam; the per-i
// diagonal rides on the engine's A-scale (indexed by the reduction index r).
namespace {

template <int V>
int residual_pass(const Plan& pl, const double* X, const double* W, const double* Bf,
                  const double* Cf, const double* flag, double* part, cudaStream_t st) {
  using Cfg = ResCfg<V>;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(residual_kernel<Cfg>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES));
    attr = true;
  }
  BtGemmArgs g{};
  g.M = pl.J;
  g.N = pl.K;
  g.Kin = pl.R;
  g.Kout = 1;
  g.A = BtOperand{Bf, pl.R, 0, 1, 0};
  g.B = BtOperand{Cf, pl.R, 0, 1, 0};
  g.ascale = W;
  g.s_ascale_b = pl.R;
  g.alpha = 1.0;
  const int64_t tiles = pl.I * bt_cdiv(pl.J, Cfg::BM) * bt_cdiv(pl.K, Cfg::BN);
  residual_kernel<Cfg><<<pl.res_grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(g, X, pl.J, pl.K, tiles,
                                                                           flag, part);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// CP-ALS state + phase API.  A sweep is
//   mttkrp(1) -> [sum over ranks] -> solve(1) -> finish(1)
//   mttkrp(2) -> [sum over ranks] -> solve(2) -> finish(2)
//   mttkrp(3) ->                     solve(3) -> [sum gbuf]  -> finish(3)
//   residual  -> [sum over ranks] -> residual_finish
// where the bracketed sums are the only cross-GPU exchanges when the tensor
// is sharded along mode 3 (A, B replicated; C row-sharded).  One GPU runs the
// same phases with the sums skipped (bt_cp_als_f64).
// ---------------------------------------------------------------------------

namespace {

__global__ void reduce_m1_kernel(const double* __restrict__ part, int64_t I, int64_t jt,
                                 int64_t R, double* __restrict__ out) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < I * R;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / R, r = idx % R;
    double s = 0.0;
    for (int64_t t = 0; t < jt; ++t) s += part[(i * jt + t) * R + r];
    out[idx] = s;
  }
}

__global__ void reduce_parts_kernel(const double* __restrict__ part, int64_t nparts,
                                    int64_t stride, int64_t n, double* __restrict__ out) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t p = 0; p < nparts; ++p) s += part[p * stride + idx];
    out[idx] = s;
  }
}

unsigned grid_n(int64_t n) { return static_cast<unsigned>(std::min<int64_t>(bt_cdiv(n, 256), 4096)); }

}  // namespace

// G = F^T F (R x R) on the DMMA engine (symmetric, split-K over rows)
static int factor_gram(const Plan& pl, const double* f, int64_t rows, double* g, double* ws,
                       cudaStream_t st) {
  if (rows == 0) {
    BT_CUDA_CHECK(cudaMemsetAsync(g, 0, sizeof(double) * pl.R * pl.R, st));
    return BT_OK;
  }
  BtGemmArgs a{};
  a.M = pl.R;
  a.N = pl.R;
  a.Kin = rows;
  a.Kout = 1;
  a.A = BtOperand{f, 1, 0, pl.R, 0};
  a.B = BtOperand{f, 1, 0, pl.R, 0};
  a.C = g;
  a.sCm = pl.R;
  a.sCn = 1;
  a.alpha = 1.0;
  a.symmetric = 1;
  a.ws = ws;
  return bt_gemm_run(a, 1, st, 0, std::max<int64_t>(pl.solve_parts_max, 64) * pl.R * pl.R);
}

struct bt_cp_state {
  Plan pl;
  CpState s;
  double* ws;
  double* dhist;
  int max_iters;
  int fit_mode;
  cudaStream_t st;
  const double* X;
  double* F[3];
  double* lam;
  // single-GPU driver only: the R x R pinv of mode k depends only on the
  // other modes' Grams, so it runs on `side` while mode k's MTTKRP runs on st
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

static int64_t cp_total_ws(const Plan& pl) { return pl.total + 16; }

extern "C" int bt_cp_tree_variant(const bt_cp_problem* pb) {
  return pb ? cp_tree_variant(pb->I, pb->J, pb->K, pb->R) : -1;
}

extern "C" int64_t bt_cp_als_ws_bytes(const bt_cp_problem* pb) {
  Plan pl = make_plan(pb);
  return cp_total_ws(pl) * 8;
}

extern "C" int64_t bt_cp_state_ws_bytes(const bt_cp_problem* pb) { return bt_cp_als_ws_bytes(pb); }

extern "C" int bt_cp_state_create(const bt_cp_problem* pb, double* a, double* b, double* c,
                                  double* lam, int max_iters, int fit_mode, void* wsv,
                                  int64_t ws_bytes, void* stream, void** out) {
  BT_REQUIRE(pb->I >= 1 && pb->J >= 1 && pb->K >= 0, BT_E_SHAPE, "cp_als: empty tensor");
  BT_REQUIRE(pb->R >= 1, BT_E_SHAPE, "CP rank must be at least 1");
  BT_REQUIRE(pb->R <= PINV_MAX_R, BT_E_SHAPE, "cp_als: rank %lld above the on-chip limit %d",
             (long long)pb->R, PINV_MAX_R);
  BT_REQUIRE(max_iters >= 1, BT_E_VALUE, "max_iters must be at least 1");
  auto* S = new bt_cp_state();
  S->pl = make_plan(pb);
  if (ws_bytes < cp_total_ws(S->pl) * 8) {
    delete S;
    bt_set_error("cp_als: workspace too small");
    return BT_E_VALUE;
  }
  S->ws = static_cast<double*>(wsv);
  S->st = bt_stream(stream);
  S->X = pb->x;
  S->F[0] = a;
  S->F[1] = b;
  S->F[2] = c;
  S->lam = lam;
  S->max_iters = max_iters;
  S->fit_mode = fit_mode;
  const int64_t RR = S->pl.R * S->pl.R;
  double* sb = S->ws + S->pl.off_state;
  S->s.gram[0] = sb;
  S->s.gram[1] = sb + RR;
  S->s.gram[2] = sb + 2 * RR;
  S->s.vp = sb + 3 * RR;
  S->s.norms = sb + 4 * RR;
  S->s.lam = lam;
  S->s.scal = sb + 4 * RR + S->pl.R;
  S->s.iter = reinterpret_cast<int*>(S->s.scal + 6);
  bt_keep_async_pool();
  cudaError_t e = cudaMallocAsync(&S->dhist, sizeof(double) * max_iters, S->st);
  if (e != cudaSuccess) {
    delete S;
    bt_set_error("cp_als: %s", cudaGetErrorString(e));
    return BT_E_CUDA;
  }
  S->s.fit_hist = S->dhist;
  *out = S;
  return BT_OK;
}

extern "C" int bt_cp_state_destroy(void* state) {
  auto* S = static_cast<bt_cp_state*>(state);
  if (!S) return BT_OK;
  if (S->ev_fork) cudaEventDestroy(S->ev_fork);
  if (S->ev_join) cudaEventDestroy(S->ev_join);
  if (S->side) {
    cudaStreamSynchronize(S->side);
    cudaStreamDestroy(S->side);
  }
  cudaFreeAsync(S->dhist, S->st);
  delete S;
  return BT_OK;
}

// Local init contributions: buf = [C^T C (R*R), ||X_local||^2, 0]; A, B Grams are
// replicated and computed in place.  norm_x > 0 in the problem skips the sum.
extern "C" int bt_cp_init_local(void* state, double norm_x, double* buf) {
  auto* S = static_cast<bt_cp_state*>(state);
  const Plan& pl = S->pl;
  const int R = static_cast<int>(pl.R);
  BT_TRY(factor_gram(pl, S->F[0], pl.I, S->s.gram[0], S->ws + pl.off_gp, S->st));
  BT_TRY(factor_gram(pl, S->F[1], pl.J, S->s.gram[1], S->ws + pl.off_gp, S->st));
  BT_TRY(factor_gram(pl, S->F[2], pl.K, buf, S->ws + pl.off_gp, S->st));
  if (norm_x > 0.0) {
    const double x2 = norm_x * norm_x;
    BT_CUDA_CHECK(cudaMemcpyAsync(buf + pl.R * pl.R, &x2, 8, cudaMemcpyHostToDevice, S->st));
  } else {
    BT_TRY(bt_sumsq_f64(S->X, pl.I * pl.J * pl.K, buf + pl.R * pl.R, S->ws + pl.off_res, 2048 * 8,
                        S->st));
  }
  return BT_OK;
}

__global__ void init_finish_kernel(const double* __restrict__ buf, int R, double* __restrict__ gc,
                                   double* __restrict__ scal) {
  for (int idx = threadIdx.x; idx < R * R; idx += blockDim.x) gc[idx] = buf[idx];
  if (threadIdx.x == 0) scal[0] = buf[R * R];
}

extern "C" int bt_cp_init_finish(void* state, const double* buf) {
  auto* S = static_cast<bt_cp_state*>(state);
  init_finish_kernel<<<1, 256, 0, S->st>>>(buf, static_cast<int>(S->pl.R), S->s.gram[2], S->s.scal);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// MTTKRP of `mode` over the local tensor into out (I x R, J x R, or K_local x R).
// Modes 1/2 are partial sums over the local mode-3 slab (sum across ranks);
// mode 3 rows are complete locally.  Mode 1 also (re)computes P = X x3 C.
extern "C" int bt_cp_mttkrp(void* state, int mode, double* out) {
  BT_NVTX("bt_cp_mttkrp");
  auto* S = static_cast<bt_cp_state*>(state);
  const Plan& pl = S->pl;
  double* ws = S->ws;
  cudaStream_t st = S->st;
  if (pl.qtree && pl.K > 0) {
    if (mode == 1 && pl.m1_via_t) {
      int rc = use_at_tma() ? bt_gemm_at_tma(S->X, pl.K, pl.J * pl.K, S->F[1], pl.R, ws + pl.off_t, pl.R,
                                             pl.K * pl.R, pl.K, pl.R, pl.J, pl.I, st)
                            : BT_E_VALUE;
      if (rc == BT_E_VALUE) {
        BtGemmArgs g = tslab_args(pl, S->X, S->F[1], ws + pl.off_t);
        g.ws = ws + pl.off_m3ws;
        rc = bt_gemm_run(g, pl.I, st, 1, 0);
      }
      BT_TRY(rc);
      mode2_from_q_kernel<<<static_cast<unsigned>(pl.I), 256, 0, st>>>(ws + pl.off_t, S->F[2], pl.K,
                                                                       static_cast<int>(pl.R), out);
      BT_LAUNCH_CHECK();
      return BT_OK;
    }
    if (mode == 1) {
      // the tree kernel without its P store: M1 partials per (i, j-tile) from
      // the fused epilogue (23 TF/s at K = 128 vs 20 for the engine GEMM with
      // the Khatri-Rao B-scale)
      BT_TRY(run_tree(pl, S->X, S->F[2], S->F[1], nullptr, ws + pl.off_m1, 0, st));
      reduce_m1_kernel<<<grid_n(pl.I * pl.R), 256, 0, st>>>(ws + pl.off_m1, pl.I, pl.jtiles, pl.R,
                                                            out);
      BT_LAUNCH_CHECK();
      return BT_OK;
    }
    if (mode == 2) {
      int rc = use_at_tma() ? bt_gemm_at_tma(S->X, pl.J * pl.K, 0, S->F[0], pl.R, ws + pl.off_p, pl.R, 0,
                                             pl.J * pl.K, pl.R, pl.I, 1, st)
                            : BT_E_VALUE;
      if (rc == BT_E_VALUE) {
        BtGemmArgs g = qtree_args(pl, S->X, S->F[0], ws + pl.off_p);
        g.ws = ws + pl.off_m3ws;
        rc = bt_gemm_run(g, 1, st, 0, pl.m3_ws_elems);
      }
      BT_TRY(rc);
      mode2_from_q_kernel<<<static_cast<unsigned>(pl.J), 256, 0, st>>>(ws + pl.off_p, S->F[2], pl.K,
                                                                       static_cast<int>(pl.R), out);
      BT_LAUNCH_CHECK();
      return BT_OK;
    }
    if (mode == 3) {
      // m3[k][r] = sum_j Q[j][k][r] B[j][r]: j-chunk partials, fixed-order sum
      const int64_t KR = pl.K * pl.R;
      const int64_t bx = std::max<int64_t>(1, std::min<int64_t>(bt_cdiv(KR, 256), 2048));
      mode2_from_p_kernel<<<dim3(static_cast<unsigned>(bx), static_cast<unsigned>(pl.s3)), 256, 0,
                            st>>>(ws + pl.off_p, S->F[1], pl.J, KR, pl.R, pl.chunk3,
                                  ws + pl.off_m2);
      BT_LAUNCH_CHECK();
      reduce_parts_kernel<<<grid_n(KR), 256, 0, st>>>(ws + pl.off_m2, pl.s3, KR, KR, out);
      BT_LAUNCH_CHECK();
      return BT_OK;
    }
  }
  if (mode == 1) {
    if (pl.K > 0) {
      BT_TRY(run_tree(pl, S->X, S->F[2], S->F[1], ws + pl.off_p, ws + pl.off_m1, 1, st));
      reduce_m1_kernel<<<grid_n(pl.I * pl.R), 256, 0, st>>>(ws + pl.off_m1, pl.I, pl.jtiles, pl.R,
                                                            out);
    } else {
      BT_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(double) * pl.I * pl.R, st));
      return BT_OK;
    }
    BT_LAUNCH_CHECK();
  } else if (mode == 2) {
    if (pl.K > 0) {
      BT_TRY(run_mode2(pl, ws + pl.off_p, S->F[0], ws + pl.off_m2, st));
      const int64_t n = pl.J * pl.R;
      reduce_parts_kernel<<<grid_n(n), 256, 0, st>>>(ws + pl.off_m2, pl.s2, n, n, out);
      BT_LAUNCH_CHECK();
    } else {
      BT_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(double) * pl.J * pl.R, st));
    }
  } else if (mode == 3) {
    if (pl.K > 0) BT_TRY(run_mode3(pl, S->X, S->F[0], S->F[1], out, ws + pl.off_m3ws, st));
  } else {
    bt_set_error("mode %d out of range", mode);
    return BT_E_SHAPE;
  }
  return BT_OK;
}

// Local solve of `mode` from the (summed) MTTKRP m: gbuf = [F_un^T F_un, <F_un, M>, 0].
// For mode 3 (row-sharded) gbuf must be summed across ranks before finish.
static int cp_solve_impl(bt_cp_state* S, int mode, const double* m, double* gbuf, bool pinv_done) {
  const Plan& pl = S->pl;
  const int k = mode - 1;
  const int64_t rows[3] = {pl.I, pl.J, pl.K};
  const int go0 = (k == 0) ? 1 : 0, go1 = (k == 2) ? 1 : 2;
  return run_solve_rows(pl, S->s, S->ws, m, 1, 0, pl.R, rows[k], go0, go1, S->F[k], k == 2, gbuf,
                        S->st, pinv_done);
}

extern "C" int bt_cp_solve(void* state, int mode, const double* m, double* gbuf) {
  BT_NVTX("bt_cp_solve");
  return cp_solve_impl(static_cast<bt_cp_state*>(state), mode, m, gbuf, false);
}

// fork mode `mode`'s pinv(G_o0 o G_o1) onto the side stream (joined by
// cp_pinv_join before the solve)
static int cp_pinv_fork(bt_cp_state* S, int mode, int warm) {
  const int k = mode - 1;
  const int go0 = (k == 0) ? 1 : 0, go1 = (k == 2) ? 1 : 2;
  BT_CUDA_CHECK(cudaEventRecord(S->ev_fork, S->st));
  BT_CUDA_CHECK(cudaStreamWaitEvent(S->side, S->ev_fork, 0));
  BT_TRY(run_pinv(S->s.gram[go0], S->s.gram[go1], static_cast<int>(S->pl.R), S->s.vp, S->side,
                  S->ws + S->pl.off_jstore + k * 256, warm));
  BT_CUDA_CHECK(cudaEventRecord(S->ev_join, S->side));
  return BT_OK;
}

static int cp_pinv_join(bt_cp_state* S) {
  BT_CUDA_CHECK(cudaStreamWaitEvent(S->st, S->ev_join, 0));
  return BT_OK;
}

extern "C" int bt_cp_solve_finish(void* state, int mode, int it, const double* gbuf) {
  auto* S = static_cast<bt_cp_state*>(state);
  // it == -1: take the index from the state's device counter (graph replay)
  BT_REQUIRE(it >= -1 && it < S->max_iters, BT_E_VALUE, "sweep index out of range");
  const Plan& pl = S->pl;
  const int k = mode - 1;
  const int64_t rows[3] = {pl.I, pl.J, pl.K};
  return run_solve_finish(pl, S->s, gbuf, rows[k], S->F[k], k, k == 2, it, S->fit_mode, S->st);
}

// Explicit residual partial ||X_local - Xhat_local||^2 into res2 (device scalar;
// writes 0 when the Gram identity was judged accurate).  Sum across ranks.
extern "C" int bt_cp_residual(void* state, double* res2) {
  BT_NVTX("bt_cp_residual");
  auto* S = static_cast<bt_cp_state*>(state);
  const Plan& pl = S->pl;
  if (S->fit_mode == 2 || pl.K == 0) {
    BT_CUDA_CHECK(cudaMemsetAsync(res2, 0, sizeof(double), S->st));
    return BT_OK;
  }
  double* W = S->ws + pl.off_w;
  double* rpart = S->ws + pl.off_res;
  lam_scale_kernel<<<grid_n(pl.I * pl.R), 256, 0, S->st>>>(S->F[0], S->lam, pl.I,
                                                           static_cast<int>(pl.R), W);
  BT_LAUNCH_CHECK();
  if (pl.R <= 16) {
    // res_grid CTAs of 256 threads; every CTA writes its partial
    if (pl.R <= 8)
      residual_small_kernel<8><<<pl.res_grid, 256, 0, S->st>>>(
          S->X, W, S->F[1], S->F[2], pl.I, pl.J, pl.K, static_cast<int>(pl.R), S->s.scal + 3, rpart);
    else
      residual_small_kernel<16><<<pl.res_grid, 256, 0, S->st>>>(
          S->X, W, S->F[1], S->F[2], pl.I, pl.J, pl.K, static_cast<int>(pl.R), S->s.scal + 3, rpart);
    BT_LAUNCH_CHECK();
  } else if (pl.R % 2 == 0) {
    BT_TRY(residual_pass<2>(pl, S->X, W, S->F[1], S->F[2], S->s.scal + 3, rpart, S->st));
  } else {
    BT_TRY(residual_pass<1>(pl, S->X, W, S->F[1], S->F[2], S->s.scal + 3, rpart, S->st));
  }
  residual_reduce_kernel<<<1, 32, 0, S->st>>>(rpart, pl.res_grid, res2);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

extern "C" int bt_cp_residual_finish(void* state, int it, const double* res2) {
  auto* S = static_cast<bt_cp_state*>(state);
  residual_finish_kernel<<<1, 32, 0, S->st>>>(res2, S->s, it);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// Synchronous read of the fit of sweep `it` (for the tol > 0 convergence test).
extern "C" int bt_cp_read_fit(void* state, int it, double* fit) {
  auto* S = static_cast<bt_cp_state*>(state);
  BT_CUDA_CHECK(cudaMemcpyAsync(fit, S->dhist + it, 8, cudaMemcpyDeviceToHost, S->st));
  BT_CUDA_CHECK(cudaStreamSynchronize(S->st));
  return BT_OK;
}

// x = F0 * lam (KruskalRep.x, decomp.py:403) and the fit history to the host.
extern "C" int bt_cp_state_finish(void* state, int n_iters, double* fit_history) {
  auto* S = static_cast<bt_cp_state*>(state);
  const Plan& pl = S->pl;
  lam_scale_kernel<<<grid_n(pl.I * pl.R), 256, 0, S->st>>>(S->F[0], S->lam, pl.I,
                                                           static_cast<int>(pl.R), S->F[0]);
  BT_LAUNCH_CHECK();
  if (n_iters > 0 && fit_history) {
    BT_CUDA_CHECK(cudaMemcpyAsync(fit_history, S->dhist, sizeof(double) * n_iters,
                                  cudaMemcpyDeviceToHost, S->st));
  }
  BT_CUDA_CHECK(cudaStreamSynchronize(S->st));
  return BT_OK;
}

// Diagnostic: clock64 stamps of sweep 1's phases in the fused small kernel
// (P, mode 1 MTTKRP, solve 1, mode 2, solve 2, mode 3, solve 3, fit, end).
extern "C" int bt_cp_cluster_clocks(long long* out16) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out16, g_cluster_clk, sizeof(long long) * 16);
}

extern "C" int bt_cp_small_clocks(long long* out) {
  BT_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_small_clk, sizeof(long long) * 13));
  return BT_OK;
}

// The cluster path of bt_cp_als_f64 (cp_cluster.cuh): X resident in the
// distributed shared memory of 8 CTAs.  Returns 1 when it ran, 0 when the
// problem is not eligible (the one-CTA kernel is tried next).
static int cp_cluster_try(const bt_cp_problem* pb, double* a, double* b, double* c, double* lam,
                          int max_iters, double tol, int fit_mode, double* fit_history,
                          int* n_iters, int* converged, cudaStream_t st, int* rc) {
  // read per call: the parity tests switch paths in-process
  const bool off = getenv("BT_CP_CLUSTER") && getenv("BT_CP_CLUSTER")[0] == '0';
  *rc = BT_OK;
  const int64_t I = pb->I, J = pb->J, K = pb->K, R = pb->R;
  if (off || R > SMALL_RS || I < 1 || J < 1 || K < 1 || I * J * K > (int64_t(1) << 17) ||
      I > 1024 || J > 1024 || K > 1024 || pb->norm_x <= 0.0)
    return 0;
  const int NP = R <= 8 ? 8 : 16;
  const size_t smem = static_cast<size_t>(cluster_layout(I, J, K, R, NP).total) * 8;
  if (smem > 200 * 1024) return 0;
  double* dbuf = nullptr;
  bt_keep_async_pool();
  cudaError_t e = cudaMallocAsync(&dbuf, sizeof(double) * (max_iters + 2), st);
  if (e != cudaSuccess) {
    bt_set_error("cp_als: %s", cudaGetErrorString(e));
    *rc = BT_E_CUDA;
    return 1;
  }
  int* info = reinterpret_cast<int*>(dbuf + max_iters);
  const double x2 = pb->norm_x * pb->norm_x;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL_CS);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL_CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const double* xp = pb->x;
  const int Ii = (int)I, Ji = (int)J, Ki = (int)K, Ri = (int)R;
  cudaError_t le;
  if (NP == 8) {
    cudaFuncSetAttribute(cp_cluster_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    le = cudaLaunchKernelEx(&cfg, cp_cluster_kernel<8>, xp, Ii, Ji, Ki, Ri, a, b, c, lam, x2,
                            max_iters, tol, fit_mode, dbuf, info);
  } else {
    cudaFuncSetAttribute(cp_cluster_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    le = cudaLaunchKernelEx(&cfg, cp_cluster_kernel<16>, xp, Ii, Ji, Ki, Ri, a, b, c, lam, x2,
                            max_iters, tol, fit_mode, dbuf, info);
  }
  if (le != cudaSuccess) {
    // a cluster that cannot be placed is not an error: the one-CTA kernel runs instead
    cudaGetLastError();
    cudaFreeAsync(dbuf, st);
    return 0;
  }
  bt_count_launch();
  // history and (n_iters, converged) in one read-back, one synchronisation
  std::vector<double> hbuf(static_cast<size_t>(max_iters) + 2);
  cudaMemcpyAsync(hbuf.data(), dbuf, sizeof(double) * hbuf.size(), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dbuf, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    bt_set_error("cp_cluster: %s", cudaGetErrorString(e));
    *rc = BT_E_CUDA;
    return 1;
  }
  int hinfo[2];
  std::memcpy(hinfo, hbuf.data() + max_iters, sizeof(hinfo));
  if (fit_history)
    for (int k = 0; k < hinfo[0] && k < max_iters; ++k) fit_history[k] = hbuf[k];
  *n_iters = hinfo[0];
  *converged = hinfo[1];
  return 1;
}

// One-GPU driver over the phase API (no cross-rank sums).
// The fused one-CTA path of bt_cp_als_f64 for tensors that fit one SM.
// Returns 1 when it ran (outputs written), 0 when the problem is not eligible.
static int cp_small_try(const bt_cp_problem* pb, double* a, double* b, double* c, double* lam,
                        int max_iters, double tol, int fit_mode, double* fit_history,
                        int* n_iters, int* converged, cudaStream_t st, int* rc) {
  const bool off = getenv("BT_CP_SMALL") && getenv("BT_CP_SMALL")[0] == '0';
  *rc = BT_OK;
  const int64_t I = pb->I, J = pb->J, K = pb->K, R = pb->R;
  if (off || R > SMALL_RS || I < 1 || J < 1 || K < 1 || I * J * K > (int64_t(1) << 17) ||
      I > 1024 || J > 1024 || K > 1024 || pb->norm_x <= 0.0)
    return 0;
  const int NP = R <= 8 ? 8 : 16;
  const size_t smem = static_cast<size_t>(small_layout(I, J, K, R, NP).total) * 8;
  if (smem > 200 * 1024) return 0;
  double* dbuf = nullptr;
  bt_keep_async_pool();
  cudaError_t e = cudaMallocAsync(&dbuf, sizeof(double) * (max_iters + 2), st);
  if (e != cudaSuccess) {
    bt_set_error("cp_als: %s", cudaGetErrorString(e));
    *rc = BT_E_CUDA;
    return 1;
  }
  int* info = reinterpret_cast<int*>(dbuf + max_iters);
  const double x2 = pb->norm_x * pb->norm_x;
  if (NP == 8) {
    cudaFuncSetAttribute(cp_small_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cp_small_kernel<8><<<1, 512, smem, st>>>(pb->x, (int)I, (int)J, (int)K, (int)R, a, b, c, lam,
                                             x2, max_iters, tol, fit_mode, dbuf, info);
  } else {
    cudaFuncSetAttribute(cp_small_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cp_small_kernel<16><<<1, 512, smem, st>>>(pb->x, (int)I, (int)J, (int)K, (int)R, a, b, c,
                                              lam, x2, max_iters, tol, fit_mode, dbuf, info);
  }
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) {
    bt_set_error("cp_small_kernel: %s", cudaGetErrorString(le));
    cudaFreeAsync(dbuf, st);
    *rc = BT_E_CUDA;
    return 1;
  }
  bt_count_launch();
  int hinfo[2] = {0, 0};
  cudaMemcpyAsync(hinfo, info, sizeof(hinfo), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  if (hinfo[0] > 0 && fit_history)
    cudaMemcpyAsync(fit_history, dbuf, sizeof(double) * hinfo[0], cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dbuf, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    bt_set_error("cp_small: %s", cudaGetErrorString(e));
    *rc = BT_E_CUDA;
    return 1;
  }
  *n_iters = hinfo[0];
  *converged = hinfo[1];
  return 1;
}

// cp_mid.cu: two-pass sweep for R <= 16 on tensors larger than one SM
int bt_cp_mid_try(const bt_cp_problem* pb, double* a, double* b, double* c, double* lam,
                  int max_iters, double tol, int fit_mode, double* fit_history, int* n_iters,
                  int* converged, cudaStream_t st, int* rc);

extern "C" int bt_cp_als_f64(const bt_cp_problem* pb, double* a, double* b, double* c,
                             double* lam, int max_iters, double tol, int fit_mode,
                             double* fit_history, int* n_iters, int* converged, double* phase_ms,
                             void* wsv, int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_cp_als_f64");
  if (phase_ms == nullptr && max_iters >= 1) {
    int rc = BT_OK;
    if (cp_cluster_try(pb, a, b, c, lam, max_iters, tol, fit_mode, fit_history, n_iters, converged,
                       bt_stream(stream), &rc))
      return rc;
    if (cp_small_try(pb, a, b, c, lam, max_iters, tol, fit_mode, fit_history, n_iters, converged,
                     bt_stream(stream), &rc))
      return rc;
    if (bt_cp_mid_try(pb, a, b, c, lam, max_iters, tol, fit_mode, fit_history, n_iters, converged,
                      bt_stream(stream), &rc))
      return rc;
  }
  void* h = nullptr;
  BT_TRY(bt_cp_state_create(pb, a, b, c, lam, max_iters, fit_mode, wsv, ws_bytes, stream, &h));
  auto* S = static_cast<bt_cp_state*>(h);
  const Plan& pl = S->pl;
  double* ws = S->ws;
  cudaStream_t st = S->st;
  double* m1 = ws + pl.off_m1d;
  double* m2 = ws + pl.off_m2d;
  double* m3 = ws + pl.off_m3;
  double* gbuf = ws + pl.off_gbuf;
  double* res2 = ws + pl.off_res1;
  int rc = BT_OK;
  std::vector<cudaEvent_t> ev;
  auto mark = [&]() -> int {
    if (!phase_ms) return BT_OK;
    cudaEvent_t e;
    BT_CUDA_CHECK(cudaEventCreate(&e));
    BT_CUDA_CHECK(cudaEventRecord(e, st));
    ev.push_back(e);
    return BT_OK;
  };
  double prev = -INFINITY;
  int it = 0, conv = 0;
  // one ALS sweep; ix < 0: the kernels take the sweep index from the device
  // counter (graph replay), which the sweep then advances
  // the pinv of each mode overlaps that mode's MTTKRP (side stream; joined
  // before the solve).  With per-phase events requested it stays inline so
  // the phase times keep their meaning.
  const bool overlap = phase_ms == nullptr;
  if (overlap) {
    if (cudaStreamCreateWithFlags(&S->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&S->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&S->ev_join, cudaEventDisableTiming) != cudaSuccess) {
      bt_set_error("cp_als: cannot create the pinv side stream");
      bt_cp_state_destroy(h);
      return BT_E_CUDA;
    }
  }
  // sweep 1 (eager) factors each mode's V cold; later sweeps (and the graph
  // captured from sweep 2) warm-start from the stored rotation
  int warm = 0;
  auto mode_step = [&](int mode, double* mbuf, int ix) -> int {
    BT_TRY(mark());
    if (overlap) BT_TRY(cp_pinv_fork(S, mode, warm));
    BT_TRY(bt_cp_mttkrp(h, mode, mbuf));
    BT_TRY(mark());
    if (overlap) BT_TRY(cp_pinv_join(S));
    BT_TRY(cp_solve_impl(S, mode, mbuf, gbuf, overlap));
    BT_TRY(bt_cp_solve_finish(h, mode, ix, gbuf));
    return BT_OK;
  };
  auto sweep = [&](int ix) -> int {
    BT_TRY(mode_step(1, m1, ix));
    BT_TRY(mode_step(2, m2, ix));
    BT_TRY(mode_step(3, m3, ix));
    warm = 1;
    BT_TRY(bt_cp_residual(h, res2));
    BT_TRY(bt_cp_residual_finish(h, ix, res2));
    BT_TRY(mark());
    if (ix < 0) {
      advance_iter_kernel<<<1, 32, 0, S->st>>>(S->s.iter);
      BT_LAUNCH_CHECK();
    }
    return BT_OK;
  };
  // Small problems are launch-latency bound (C1: ~25 launches per sweep of a
  // few us each): after one eager sweep the sweep is captured once as a CUDA
  // graph and replayed.  Not used when per-phase events are requested.
  const bool use_graph = (phase_ms == nullptr) && max_iters >= 3 &&
                         (double)pl.I * pl.J * pl.K * pl.R <= 1e10 && [] {
                           const char* e = getenv("BT_CP_GRAPH");
                           return !(e && e[0] == '0');
                         }();
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  do {
    if ((rc = bt_cp_init_local(h, pb->norm_x, ws + pl.off_init)) != BT_OK) break;
    if ((rc = bt_cp_init_finish(h, ws + pl.off_init)) != BT_OK) break;
    for (it = 1; it <= max_iters; ++it) {
      const int ix = it - 1;
      if (use_graph && it >= 2) {
        if (!gexec) {
          set_iter_kernel<<<1, 32, 0, st>>>(S->s.iter, ix);
          BT_LAUNCH_CHECK();
          // capture on a private stream (the caller's may be the legacy
          // default stream, which cannot be captured); replay on the caller's
          cudaStream_t cs = nullptr;
          if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess ||
              cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            if (cs) cudaStreamDestroy(cs);
            bt_set_error("cp_als: cannot start the sweep graph capture");
            rc = BT_E_CUDA;
            break;
          }
          S->st = cs;
          const int cap_rc = sweep(-1);
          const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
          S->st = st;
          cudaStreamDestroy(cs);
          cudaError_t ei = cudaSuccess;
          if (cap_rc == BT_OK && ec == cudaSuccess) ei = cudaGraphInstantiate(&gexec, graph, 0);
          if (cap_rc != BT_OK || ec != cudaSuccess || ei != cudaSuccess) {
            char inner[512];
            snprintf(inner, sizeof(inner), "%s", bt_last_error());
            bt_set_error("cp_als: sweep graph capture failed (rc %d: %s; end %s; instantiate %s)",
                         cap_rc, inner, cudaGetErrorString(ec), cudaGetErrorString(ei));
            cudaGetLastError();
            rc = BT_E_CUDA;
            break;
          }
        }
        if (cudaGraphLaunch(gexec, st) != cudaSuccess) {
          bt_set_error("cp_als: graph launch failed");
          rc = BT_E_CUDA;
          break;
        }
      } else {
        if ((rc = sweep(ix)) != BT_OK) break;
      }
      if (tol > 0.0) {
        double fit = 0.0;
        if ((rc = bt_cp_read_fit(h, ix, &fit)) != BT_OK) break;
        if (std::fabs(fit - prev) < tol) {
          conv = 1;
          break;
        }
        prev = fit;
      }
    }
    if (rc != BT_OK) break;
    if (it > max_iters) it = max_iters;
    rc = bt_cp_state_finish(h, it, fit_history);
  } while (false);
  if (rc == BT_OK) {
    *n_iters = it;
    *converged = conv;
    if (phase_ms) {
      // per sweep: [t0 mttkrp1 t1 solve1 t2 mttkrp2 t3 solve2 t4 mttkrp3 t5 solve3+fit t6]
      for (int k = 0; k < 4; ++k) phase_ms[k] = 0.0;
      for (size_t base = 0; base + 7 <= ev.size(); base += 7) {
        float ms = 0.f;
        auto el = [&](int x, int y) {
          cudaEventElapsedTime(&ms, ev[base + x], ev[base + y]);
          return static_cast<double>(ms);
        };
        phase_ms[0] += el(0, 1);
        phase_ms[1] += el(2, 3);
        phase_ms[2] += el(4, 5);
        phase_ms[3] += el(1, 2) + el(3, 4) + el(5, 6);
      }
    }
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  if (graph) cudaGraphDestroy(graph);
  for (auto e : ev) cudaEventDestroy(e);
  bt_cp_state_destroy(h);
  return rc;
}

extern "C" int64_t bt_mttkrp_ws_bytes(const bt_cp_problem* pb, int mode) {
  Plan pl = make_plan(pb, 0);
  (void)mode;
  return pl.total * 8;
}

extern "C" int bt_mttkrp_f64(const bt_cp_problem* pb, int mode, const double* a, const double* b,
                             const double* c, double* out, void* wsv, int64_t ws_bytes,
                             void* stream) {
  BT_NVTX("bt_mttkrp_f64");
  BT_REQUIRE(mode >= 1 && mode <= 3, BT_E_SHAPE, "mttkrp: mode %d out of range", mode);
  cudaStream_t st = bt_stream(stream);
  Plan pl = make_plan(pb, 0);
  BT_REQUIRE(ws_bytes >= pl.total * 8, BT_E_VALUE, "mttkrp: workspace too small");
  double* ws = static_cast<double*>(wsv);
  double* P = ws + pl.off_p;
  if (mode == 1) {
    BT_TRY(run_tree(pl, pb->x, c, b, P, ws + pl.off_m1, 0, st));
    reduce_m1_kernel<<<static_cast<unsigned>(std::min<int64_t>(bt_cdiv(pl.I * pl.R, 256), 4096)),
                       256, 0, st>>>(ws + pl.off_m1, pl.I, pl.jtiles, pl.R, out);
    BT_LAUNCH_CHECK();
  } else if (mode == 2) {
    BT_TRY(run_tree(pl, pb->x, c, b, P, ws + pl.off_m1, 1, st));
    BT_TRY(run_mode2(pl, P, a, ws + pl.off_m2, st));
    const int64_t n = pl.J * pl.R;
    reduce_parts_kernel<<<static_cast<unsigned>(std::min<int64_t>(bt_cdiv(n, 256), 4096)), 256, 0,
                          st>>>(ws + pl.off_m2, pl.s2, n, n, out);
    BT_LAUNCH_CHECK();
  } else {
    BT_TRY(run_mode3(pl, pb->x, a, b, out, ws + pl.off_m3ws, st));
  }
  return BT_OK;
}

extern "C" int bt_pinv_sym_f64(const double* v, int64_t R, double* vp, void* stream) {
  BT_NVTX("bt_pinv_sym_f64");
  BT_REQUIRE(R >= 1 && R <= PINV_MAX_R, BT_E_SHAPE, "pinv: size %lld outside [1, %d]",
             (long long)R, PINV_MAX_R);
  return run_pinv(v, nullptr, static_cast<int>(R), vp, bt_stream(stream));
}

// diagnostics: sweeps of the last warp-Jacobi eigen path in this module
extern "C" int bt_debug_jacobi_sweeps(void) {
  int v = -1;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&v, g_jacobi_sweeps, sizeof(int));
  return v;
}

extern "C" int64_t bt_debug_pinv1s(int which) {
  long long v[2] = {-1, -1};
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(v, g_pinv1s_dbg, sizeof(v));
  return v[which & 1];
}

// diagnostics: the ring of (sweeps << 40 | cycles) entries; returns the call count
extern "C" int64_t bt_debug_pinv1s_log(long long* out512) {
  unsigned n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out512, g_pinv1s_log, 512 * sizeof(long long));
  cudaMemcpyFromSymbol(&n, g_pinv1s_n, sizeof(n));
  return n;
}
