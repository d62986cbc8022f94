// TMA-fed DMMA SYRK for the unfolding Gram of a non-last mode (K7):
//   G[i][i'] = sum_{o, c} X(o, i, c) X(o, i', c)
// with X viewed as (outer, n, inner), inner contiguous -- the reference's
// `svd(unfold(t, k))` (decomp.py:172, 227) replaced by the Gram + symmetric
// eigensolver.  C3 mode 1 (n = 1024, inner = 524288): 5.5e11 unique-half
// flops, the largest single kernel of the Tucker path.
//
// The lower triangle is cut into 64 x 64 blocks (diagonal blocks in full) and
// the blocks are paired into CTA tiles that share one 64-column block b: the
// tile loads two 64-row boxes a1, a2 as its 128-row A operand and the
// 64-row box b as B, and computes X_a1 X_b^T and X_a2 X_b^T (a block with
// a < b is the transpose of the lower block (b, a) and is stored transposed).
// Column b takes its lower blocks a = b .. nb-1; when their count is odd the
// block (b+1, b) is handed to column b+1 (as a = b), so every tile is full
// but possibly the last.  For n = 1024 that is 68 tiles over 136 blocks (5.6%
// above the unique half) where 128 x 64 tiles over the 128-block triangle
// computed 72 (12.4% above).  Each tile's reduction (outer x inner, in
// 16-wide k-tiles) is split over `splits` CTAs, the split count chosen so the
// CTA count fills whole waves of 2 CTAs per SM.  Four DMMA warps of 64 x 32,
// 4 stages of 24 KB (three 64-row boxes of the same tensor, 128-byte
// swizzle), the last warp out of a stage re-arms and refills it (as cp.cu's
// tree_p_tma_kernel).  Partials go to ws[split][n][n]
// and bt_gemm_reduce_kernel sums them in a fixed order and mirrors the upper
// triangle (bit-reproducible).
#include <algorithm>

#include "gemm.cuh"
#include "tma.cuh"

__global__ void bt_gemm_reduce_kernel(BtGemmArgs g, int64_t bm, int64_t bn);

namespace {

struct SyrkCfg {
  static constexpr int BM = 128, BN = 64, BK = 16, STAGES = 4;
  static constexpr int WM = 2, WN = 2, THREADS = WM * WN * 32;
  static constexpr int TM = BM / WM, TN = BN / WN, FM = TM / 8, FN = TN / 8;
  static constexpr int A_STAGE = BM * BK, B_STAGE = BN * BK;  // doubles
  static constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
};

__device__ __forceinline__ void syrk_issue(const CUtensorMap* xmap, double* as, double* bs, uint64_t* bar,
                                           int kt, int kti, int r1, int r2, int rb, uint64_t pol) {
  const int o = kt / kti, k0 = (kt - o * kti) * SyrkCfg::BK;
  mbar_arrive_expect_tx(bar, SyrkCfg::STAGE_BYTES);
  tma_load_3d(as, xmap, bar, k0, r1, o, pol);
  tma_load_3d(as + (SyrkCfg::BM / 2) * SyrkCfg::BK, xmap, bar, k0, r2, o, pol);
  tma_load_3d(bs, xmap, bar, k0, rb, o, pol);
}

// Tile t of the pairing described above -> column block b and row blocks
// a1, a2 (a2 = -1 for a single-block last tile).  Host and device share it.
__host__ __device__ inline int syrk_tile(int t, int nb, int* b, int* a1, int* a2) {
  int carry = 0, base = 0;
  for (int c = 0; c < nb; ++c) {
    const int cnt = nb - c + carry;
    const int leave = ((cnt & 1) && c + 1 < nb) ? 1 : 0;  // (c+1, c) moves to column c+1
    const int used = cnt - leave;
    const int nt = (used + 1) / 2;
    if (b != nullptr && t < base + nt) {
      const int p0 = 2 * (t - base);
      int e[2];
      for (int q = 0; q < 2; ++q) {
        int p = p0 + q;
        if (p >= used) {
          e[q] = -1;
          continue;
        }
        if (carry) {
          if (p == 0) {
            e[q] = c - 1;
            continue;
          }
          --p;
        }
        int r = c + p;
        if (leave && r >= c + 1) ++r;
        e[q] = r;
      }
      *b = c;
      *a1 = e[0];
      *a2 = e[1];
      return base + nt;
    }
    base += nt;
    carry = leave;
  }
  return base;  // the tile count when b == nullptr
}

__global__ void __launch_bounds__(SyrkCfg::THREADS, 2)
    syrk_tma_kernel(const __grid_constant__ CUtensorMap xmap, int n, int kti, int KT, int splits, int tiles,
                    double* __restrict__ ws) {
  using T = SyrkCfg;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[T::STAGES];
  __shared__ int left_cnt[T::STAGES];
  // work unit -> (tile, split), split-major so a wave's CTAs share k windows
  const int unit = blockIdx.x;
  const int tile = unit % tiles, split = unit / tiles;
  int tb, ta1, ta2;
  syrk_tile(tile, (n + 63) / 64, &tb, &ta1, &ta2);
  const int r1 = ta1 * 64, r2 = (ta2 >= 0 ? ta2 : ta1) * 64, rb = tb * 64;
  const int per = (KT + splits - 1) / splits;
  const int kt0 = split * per, kt1 = min(KT, kt0 + per);
  const int nk = max(0, kt1 - kt0);
  double* As = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  double* Bs = As + T::STAGES * T::A_STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol = l2_policy_evict_first();
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&xmap);
    for (int s = 0; s < T::STAGES; ++s) {
      mbar_init(&full[s], 1);
      left_cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < T::STAGES && s < nk; ++s)
      syrk_issue(&xmap, As + s * T::A_STAGE, Bs + s * T::B_STAGE, &full[s], kt0 + s, kti, r1, r2, rb, pol);
  }
  __syncthreads();
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % T::WM) * T::TM;
  const int wn0 = (warp / T::WM) * T::TN;
  double acc[T::FM][T::FN][2];
#pragma unroll
  for (int a = 0; a < T::FM; ++a)
#pragma unroll
    for (int b = 0; b < T::FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  constexpr int KSTEPS = T::BK / 4;
  // k per lane quad per k-step: {0, 3, 12, 15} ^ {0, 1, 4, 5} (conflict-free
  // for row-major 128-byte-swizzled boxes, see tree_p_tma_kernel)
  const int kq = 3 * (tq & 1) + 12 * (tq >> 1);
  double afr[2][T::FM], bfr[2][T::FN];
  auto load_frags = [&](int buf, const double* as, const double* bs, int ks) {
    const int k = kq ^ ((ks & 1) + 4 * (ks >> 1));
    const int col = 2 * ((k >> 1) ^ gq) + (k & 1);
#pragma unroll
    for (int a = 0; a < T::FM; ++a) afr[buf][a] = as[(wm0 + a * 8 + gq) * T::BK + col];
#pragma unroll
    for (int b = 0; b < T::FN; ++b) bfr[buf][b] = bs[(wn0 + b * 8 + gq) * T::BK + col];
  };
  if (nk > 0) {
    mbar_wait(&full[0], 0u);
    load_frags(0, As, Bs, 0);
  }
  for (int j = 0; j < nk; ++j) {
    const int s = j % T::STAGES;
    const double* as = As + s * T::A_STAGE;
    const double* bs = Bs + s * T::B_STAGE;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      if (ks + 1 < KSTEPS) {
        load_frags((ks + 1) & 1, as, bs, ks + 1);
      } else {
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
            const int nj = j + T::STAGES;
            if (nj < nk) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              syrk_issue(&xmap, As + s * T::A_STAGE, Bs + s * T::B_STAGE, &full[s], kt0 + nj, kti, r1, r2,
                         rb, pol);
            }
          }
        }
        if (j + 1 < nk) {
          const int s1 = (j + 1) % T::STAGES;
          mbar_wait(&full[s1], static_cast<unsigned>(((j + 1) / T::STAGES) & 1));
          load_frags(0, As + s1 * T::A_STAGE, Bs + s1 * T::B_STAGE, 0);
        }
      }
#pragma unroll
      for (int a = 0; a < T::FM; ++a)
#pragma unroll
        for (int b = 0; b < T::FN; ++b) dmma884(acc[a][b][0], acc[a][b][1], afr[ks & 1][a], bfr[ks & 1][b]);
    }
  }
  // partial blocks -> ws[split][n][n]: (a, b) in place when a >= b, else
  // transposed into the lower block (b, a)
  double* wsb = ws + static_cast<int64_t>(split) * n * n;
  const int a = (wm0 == 0) ? ta1 : ta2;
  if (a < 0) return;
  if (a >= tb) {
#pragma unroll
    for (int fi = 0; fi < T::FM; ++fi) {
      const int m = a * 64 + fi * 8 + gq;
      if (m >= n) continue;
#pragma unroll
      for (int fj = 0; fj < T::FN; ++fj) {
        const int c = rb + wn0 + fj * 8 + 2 * tq;
        double* p = wsb + static_cast<int64_t>(m) * n + c;
        if (c + 1 < n && (n & 1) == 0) {   // 16-byte aligned rows only for even n
          *reinterpret_cast<double2*>(p) = make_double2(acc[fi][fj][0], acc[fi][fj][1]);
        } else {
          if (c < n) p[0] = acc[fi][fj][0];
          if (c + 1 < n) p[1] = acc[fi][fj][1];
        }
      }
    }
  } else {
#pragma unroll
    for (int fi = 0; fi < T::FM; ++fi) {
      const int m = a * 64 + fi * 8 + gq;   // a < tb: m < n
#pragma unroll
      for (int fj = 0; fj < T::FN; ++fj) {
        const int c = rb + wn0 + fj * 8 + 2 * tq;
        if (c < n) wsb[static_cast<int64_t>(c) * n + m] = acc[fi][fj][0];
        if (c + 1 < n) wsb[static_cast<int64_t>(c + 1) * n + m] = acc[fi][fj][1];
      }
    }
  }
}

// splits of each tile's reduction: the smallest count whose CTA total fills
// its last wave of 2 CTAs per SM to >= 98% (else the best fill), at least 8
// k-tiles per split
int syrk_splits(int64_t tiles, int64_t KT) {
  const int64_t slots = 2 * bt_num_sms();
  int best = 1;
  double best_eff = 0.0;
  for (int64_t s = 1; s <= 32 && s * 8 <= KT; ++s) {
    const int64_t ctas = tiles * s;
    const double eff = static_cast<double>(ctas) / static_cast<double>(bt_cdiv(ctas, slots) * slots);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = static_cast<int>(s);
    }
    if (eff >= 0.98) break;
  }
  return best;
}

}  // namespace

// workspace (doubles) of bt_syrk_tma for an n x n Gram
int64_t bt_syrk_tma_ws_elems(int64_t n, int64_t kt_total) {
  if (n > INT32_MAX) return 0;
  const int64_t tiles = syrk_tile(0, static_cast<int>((n + 63) / 64), nullptr, nullptr, nullptr);
  return syrk_splits(tiles, kt_total) * n * n;
}

// G (n x n) = X_(mode) X_(mode)^T for X viewed as (outer, n, inner) with
// inner contiguous.  BT_E_VALUE when the TMA map cannot address the shape
// (the caller then takes the engine).
int bt_syrk_tma(const double* x, int64_t outer, int64_t n, int64_t inner, double* g, double* ws,
                int64_t ws_elems, cudaStream_t st) {
  using T = SyrkCfg;
  if (inner % 2 != 0 || n > INT32_MAX || inner > INT32_MAX || outer > INT32_MAX ||
      (reinterpret_cast<uintptr_t>(x) & 15u) != 0)
    return BT_E_VALUE;
  const int64_t kti = (inner + T::BK - 1) / T::BK;
  const int64_t KT = kti * outer;
  if (KT > INT32_MAX) return BT_E_VALUE;
  const int64_t tiles = syrk_tile(0, static_cast<int>((n + 63) / 64), nullptr, nullptr, nullptr);
  const int64_t splits = syrk_splits(tiles, KT);
  if (splits * n * n > ws_elems || tiles * splits > INT32_MAX) return BT_E_VALUE;
  CUtensorMap xmap;
  BT_TRY(bt_tma_map_f64_3d(&xmap, x, inner, n, outer, inner, n * inner, T::BK, T::BM / 2, 1));
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(syrk_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       T::SMEM_BYTES));
    attr = true;
  }
  syrk_tma_kernel<<<static_cast<unsigned>(tiles * splits), T::THREADS, T::SMEM_BYTES, st>>>(
      xmap, static_cast<int>(n), static_cast<int>(kti), static_cast<int>(KT), static_cast<int>(splits),
      static_cast<int>(tiles), ws);
  BT_LAUNCH_CHECK();
  // fixed-order sum of the splits + mirror of the upper triangle
  BtGemmArgs r{};
  r.M = n;
  r.N = n;
  r.C = g;
  r.sCm = n;
  r.sCn = 1;
  r.splits = static_cast<int>(splits);
  r.ws = ws;
  r.symmetric = 1;
  r.alpha = 1.0;
  r.beta = 0.0;
  const unsigned rgrid = static_cast<unsigned>(std::min<int64_t>(bt_cdiv(n * n, 256), 4096));
  // mirror rule on 64-blocks: every lower 64 x 64 block (diagonal blocks in
  // full) was written
  bt_gemm_reduce_kernel<<<dim3(rgrid, 1), 256, 0, st>>>(r, T::BM / 2, T::BM / 2);
  BT_LAUNCH_CHECK();
  return BT_OK;
}
