// TMA-fed FP64 DMMA GEMM for the "transposed A" shape of the CP dimension
// tree:  C[b][m][n] = sum_k A[b][k][m] * B[k][n]
// with A row-major over (k, m) -- m contiguous, the C-order tensor read in
// place -- and B a row-major (k, n) factor.  The Q tree's
// Q[(j,k)][r] = sum_i X[i][(j,k)] A[i][r] (decomp.py:384-388's mode-2/3
// MTTKRPs share it) and the short-slab T[i] = X[i]^T B are this shape.
//
// Structure (same as cp.cu's tree_p_tma_kernel): 128 x 64 output tile, four
// DMMA warps of 64 x 32, 4 stages of 24 KB filled by cp.async.bulk.tensor
// (A: eight 16 x 16 boxes, B: four), 128-byte swizzle, the last warp out of
// a stage re-arms and refills it, 2 CTAs per SM.  Smem holds each box as
// [k][16 m] rows of 128 bytes whose 16-byte chunk c sits at c ^ (k & 7);
// the k-step gives lane quad tq the reduction index k = (ks & 1) + 2 tq +
// 8 (ks >> 1), so the 8-byte fragment reads of a half-warp (4 m-pairs x 4
// k) cover 16 distinct slots for both operands (bits 1-2 of k & 7 differ
// across tq).  Fixed summation order: bit-reproducible.
#include "gemm.cuh"
#include "tma.cuh"

namespace {

template <int BN_>
struct AtCfg {
  static constexpr int BM = 128, BN = BN_, BK = 16, STAGES = 4;
  static constexpr int WM = 2, WN = 2, THREADS = WM * WN * 32;
  static constexpr int TM = BM / WM, TN = BN / WN, FM = TM / 8, FN = TN / 8;
  static constexpr int A_STAGE = BK * BM, B_STAGE = BK * BN;  // doubles
  static constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
};

template <class T>
__device__ __forceinline__ void at_issue(const CUtensorMap* amap, const CUtensorMap* bmap, double* as,
                                         double* bs, uint64_t* bar, int k0, int m0, int n0, int b,
                                         uint64_t pol_a, uint64_t pol_b) {
  mbar_arrive_expect_tx(bar, T::STAGE_BYTES);
#pragma unroll
  for (int q = 0; q < T::BM / 16; ++q)
    tma_load_3d(as + q * 16 * T::BK, amap, bar, m0 + 16 * q, k0, b, pol_a);
#pragma unroll
  for (int q = 0; q < T::BN / 16; ++q)
    tma_load_2d(bs + q * 16 * T::BK, bmap, bar, n0 + 16 * q, k0, pol_b);
}

// TOUT: store C^T (C[b][n][m], m contiguous: ldc is the n stride) -- the
// layout of a mode product x x_k U^T over a non-last mode
template <int BN, bool TOUT>
__global__ void __launch_bounds__(AtCfg<BN>::THREADS, 2)
    gemm_at_tma_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                       int64_t M, int64_t N, int64_t Kdim, double* __restrict__ C, int64_t ldc,
                       int64_t sCb) {
  using T = AtCfg<BN>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[T::STAGES];
  __shared__ int left_cnt[T::STAGES];
  const int m0 = blockIdx.x * T::BM, n0 = blockIdx.y * T::BN, bz = blockIdx.z;
  const int KT = static_cast<int>((Kdim + T::BK - 1) / T::BK);
  double* As = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  double* Bs = As + T::STAGES * T::A_STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol_a = l2_policy_evict_first();
  const uint64_t pol_b = l2_policy_evict_last();
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&amap);
    tma_prefetch_desc(&bmap);
    for (int s = 0; s < T::STAGES; ++s) {
      mbar_init(&full[s], 1);
      left_cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < T::STAGES && s < KT; ++s)
      at_issue<T>(&amap, &bmap, As + s * T::A_STAGE, Bs + s * T::B_STAGE, &full[s], s * T::BK, m0, n0,
                  bz, pol_a, pol_b);
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
  const int g2 = gq >> 1, g1 = gq & 1;
  double afr[2][T::FM], bfr[2][T::FN];
  // element (row r of 16 within box q, reduction k) of a [q][k][16] stage
  auto load_frags = [&](int buf, const double* as, const double* bs, int ks) {
    const int k = (ks & 1) + 2 * tq + 8 * (ks >> 1);
    const int x = k & 7;
#pragma unroll
    for (int a = 0; a < T::FM; ++a) {
      const int q = (wm0 >> 4) + (a >> 1);
      afr[buf][a] = as[q * 16 * T::BK + k * 16 + 2 * ((4 * (a & 1) + g2) ^ x) + g1];
    }
#pragma unroll
    for (int b = 0; b < T::FN; ++b) {
      const int q = (wn0 >> 4) + (b >> 1);
      bfr[buf][b] = bs[q * 16 * T::BK + k * 16 + 2 * ((4 * (b & 1) + g2) ^ x) + g1];
    }
  };
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
              at_issue<T>(&amap, &bmap, As + s * T::A_STAGE, Bs + s * T::B_STAGE, &full[s], nk * T::BK,
                          m0, n0, bz, pol_a, pol_b);
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
  double* Cb = C + bz * sCb;
#pragma unroll
  for (int fi = 0; fi < T::FM; ++fi) {
    const int64_t m = m0 + wm0 + fi * 8 + gq;
    if (m >= M) continue;
#pragma unroll
    for (int fj = 0; fj < T::FN; ++fj) {
      const int64_t n = n0 + wn0 + fj * 8 + 2 * tq;
      if (TOUT) {
        // 8 consecutive m per (fj, h) across gq: 64-byte runs
        if (n < N) Cb[n * ldc + m] = acc[fi][fj][0];
        if (n + 1 < N) Cb[(n + 1) * ldc + m] = acc[fi][fj][1];
      } else {
        double* p = Cb + m * ldc + n;
        if (n + 1 < N) {
          *reinterpret_cast<double2*>(p) = make_double2(acc[fi][fj][0], acc[fi][fj][1]);
        } else if (n < N) {
          p[0] = acc[fi][fj][0];
        }
      }
    }
  }
}

template <int BN, bool TOUT>
int launch_at(const CUtensorMap& amap, const CUtensorMap& bmap, int64_t M, int64_t N, int64_t Kdim,
              double* c, int64_t ldc, int64_t sCb, int64_t batch, cudaStream_t st) {
  using T = AtCfg<BN>;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(gemm_at_tma_kernel<BN, TOUT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM_BYTES));
    attr = true;
  }
  dim3 grid(static_cast<unsigned>(bt_cdiv(M, T::BM)), static_cast<unsigned>(bt_cdiv(N, T::BN)),
            static_cast<unsigned>(batch));
  gemm_at_tma_kernel<BN, TOUT><<<grid, T::THREADS, T::SMEM_BYTES, st>>>(amap, bmap, M, N, Kdim, c, ldc,
                                                                        sCb);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

}  // namespace

// C[b] = A[b]^T B with A[b] the (Kdim x M) row-major block at a + b * sAb
// (row stride lda) and B (Kdim x N, row stride ldb).  C[b] is (M x N) with
// row stride ldc, or with transpose_out (N x M) with row stride ldc; batch
// stride sCb.  N <= 32 takes the 128 x 32 tile.  Returns BT_E_VALUE when the
// shape is outside what the TMA maps can address (the caller then uses the
// cp.async engine).
int bt_gemm_at_tma_ex(const double* a, int64_t lda, int64_t sAb, const double* b, int64_t ldb,
                      double* c, int64_t ldc, int64_t sCb, int64_t M, int64_t N, int64_t Kdim,
                      int64_t batch, int transpose_out, cudaStream_t st) {
  const bool ok = M % 2 == 0 && lda % 2 == 0 && ldb % 2 == 0 &&
                  (transpose_out || (ldc % 2 == 0 && (batch == 1 || sCb % 2 == 0))) &&
                  N % 2 == 0 && (batch == 1 || sAb % 2 == 0) &&
                  ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                    reinterpret_cast<uintptr_t>(c)) & 15u) == 0 &&
                  M <= INT32_MAX && N <= INT32_MAX && Kdim <= INT32_MAX && batch <= 65535 &&
                  bt_cdiv(N, 32) <= 65535 && Kdim >= 1;
  if (!ok) return BT_E_VALUE;
  CUtensorMap amap, bmap;
  BT_TRY(bt_tma_map_f64_3d(&amap, a, M, Kdim, batch, lda, batch > 1 ? sAb : lda * Kdim, 16,
                           AtCfg<64>::BK, 1));
  BT_TRY(bt_tma_map_f64_2d(&bmap, b, N, Kdim, ldb, 16, AtCfg<64>::BK));
  if (N <= 32)
    return transpose_out ? launch_at<32, true>(amap, bmap, M, N, Kdim, c, ldc, sCb, batch, st)
                         : launch_at<32, false>(amap, bmap, M, N, Kdim, c, ldc, sCb, batch, st);
  return transpose_out ? launch_at<64, true>(amap, bmap, M, N, Kdim, c, ldc, sCb, batch, st)
                       : launch_at<64, false>(amap, bmap, M, N, Kdim, c, ldc, sCb, batch, st);
}

int bt_gemm_at_tma(const double* a, int64_t lda, int64_t sAb, const double* b, int64_t ldb, double* c,
                   int64_t ldc, int64_t sCb, int64_t M, int64_t N, int64_t Kdim, int64_t batch,
                   cudaStream_t st) {
  return bt_gemm_at_tma_ex(a, lda, sAb, b, ldb, c, ldc, sCb, M, N, Kdim, batch, 0, st);
}
