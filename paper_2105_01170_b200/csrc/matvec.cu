// K11: structured matvecs for many right-hand sides (reconstruct.py:271-315;
// the reference loops over terms and over every grid cell in Python and
// handles one vector at a time).
//
//   Kron-sum : Z_j = D_j X (one batched DMMA GEMM over all terms and RHS),
//              then y[:, block i] = sum_{cells (i,c) of class k} sum_j
//              (coeffs[k,j] / sqrt(eta_k)) Z_j[:, c]        (CTA per block row)
//   BLR      : Z = R^T X (DMMA GEMM); yb_i = sum_{cells (i,j)} (S_k/sqrt(eta_k)) Z_j
//              (CTA per block row, the per-cell 2-D products on DMMA with
//              cp.async double buffering); y = L yb (DMMA GEMM)
//   multilevel (no reference counterpart; cli.py:247-248 densifies):
//              y = sum_r (S1_r (x) S2_r (x) S3_r) x as three batched DMMA mode
//              products over the volume batch, the last one reducing over r.
// Flop counts per RHS equal the reference's FlopCounter formulas.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gemm.cuh"

int bt_gemm_run(BtGemmArgs g, int64_t batch, cudaStream_t st, int want_splits, int64_t ws_elems);
// gemm_tma.cu: C[b] = A[b]^T B on the TMA-fed DMMA kernel (BT_E_VALUE: shape not addressable)
int bt_gemm_at_tma_ex(const double* a, int64_t lda, int64_t sAb, const double* b, int64_t ldb,
                      double* c, int64_t ldc, int64_t sCb, int64_t M, int64_t N, int64_t Kdim,
                      int64_t batch, int transpose_out, cudaStream_t st);
int64_t bt_gemm_ws_elems(BtGemmArgs g, int64_t batch);

namespace {

int grid1d(int64_t n) { return static_cast<int>(std::min<int64_t>(bt_cdiv(n, 256), 8192)); }

// X2[(c * nrhs + s)][b] = x[s][c * n + b]
__global__ void kron_permute_kernel(const double* __restrict__ x, int64_t nrhs, int64_t q,
                                    int64_t n, double* __restrict__ x2) {
  const int64_t total = nrhs * q * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx % n;
    const int64_t s = (idx / n) % nrhs;
    const int64_t c = idx / (n * nrhs);
    x2[idx] = x[(s * q + c) * n + b];
  }
}

// W[k][j] = coeffs[k][j] / sqrt(eta_k)   (reconstruct.py:97)
__global__ void kron_weights_kernel(const double* __restrict__ coeffs, const int64_t* __restrict__ eta,
                                    int64_t p, int64_t r, double* __restrict__ w) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < p * r;
       idx += (int64_t)gridDim.x * blockDim.x)
    w[idx] = coeffs[idx] / sqrt(static_cast<double>(eta[idx / r]));
}

// y[s][i*m + a] = sum_{cells (i,c,k)} sum_j W[k][j] Z[j][a][c*nrhs + s]
__global__ void __launch_bounds__(256)
    kron_combine_kernel(const double* __restrict__ z, const double* __restrict__ w,
                        const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ row_cells,
                        int64_t p, int64_t r, int64_t m, int64_t q, int64_t nrhs, int64_t ell,
                        double* __restrict__ y) {
  const int64_t i = blockIdx.x;
  const int64_t ms = m * nrhs;
  const int64_t zj = m * q * nrhs;  // stride between terms
  for (int64_t e = threadIdx.x + (int64_t)blockIdx.y * blockDim.x; e < ms;
       e += (int64_t)gridDim.y * blockDim.x) {
    const int64_t a = e / nrhs, s = e % nrhs;
    double acc = 0.0;
    for (int64_t cc = row_ptr[i]; cc < row_ptr[i + 1]; ++cc) {
      const int64_t code = row_cells[cc];
      const int64_t c = code / p, k = code % p;
      const double* zc = z + a * q * nrhs + c * nrhs + s;
      const double* wk = w + k * r;
      for (int64_t j = 0; j < r; ++j) acc = fma(wk[j], zc[j * zj], acc);
    }
    y[s * ell * m + i * m + a] = acc;
  }
}

// ---------------------------------------------------------------------------
// BLR middle product on DMMA
// ---------------------------------------------------------------------------

// Shat[k] = S[k] / sqrt(eta_k)  (reconstruct.py:305), padded to (RLP x RRP)
__global__ void blr_scale_kernel(const double* __restrict__ mid, const int64_t* __restrict__ eta,
                                 int64_t p, int64_t rl, int64_t rr, double* __restrict__ out) {
  const int64_t tot = p * rl * rr;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x)
    out[idx] = mid[idx] / sqrt(static_cast<double>(eta[idx / (rl * rr)]));
}

// yb[s][i][rho'] = sum_{cells (i, j, k)} sum_rho Shat[k][rho'][rho] Z[s*q + j][rho]
// CTA: one block row i, one RHS tile of NB; output tile RLP x NB.
template <int RLP, int RRP, int NB>
__global__ void __launch_bounds__(256)
    blr_middle_kernel(const double* __restrict__ shat, const double* __restrict__ z,
                      const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ row_cells,
                      int64_t p, int64_t rl, int64_t rr, int64_t q, int64_t nrhs, int64_t ell,
                      double* __restrict__ yb) {
  constexpr int LDS = bt_ld(RRP);  // S tile [rho'][rho] (k-contig for A)
  constexpr int LDZ = bt_ld(RRP);  // Z tile [s][rho]   (k-contig for B)
  constexpr int WM = RLP / 16 > 0 ? (RLP >= 32 ? 2 : 1) : 1;
  constexpr int WN = 8 / WM;
  constexpr int TM = RLP / WM, TN = NB / WN;
  constexpr int FM = TM / 8, FN = TN / 8;
  static_assert(FM >= 1 && FN >= 1, "tile too small");
  extern __shared__ __align__(16) double sm[];
  double* Ss = sm;                     // 2 stages of RLP x LDS
  double* Zs = Ss + 2 * RLP * LDS;     // 2 stages of NB x LDZ
  const int64_t i = blockIdx.x;
  const int64_t s0 = blockIdx.y * (int64_t)NB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % WM) * TM, wn0 = (warp / WM) * TN;
  const int64_t c0 = row_ptr[i], c1 = row_ptr[i + 1];
  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  auto load = [&](int stage, int64_t cell) {
    const int64_t code = row_cells[cell];
    const int64_t j = code / p, k = code % p;
    double* sd = Ss + stage * RLP * LDS;
    double* zd = Zs + stage * NB * LDZ;
    const double* sk = shat + k * rl * rr;
    for (int idx = threadIdx.x; idx < RLP * RRP; idx += 256) {
      const int a = idx / RRP, b = idx % RRP;
      const bool v = a < rl && b < rr;
      cp_async8(sd + a * LDS + b, v ? sk + a * rr + b : sk, v ? 8 : 0);
    }
    for (int idx = threadIdx.x; idx < NB * RRP; idx += 256) {
      const int sl = idx / RRP, b = idx % RRP;
      const int64_t s = s0 + sl;
      const bool v = s < nrhs && b < rr;
      const double* src = z + (s * q + j) * rr + b;
      cp_async8(zd + sl * LDZ + b, v ? src : z, v ? 8 : 0);
    }
  };

  if (c0 < c1) load(0, c0);
  cp_async_commit();
  for (int64_t cell = c0; cell < c1; ++cell) {
    const int stage = static_cast<int>((cell - c0) & 1);
    if (cell + 1 < c1) load(stage ^ 1, cell + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* sd = Ss + stage * RLP * LDS;
    const double* zd = Zs + stage * NB * LDZ;
#pragma unroll
    for (int kk = 0; kk < RRP; kk += 4) {
      double av[FM], bv[FN];
#pragma unroll
      for (int a = 0; a < FM; ++a) av[a] = sd[(wm0 + a * 8 + gq) * LDS + kk + tq];
#pragma unroll
      for (int b = 0; b < FN; ++b) bv[b] = zd[(wn0 + b * 8 + gq) * LDZ + kk + tq];
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int64_t rho = wm0 + a * 8 + gq;
    if (rho >= rl) continue;
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t s = s0 + wn0 + b * 8 + 2 * tq + h;
        if (s < nrhs) yb[(s * ell + i) * rl + rho] = acc[a][b][h];
      }
  }
}

// Row-group variant of the middle products for dense-map patterns (every
// cell's class read from cell_class): a CTA owns BM / RLP consecutive block
// rows and 64 right-hand sides and walks the block columns j, so each Z_j
// tile is loaded once for all its block rows and every stage feeds 32 DMMAs
// per warp (4 warps of 64x32 -- the engine's tuned tile).  The A tile stacks
// the rows' middles S_{class(i, j)} (zero for uncovered cells); BK = 16 over
// the rr columns.  The block columns are split over gridDim.z with partials
// reduced in a fixed order (deterministic).
// BN = 64: 4 warps of 64x32 (2 x 2); BN = 32 / 16 (few right-hand sides: C3's
// 16): 4 warps of 32 x BN stacked along the rows, so the tile carries no
// all-zero RHS columns (the 64-wide tile ran 16 RHS at 7.6 TF/s, 3/4 of its
// DMMAs on padding).
template <int BN_>
struct BlrRows {
  static constexpr int BM = 128, BN = BN_, BK = 16, STAGES = 3, THREADS = 128;
  static constexpr int LDA = bt_ld(BK), LDB = bt_ld(BK);
  static constexpr int A_STAGE = BM * LDA, B_STAGE = BN * LDB;
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * 8;
  static constexpr int WM = BN_ >= 64 ? 2 : 4;                 // warps along the rows
  static constexpr int TM = BM / WM, TN = BN / (4 / WM), FM = TM / 8, FN = TN / 8;
  static constexpr int BCH = BN * 8 / THREADS;                // 16-byte B chunks per thread
  static_assert(BN_ == 16 || BN_ == 32 || BN_ == 64, "RHS tile of 16, 32 or 64");
};
inline int blr_rows_bn(int64_t nrhs) { return nrhs <= 16 ? 16 : (nrhs <= 32 ? 32 : 64); }

template <int RLP, int BN_>
__global__ void __launch_bounds__(BlrRows<BN_>::THREADS)
    blr_rows_kernel(const double* __restrict__ shat, const double* __restrict__ z,
                    const int32_t* __restrict__ cell_class, int64_t rl, int64_t rr, int64_t q,
                    int64_t nrhs, int64_t ell, int64_t jchunk, double* __restrict__ out,
                    int64_t out_split_stride) {
  using Cfg = BlrRows<BN_>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES, THREADS = Cfg::THREADS;
  constexpr int LDA = Cfg::LDA, LDB = Cfg::LDB, A_STAGE = Cfg::A_STAGE, B_STAGE = Cfg::B_STAGE;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, FM = Cfg::FM, FN = Cfg::FN, BCH = Cfg::BCH;
  constexpr int R = BM / RLP;  // block rows per CTA
  extern __shared__ __align__(16) double sm[];
  double* As = sm;
  double* Bs = sm + STAGES * A_STAGE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WM) * TM, wn0 = (warp / Cfg::WM) * TN;
  const int64_t i0 = blockIdx.x * (int64_t)R;
  const int64_t s0 = blockIdx.y * (int64_t)BN;
  const int64_t j0 = blockIdx.z * jchunk;
  const int64_t j1 = std::min<int64_t>(q, j0 + jchunk);
  const int ktc = static_cast<int>((rr + BK - 1) / BK);
  const int64_t T = (j1 > j0 ? (j1 - j0) : 0) * ktc;
  const int64_t zrow = q * rr;  // stride between right-hand sides in Z

  // per-thread chunk coordinates (16-byte chunks: 8 per 16-wide row)
  // A: 128 rows x 8 chunks = 1024 -> 8 per thread; B: 64 x 8 = 512 -> 4 per thread
  int a_r[8], a_c[8];
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int idx = threadIdx.x + it * THREADS;
    a_r[it] = idx >> 3;
    a_c[it] = (idx & 7) * 2;
  }
  int b_r[BCH], b_c[BCH];
#pragma unroll
  for (int it = 0; it < BCH; ++it) {
    const int idx = threadIdx.x + it * THREADS;
    b_r[it] = idx >> 3;
    b_c[it] = (idx & 7) * 2;
  }
  int64_t l_j = j0;
  int l_kt = 0;
  int cls[R];
  auto load_stage = [&](int stage) {
    if (l_kt == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        cls[r] = (i0 + r < ell) ? __ldg(cell_class + (i0 + r) * q + l_j) : -1;
    }
    const int k0 = l_kt * BK;
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * B_STAGE;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int m = a_r[it];
      const int r = m / RLP, rho = m - r * RLP;
      const int k = cls[r];
      const int64_t cl = rr - k0 - a_c[it];
      const int valid = (k >= 0 && rho < rl && cl > 0) ? static_cast<int>(cl >= 2 ? 16 : cl * 8) : 0;
      const double* src = valid ? shat + (static_cast<int64_t>(k) * rl + rho) * rr + k0 + a_c[it]
                                : shat;
      cp_async16(as + m * LDA + a_c[it], src, valid);
    }
#pragma unroll
    for (int it = 0; it < BCH; ++it) {
      const int n = b_r[it];
      const int64_t s = s0 + n;
      const int64_t cl = rr - k0 - b_c[it];
      const int valid = (s < nrhs && cl > 0) ? static_cast<int>(cl >= 2 ? 16 : cl * 8) : 0;
      const double* src = valid ? z + s * zrow + l_j * rr + k0 + b_c[it] : z;
      cp_async16(bs + n * LDB + b_c[it], src, valid);
    }
    if (++l_kt == ktc) {
      l_kt = 0;
      ++l_j;
    }
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < T) load_stage(st);
    cp_async_commit();
  }
  int stage = 0, next_stage = STAGES - 1;
  double afr[2][FM], bfr[2][FN];
  for (int64_t t = 0; t < T; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const double* as = As + stage * A_STAGE;
    const double* bs = Bs + stage * B_STAGE;
    auto frags = [&](int buf, int kk) {
#pragma unroll
      for (int a = 0; a < FM; ++a) afr[buf][a] = as[(wm0 + a * 8 + gq) * LDA + kk + tq];
#pragma unroll
      for (int b = 0; b < FN; ++b) bfr[buf][b] = bs[(wn0 + b * 8 + gq) * LDB + kk + tq];
    };
    frags(0, 0);
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      if (ks + 1 < BK / 4) frags((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][0], acc[a][b][1], afr[ks & 1][a], bfr[ks & 1][b]);
      if (ks == 0) {
        if (t + STAGES - 1 < T) load_stage(next_stage);
        cp_async_commit();
      }
    }
    stage = (stage + 1 == STAGES) ? 0 : stage + 1;
    next_stage = (next_stage + 1 == STAGES) ? 0 : next_stage + 1;
  }
  cp_async_wait<0>();
  // out[(s * ell + i) * rl + rho] (+ split offset)
  double* o = out + blockIdx.z * out_split_stride;
#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int m = wm0 + a * 8 + gq;
    const int r = m / RLP, rho = m - r * RLP;
    const int64_t i = i0 + r;
    if (rho >= rl || i >= ell) continue;
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t s = s0 + wn0 + b * 8 + 2 * tq + h;
        if (s < nrhs) o[(s * ell + i) * rl + rho] = acc[a][b][h];
      }
  }
}

// yb = sum over splits of part (fixed order)
__global__ void split_sum_kernel(const double* __restrict__ part, int64_t n, int splits,
                                 double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = part[e];
    for (int sidx = 1; sidx < splits; ++sidx) acc += part[sidx * n + e];
    out[e] = acc;
  }
}

// splits of the block-column range that fill whole waves of resident CTAs
int blr_rows_splits(int64_t ctas, int64_t q, int resident) {
  const int64_t slots = static_cast<int64_t>(bt_num_sms()) * std::max(resident, 1);
  int best = 1;
  double best_eff = 0.0;
  for (int sp = 1; sp <= 16 && sp <= q; ++sp) {
    const double waves = static_cast<double>(ctas * sp) / static_cast<double>(slots);
    const double eff = waves / std::ceil(waves);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = sp;
    }
  }
  return best;
}

template <int RLP, int BN_>
int launch_blr_rows_t(const double* shat, const double* z, const int32_t* cell_class, int64_t rl,
                      int64_t rr, int64_t q, int64_t nrhs, int64_t ell, double* yb, double* part,
                      int splits, cudaStream_t st) {
  using Cfg = BlrRows<BN_>;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(blr_rows_kernel<RLP, BN_>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    attr = true;
  }
  constexpr int R = Cfg::BM / RLP;
  const int64_t jchunk = bt_cdiv(q, splits);
  dim3 grid(static_cast<unsigned>(bt_cdiv(ell, R)), static_cast<unsigned>(bt_cdiv(nrhs, Cfg::BN)),
            static_cast<unsigned>(splits));
  const int64_t nout = nrhs * ell * rl;
  blr_rows_kernel<RLP, BN_><<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(
      shat, z, cell_class, rl, rr, q, nrhs, ell, jchunk, splits > 1 ? part : yb, nout);
  BT_LAUNCH_CHECK();
  if (splits > 1) {
    split_sum_kernel<<<grid1d(nout), 256, 0, st>>>(part, nout, splits, yb);
    BT_LAUNCH_CHECK();
  }
  return BT_OK;
}

template <int RLP>
int launch_blr_rows(const double* shat, const double* z, const int32_t* cell_class, int64_t rl,
                    int64_t rr, int64_t q, int64_t nrhs, int64_t ell, double* yb, double* part,
                    int splits, cudaStream_t st) {
  const int bn = blr_rows_bn(nrhs);
  if (bn == 16)
    return launch_blr_rows_t<RLP, 16>(shat, z, cell_class, rl, rr, q, nrhs, ell, yb, part, splits, st);
  if (bn == 32)
    return launch_blr_rows_t<RLP, 32>(shat, z, cell_class, rl, rr, q, nrhs, ell, yb, part, splits, st);
  return launch_blr_rows_t<RLP, 64>(shat, z, cell_class, rl, rr, q, nrhs, ell, yb, part, splits, st);
}

template <int RLP, int BN_>
int blr_rows_resident_t() {
  using Cfg = BlrRows<BN_>;
  int per_sm = 0;
  cudaFuncSetAttribute(blr_rows_kernel<RLP, BN_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)Cfg::SMEM);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, blr_rows_kernel<RLP, BN_>, Cfg::THREADS,
                                                    Cfg::SMEM) != cudaSuccess)
    per_sm = 1;
  return per_sm;
}

template <int RLP>
int blr_rows_resident(int64_t nrhs) {
  const int bn = blr_rows_bn(nrhs);
  return bn == 16 ? blr_rows_resident_t<RLP, 16>()
                  : (bn == 32 ? blr_rows_resident_t<RLP, 32>() : blr_rows_resident_t<RLP, 64>());
}

template <int RLP, int RRP, int NB>
int launch_blr_middle(const double* shat, const double* z, const int64_t* row_ptr,
                      const int64_t* row_cells, int64_t p, int64_t rl, int64_t rr, int64_t q,
                      int64_t nrhs, int64_t ell, double* yb, cudaStream_t st) {
  constexpr size_t SM = (size_t)(2 * RLP * bt_ld(RRP) + 2 * NB * bt_ld(RRP)) * 8;
  static bool attr = false;
  if (!attr) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(blr_middle_kernel<RLP, RRP, NB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM));
    attr = true;
  }
  dim3 grid(static_cast<unsigned>(ell), static_cast<unsigned>(bt_cdiv(nrhs, NB)));
  blr_middle_kernel<RLP, RRP, NB><<<grid, 256, SM, st>>>(shat, z, row_ptr, row_cells, p, rl, rr,
                                                         q, nrhs, ell, yb);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

struct KronPlan {
  int64_t off_x2, off_w, off_z, off_gws, total;
};

KronPlan kron_plan(const bt_pattern_dev* pat, int64_t r, int64_t nrhs) {
  KronPlan k;
  int64_t o = 0;
  auto take = [&](int64_t n) {
    int64_t at = o;
    o += (n + 1) / 2 * 2;
    return at;
  };
  k.off_x2 = take(pat->q * pat->n * nrhs);
  k.off_w = take(pat->p * r);
  k.off_z = take(r * pat->m * pat->q * nrhs);
  BtGemmArgs g{};
  g.M = pat->m;
  g.N = pat->q * nrhs;
  g.Kin = pat->n;
  g.Kout = 1;
  k.off_gws = take(bt_gemm_ws_elems(g, r));
  k.total = o;
  return k;
}

struct BlrPlan {
  int64_t off_shat, off_z, off_yb, off_part, off_gws, total;
  int rows;    // 1: row-group kernel (blr_rows_kernel), 0: per-row kernel
  int splits;  // block-column splits of the row-group kernel
};

BlrPlan blr_plan(const bt_pattern_dev* pat, int64_t rl, int64_t rr, int64_t nrhs) {
  BlrPlan b;
  static const bool no_rows = getenv("BT_BLR_ROWS") && getenv("BT_BLR_ROWS")[0] == '0';
  b.rows = (!no_rows && pat->cell_class != nullptr && rl <= 64 && rr % 2 == 0) ? 1 : 0;
  b.splits = 1;
  if (b.rows) {
    const int rlp = rl <= 32 ? 32 : 64;
    const int resident = rlp == 32 ? blr_rows_resident<32>(nrhs) : blr_rows_resident<64>(nrhs);
    const int64_t ctas = bt_cdiv(pat->ell, 128 / rlp) * bt_cdiv(nrhs, blr_rows_bn(nrhs));
    b.splits = blr_rows_splits(ctas, pat->q, resident);
  }
  int64_t o = 0;
  auto take = [&](int64_t n) {
    int64_t at = o;
    o += (n + 1) / 2 * 2;
    return at;
  };
  b.off_shat = take(pat->p * rl * rr);
  b.off_z = take(pat->q * nrhs * rr);
  b.off_yb = take(nrhs * pat->ell * rl);
  b.off_part = take(b.splits > 1 ? b.splits * nrhs * pat->ell * rl : 0);
  BtGemmArgs g1{};
  g1.M = pat->q * nrhs;
  g1.N = rr;
  g1.Kin = pat->n;
  g1.Kout = 1;
  BtGemmArgs g2{};
  g2.M = nrhs * pat->ell;
  g2.N = pat->m;
  g2.Kin = rl;
  g2.Kout = 1;
  b.off_gws = take(std::max(bt_gemm_ws_elems(g1, 1), bt_gemm_ws_elems(g2, 1)));
  b.total = o;
  return b;
}

}  // namespace

extern "C" int64_t bt_matvec_kron_ws_bytes(const bt_pattern_dev* pat, int64_t r, int64_t nrhs) {
  return kron_plan(pat, r, nrhs).total * 8;
}

extern "C" int bt_matvec_kron_f64(const bt_pattern_dev* pat, const int64_t* row_ptr,
                                  const int64_t* row_cells, const double* coeffs,
                                  const double* terms, int64_t r, const double* x, int64_t nrhs,
                                  double* y, void* wsv, int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_matvec_kron_f64");
  BT_REQUIRE(r >= 1 && nrhs >= 1, BT_E_SHAPE, "matvec_kron: empty terms or RHS");
  KronPlan kp = kron_plan(pat, r, nrhs);
  BT_REQUIRE(ws_bytes >= kp.total * 8, BT_E_VALUE, "matvec_kron: workspace too small");
  cudaStream_t st = bt_stream(stream);
  double* ws = static_cast<double*>(wsv);
  const int64_t m = pat->m, n = pat->n, q = pat->q, p = pat->p, ell = pat->ell;
  double* x2 = ws + kp.off_x2;
  double* w = ws + kp.off_w;
  double* z = ws + kp.off_z;
  kron_permute_kernel<<<grid1d(nrhs * q * n), 256, 0, st>>>(x, nrhs, q, n, x2);
  BT_LAUNCH_CHECK();
  kron_weights_kernel<<<grid1d(p * r), 256, 0, st>>>(coeffs, pat->eta, p, r, w);
  BT_LAUNCH_CHECK();
  // Z[j][a][col] = sum_b D_j[a][b] X2[col][b]
  BtGemmArgs g{};
  g.M = m;
  g.N = q * nrhs;
  g.Kin = n;
  g.Kout = 1;
  g.A = BtOperand{terms, n, 0, 1, m * n};
  g.B = BtOperand{x2, n, 0, 1, 0};
  g.C = z;
  g.sCm = q * nrhs;
  g.sCn = 1;
  g.sCb = m * q * nrhs;
  g.alpha = 1.0;
  g.ws = ws + kp.off_gws;
  BT_TRY(bt_gemm_run(g, r, st, 0, kp.total - kp.off_gws));
  const int64_t ms = m * nrhs;
  dim3 grid(static_cast<unsigned>(ell), static_cast<unsigned>(std::min<int64_t>(bt_cdiv(ms, 256), 64)));
  kron_combine_kernel<<<grid, 256, 0, st>>>(z, w, row_ptr, row_cells, p, r, m, q, nrhs, ell, y);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

extern "C" int64_t bt_matvec_blr_ws_bytes(const bt_pattern_dev* pat, int64_t rl, int64_t rr,
                                          int64_t nrhs) {
  return blr_plan(pat, rl, rr, nrhs).total * 8;
}

extern "C" int bt_matvec_blr_f64(const bt_pattern_dev* pat, const int64_t* row_ptr,
                                 const int64_t* row_cells, const double* left, int64_t rl,
                                 const double* right, int64_t rr, const double* middles,
                                 const double* x, int64_t nrhs, double* y, void* wsv,
                                 int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_matvec_blr_f64");
  BT_REQUIRE(rl >= 1 && rr >= 1 && nrhs >= 1, BT_E_SHAPE, "matvec_blr: empty operand");
  BT_REQUIRE(rl <= 64 && rr <= 64, BT_E_SHAPE, "matvec_blr: side ranks above 64 not supported");
  BlrPlan bp = blr_plan(pat, rl, rr, nrhs);
  BT_REQUIRE(ws_bytes >= bp.total * 8, BT_E_VALUE, "matvec_blr: workspace too small");
  cudaStream_t st = bt_stream(stream);
  double* ws = static_cast<double*>(wsv);
  const int64_t m = pat->m, n = pat->n, q = pat->q, p = pat->p, ell = pat->ell;
  double* shat = ws + bp.off_shat;
  double* z = ws + bp.off_z;
  double* yb = ws + bp.off_yb;
  double* gws = ws + bp.off_gws;
  const int64_t gws_n = bp.total - bp.off_gws;
  blr_scale_kernel<<<grid1d(p * rl * rr), 256, 0, st>>>(middles, pat->eta, p, rl, rr, shat);
  BT_LAUNCH_CHECK();
  // Z[(s*q + c)][rho] = sum_b x[s][c*n + b] R[b][rho]
  BtGemmArgs g1{};
  g1.M = q * nrhs;
  g1.N = rr;
  g1.Kin = n;
  g1.Kout = 1;
  g1.A = BtOperand{x, n, 0, 1, 0};
  g1.B = BtOperand{right, 1, 0, rr, 0};
  g1.C = z;
  g1.sCm = rr;
  g1.sCn = 1;
  g1.alpha = 1.0;
  g1.ws = gws;
  BT_TRY(bt_gemm_run(g1, 1, st, 0, gws_n));
  // middle products
  if (bp.rows) {
    double* part = ws + bp.off_part;
    if (rl <= 32)
      BT_TRY(launch_blr_rows<32>(shat, z, pat->cell_class, rl, rr, q, nrhs, ell, yb, part,
                                 bp.splits, st));
    else
      BT_TRY(launch_blr_rows<64>(shat, z, pat->cell_class, rl, rr, q, nrhs, ell, yb, part,
                                 bp.splits, st));
  } else if (rl <= 32 && rr <= 32) {
    int rc = launch_blr_middle<32, 32, 64>(shat, z, row_ptr, row_cells, p, rl, rr, q, nrhs, ell,
                                           yb, st);
    BT_TRY(rc);
  } else {
    int rc = launch_blr_middle<64, 64, 64>(shat, z, row_ptr, row_cells, p, rl, rr, q, nrhs, ell,
                                           yb, st);
    BT_TRY(rc);
  }
  // y[(s*ell + i)][a] = sum_rho' yb[(s*ell + i)][rho'] L[a][rho']
  BtGemmArgs g2{};
  g2.M = nrhs * ell;
  g2.N = m;
  g2.Kin = rl;
  g2.Kout = 1;
  g2.A = BtOperand{yb, rl, 0, 1, 0};
  g2.B = BtOperand{left, rl, 0, 1, 0};
  g2.C = y;
  g2.sCm = m;
  g2.sCn = 1;
  g2.alpha = 1.0;
  g2.ws = gws;
  return bt_gemm_run(g2, 1, st, 0, gws_n);
}

// ---------------------------------------------------------------------------
// multilevel Kronecker sum
// ---------------------------------------------------------------------------

namespace {

struct MlPlan {
  int64_t chunk, off_u, off_w2, off_gws, off_fac, total;
};

// out[(i d1 + j) d2 + k] = in[i s0 + j s1 + k s2]: the level matrices restacked
// K-major for the TMA kernel (a few hundred KB per call)
__global__ void restack_kernel(const double* __restrict__ in, double* __restrict__ out, int64_t d0,
                               int64_t d1, int64_t d2, int64_t s0, int64_t s1, int64_t s2) {
  const int64_t n = d0 * d1 * d2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e % d2, j = (e / d2) % d1, i = e / (d1 * d2);
    out[e] = in[i * s0 + j * s1 + k * s2];
  }
}

bool ml_use_tma() {   // read per call: the route-against-route test switches it in-process
  return !(getenv("BT_ML_TMA") && getenv("BT_ML_TMA")[0] == '0');
}

MlPlan ml_plan(int64_t R, const int64_t* nin, const int64_t* nout, int64_t nrhs) {
  // nin = (N3i, N2i, N1i), nout = (N3o, N2o, N1o)
  MlPlan m;
  // U of the engine route ([a3][a2][r][i1]) or of the TMA route ([a3][a1][r][i2])
  const int64_t per_u = std::max(nin[0] * nin[1] * R * nout[2], nin[0] * nin[2] * R * nout[1]);
  const int64_t per_w = nin[0] * R * nout[1] * nout[2];
  const int64_t budget = int64_t(1) << 28;  // ~2 GiB per intermediate
  m.chunk = std::max<int64_t>(1, std::min<int64_t>(nrhs, budget / std::max(per_u, per_w)));
  int64_t o = 0;
  auto take = [&](int64_t n) {
    int64_t at = o;
    o += (n + 1) / 2 * 2;
    return at;
  };
  m.off_u = take(m.chunk * per_u);
  m.off_w2 = take(m.chunk * per_w);
  BtGemmArgs g{};
  g.M = m.chunk * nin[0] * nin[1];
  g.N = R * nout[2];
  g.Kin = nin[2];
  g.Kout = 1;
  int64_t w1 = bt_gemm_ws_elems(g, 1);
  BtGemmArgs g2{};
  g2.M = nout[1];
  g2.N = nout[2];
  g2.Kin = nin[1];
  g2.Kout = 1;
  int64_t w2 = bt_gemm_ws_elems(g2, m.chunk * nin[0]);
  BtGemmArgs g3{};
  g3.M = nout[0];
  g3.N = nout[1] * nout[2];
  g3.Kin = nin[0];
  g3.Kout = R;
  int64_t w3 = bt_gemm_ws_elems(g3, m.chunk);
  m.off_gws = take(std::max(w1, std::max(w2, w3)));
  m.off_fac = take(R * (nin[1] * nout[1] + nin[2] * nout[2] + nin[0] * nout[0]));
  m.total = o;
  return m;
}

}  // namespace

extern "C" int64_t bt_ml_matvec_ws_bytes(int64_t nterms, const int64_t* nin, const int64_t* nout,
                                         int64_t nrhs) {
  return ml_plan(nterms, nin, nout, nrhs).total * 8;
}

extern "C" int bt_ml_matvec_f64(int64_t nterms, const int64_t* nin, const int64_t* nout,
                                const double* s1, const double* s2, const double* s3,
                                const double* x, int64_t nrhs, double* y, void* wsv,
                                int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_ml_matvec_f64");
  BT_REQUIRE(nterms >= 1 && nrhs >= 1, BT_E_SHAPE, "ml_matvec: empty terms or RHS");
  const int64_t R = nterms;
  MlPlan mp = ml_plan(R, nin, nout, nrhs);
  BT_REQUIRE(ws_bytes >= mp.total * 8, BT_E_VALUE, "ml_matvec: workspace too small");
  cudaStream_t st = bt_stream(stream);
  double* ws = static_cast<double*>(wsv);
  double* U = ws + mp.off_u;
  double* W2 = ws + mp.off_w2;
  double* gws = ws + mp.off_gws;
  const int64_t gws_n = mp.total - mp.off_gws;
  const int64_t N3i = nin[0], N2i = nin[1], N1i = nin[2];
  const int64_t N3o = nout[0], N2o = nout[1], N1o = nout[2];
  // ---- TMA route: the three mode products as C[b] = A[b]^T B with the
  // tensor slab as A (its inner extent is M) and a K-major restack of the
  // level matrices as B -- no product contracts the innermost index of its
  // input, because each store rotates the layout:
  //   1. over a2:  U[(s,a3)][a1][(r,i2)]   = x[(s,a3)][a2][a1]^T S2T[a2][(r,i2)]
  //   2. over a1:  W[(s,a3)][r][i2][i1]    = U[(s,a3)][a1][r,i2]^T S3T_r[a1][i1]     (per r)
  //   3. over (a3,r), transposed store:  y[s][i3][(i2,i1)] = (W[s][(a3,r)][(i2,i1)]^T S1K[(a3,r)][i3])^T
  // C4 (128^3, 16 terms, 32 volumes): see DESIGN.md K11.  Even extents and
  // 16-byte aligned buffers only; anything else takes the engine route below.
  const bool even = !((N3i | N2i | N1i | N3o | N2o | N1o) & 1);
  if (ml_use_tma() && even && mp.chunk * N3i <= 65535 &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
        reinterpret_cast<uintptr_t>(ws)) & 15u) == 0) {
    double* S2T = ws + mp.off_fac;                 // [a2][(r,i2)]
    double* S3T = S2T + R * N2i * N2o;             // [r][a1][i1]
    double* S1K = S3T + R * N1i * N1o;             // [(a3,r)][i3]
    restack_kernel<<<grid1d(R * N2i * N2o), 256, 0, st>>>(s2, S2T, N2i, R, N2o, 1, N2o * N2i, N2i);
    BT_LAUNCH_CHECK();
    restack_kernel<<<grid1d(R * N1i * N1o), 256, 0, st>>>(s3, S3T, R, N1i, N1o, N1o * N1i, 1, N1i);
    BT_LAUNCH_CHECK();
    restack_kernel<<<grid1d(R * N3i * N3o), 256, 0, st>>>(s1, S1K, N3i, R, N3o, 1, N3o * N3i, N3i);
    BT_LAUNCH_CHECK();
    bool fell_back = false;
    for (int64_t s0 = 0; s0 < nrhs && !fell_back; s0 += mp.chunk) {
      const int64_t ns = std::min(mp.chunk, nrhs - s0);
      const double* xs = x + s0 * N3i * N2i * N1i;
      double* ys = y + s0 * N3o * N2o * N1o;
      int rc = bt_gemm_at_tma_ex(xs, N1i, N2i * N1i, S2T, R * N2o, U, R * N2o, N1i * R * N2o, N1i,
                                 R * N2o, N2i, ns * N3i, 0, st);
      if (rc == BT_E_VALUE && s0 == 0) {
        fell_back = true;   // nothing of y written yet: the engine route runs instead
        break;
      }
      BT_TRY(rc);
      for (int64_t r = 0; r < R; ++r)
        BT_TRY(bt_gemm_at_tma_ex(U + r * N2o, R * N2o, N1i * R * N2o, S3T + r * N1i * N1o, N1o,
                                 W2 + r * N2o * N1o, N1o, R * N2o * N1o, N2o, N1o, N1i, ns * N3i, 0,
                                 st));
      BT_TRY(bt_gemm_at_tma_ex(W2, N2o * N1o, N3i * R * N2o * N1o, S1K, N3o, ys, N2o * N1o,
                               N3o * N2o * N1o, N2o * N1o, N3o, N3i * R, ns, 1, st));
    }
    if (!fell_back) return BT_OK;
  }
  for (int64_t s0 = 0; s0 < nrhs; s0 += mp.chunk) {
    const int64_t ns = std::min(mp.chunk, nrhs - s0);
    const double* xs = x + s0 * N3i * N2i * N1i;
    double* ys = y + s0 * N3o * N2o * N1o;
    // U[(s,a3,a2)][(r,i1)] = sum_a1 x[(s,a3,a2)][a1] S3[r][i1][a1]
    BtGemmArgs g1{};
    g1.M = ns * N3i * N2i;
    g1.N = R * N1o;
    g1.Kin = N1i;
    g1.Kout = 1;
    g1.A = BtOperand{xs, N1i, 0, 1, 0};
    g1.B = BtOperand{s3, N1i, 0, 1, 0};
    g1.C = U;
    g1.sCm = R * N1o;
    g1.sCn = 1;
    g1.alpha = 1.0;
    g1.ws = gws;
    BT_TRY(bt_gemm_run(g1, 1, st, 0, gws_n));
    // W2[(s,a3)][r][i2][i1] = sum_a2 S2[r][i2][a2] U[(s,a3)][a2][r][i1]
    for (int64_t r = 0; r < R; ++r) {
      BtGemmArgs g2{};
      g2.M = N2o;
      g2.N = N1o;
      g2.Kin = N2i;
      g2.Kout = 1;
      g2.A = BtOperand{s2 + r * N2o * N2i, N2i, 0, 1, 0};
      g2.B = BtOperand{U + r * N1o, 1, 0, R * N1o, N2i * R * N1o};
      g2.C = W2 + r * N2o * N1o;
      g2.sCm = N1o;
      g2.sCn = 1;
      g2.sCb = R * N2o * N1o;
      g2.alpha = 1.0;
      g2.ws = gws;
      const int64_t batch = ns * N3i;
      for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        BtGemmArgs c = g2;
        c.B.ptr = g2.B.ptr + b0 * g2.B.s_b;
        c.C = g2.C + b0 * g2.sCb;
        BT_TRY(bt_gemm_run(c, std::min<int64_t>(65535, batch - b0), st, 0, gws_n));
      }
    }
    // y[s][i3][(i2,i1)] = sum_{r,a3} S1[r][i3][a3] W2[s][a3][r][(i2,i1)]
    BtGemmArgs g3{};
    g3.M = N3o;
    g3.N = N2o * N1o;
    g3.Kin = N3i;
    g3.Kout = R;
    g3.A = BtOperand{s1, N3i, N3o * N3i, 1, 0};
    g3.B = BtOperand{W2, 1, N2o * N1o, R * N2o * N1o, N3i * R * N2o * N1o};
    g3.C = ys;
    g3.sCm = N2o * N1o;
    g3.sCn = 1;
    g3.sCb = N3o * N2o * N1o;
    g3.alpha = 1.0;
    g3.ws = gws;
    BT_TRY(bt_gemm_run(g3, ns, st, 0, gws_n));
  }
  return BT_OK;
}
