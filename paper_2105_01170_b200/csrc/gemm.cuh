// FP64 DMMA tile-GEMM engine shared by every GEMM-shaped kernel of the hot
// path (MTTKRP, Gram/SYRK, TTM, explicit CP fit, BLR/Kron matvecs).
//
//   C[b][m][n] = alpha * sum_{ko,ki} A(b,m,ko,ki) * B(b,ko,ki,n) [* scale(ko,n)]
//                + beta * C[b][m][n]
//
// with the reduction index split as k = (ko, ki) so that unfoldings of a
// C-order tensor are addressed in place (no unfold copies, unlike the
// reference's tensor.py:52 moveaxis+reshape(order="F")).  A is either
// M-contiguous (sAm == 1) or K-contiguous (sAki == 1); likewise B is
// N-contiguous or K-contiguous.  Tiles are staged global->shared with
// multi-stage cp.async (zero-filled at the edges) into padded layouts whose
// 8x4 fragment reads are bank-conflict free, and multiplied with
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, the FP64 tensor-core path).
#pragma once

#include "bt_common.cuh"

struct BtOperand {
  const double* ptr;
  int64_t s_mn;  // stride along m (A) or n (B)
  int64_t s_ko;  // stride along the outer reduction index
  int64_t s_ki;  // stride along the inner reduction index
  int64_t s_b;   // batch stride
};

struct BtGemmArgs {
  int64_t M, N, Kin, Kout;
  BtOperand A, B;
  const double* bscale;  // optional per-(ko, n) multiplier of B (Khatri-Rao on the fly)
  int64_t s_scale_ko;
  int64_t s_scale_b;
  const double* ascale;  // optional per-(ko, ki) multiplier of A (diagonal in the reduction)
  int64_t s_ascale_ko;
  int64_t s_ascale_b;
  double* C;
  int64_t sCm, sCn, sCb;
  double alpha, beta;
  int splits;      // split-K factor; >1 or symmetric => partials in ws
  double* ws;      // [batch][splits][M][N]
  int symmetric;   // M == N, only lower tiles computed, result mirrored
  int64_t tiles_m, tiles_n;
};

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, bool AK_, bool BK_CONTIG_,
          int VEC_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr bool A_KCONTIG = AK_, B_KCONTIG = BK_CONTIG_;
  static constexpr int VEC = VEC_;
  static constexpr int THREADS = WM * WN * 32;
  static constexpr int TM = BM / WM, TN = BN / WN;
  static constexpr int FM = TM / 8, FN = TN / 8;
  static constexpr int LDA = A_KCONTIG ? bt_ld(BK) : bt_ld(BM);
  static constexpr int ROWS_A = A_KCONTIG ? BM : BK;
  static constexpr int LDB = B_KCONTIG ? bt_ld(BK) : bt_ld(BN);
  static constexpr int ROWS_B = B_KCONTIG ? BN : BK;
  static constexpr int A_STAGE = ROWS_A * LDA;
  static constexpr int B_STAGE = ROWS_B * LDB;
  static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
  static_assert(TM % 8 == 0 && TN % 8 == 0, "warp tile must be a multiple of 8x8");
  static_assert(BK % 4 == 0, "BK must be a multiple of 4");
};

// cp.async loader of one operand tile: `ROWS` x `COLS` smem tile whose
// contiguous global direction runs along `COLS`.  Per-thread chunk
// coordinates are computed once per CTA; each stage only adds the stage's
// base pointer and re-evaluates the edge predicates.
template <int ROWS, int COLS, int LD, int VEC, int THREADS>
struct BtTileLoader {
  static constexpr int CHUNKS = COLS / VEC;
  static constexpr int TOTAL = ROWS * CHUNKS;
  static constexpr int ITERS = (TOTAL + THREADS - 1) / THREADS;
  static_assert(COLS % VEC == 0, "tile width must be a multiple of the vector width");
  int r_[ITERS];
  int c_[ITERS];
  int64_t goff_[ITERS];

  __device__ __forceinline__ void init(int64_t row_stride) {
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int idx = threadIdx.x + it * THREADS;
      r_[it] = idx / CHUNKS;
      c_[it] = (idx % CHUNKS) * VEC;
      goff_[it] = static_cast<int64_t>(r_[it]) * row_stride + c_[it];
    }
  }

  // base already points at global (row0, col0); rows_left/cols_left are the
  // remaining valid extents from there.
  __device__ __forceinline__ void issue(double* dst, const double* base, int64_t rows_left,
                                        int64_t cols_left, const double* safe) const {
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      if (TOTAL % THREADS != 0 && threadIdx.x + it * THREADS >= TOTAL) break;
      int64_t valid = (r_[it] < rows_left) ? (cols_left - c_[it]) : 0;
      valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
      const double* src = valid > 0 ? base + goff_[it] : safe;
      double* d = dst + r_[it] * LD + c_[it];
      if (VEC == 2)
        cp_async16(d, src, static_cast<int>(valid * 8));
      else
        cp_async8(d, src, static_cast<int>(valid * 8));
    }
  }
};

// The main loop over k-tiles [kt0, kt1) of one (m0, n0) output tile.
// k-tile coordinates (ko, ki) advance incrementally (no divisions in the
// loop); fragments are double-buffered in registers so the smem reads of
// step kk+4 overlap the DMMAs of step kk.
template <class Cfg>
__device__ __forceinline__ void bt_gemm_mainloop(const BtGemmArgs& g, int64_t batch, int64_t m0,
                                                 int64_t n0, int64_t kt0, int64_t kt1,
                                                 double (&acc)[Cfg::FM][Cfg::FN][2],
                                                 double* smem) {
  double* As = smem;
  double* Bs = smem + Cfg::STAGES * Cfg::A_STAGE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WM) * Cfg::TM;
  const int wn0 = (warp / Cfg::WM) * Cfg::TN;
  const int64_t ktPerKo = (g.Kin + Cfg::BK - 1) / Cfg::BK;
  const double* Ab = g.A.ptr + batch * g.A.s_b;
  const double* Bb = g.B.ptr + batch * g.B.s_b;
  constexpr int KSTEPS = Cfg::BK / 4;

  // A: K-contig -> rows m (stride s_mn), cols ki; M-contig -> rows ki (stride s_ki), cols m
  BtTileLoader<Cfg::ROWS_A, (Cfg::A_KCONTIG ? Cfg::BK : Cfg::BM), Cfg::LDA, Cfg::VEC, Cfg::THREADS>
      la;
  BtTileLoader<Cfg::ROWS_B, (Cfg::B_KCONTIG ? Cfg::BK : Cfg::BN), Cfg::LDB, Cfg::VEC, Cfg::THREADS>
      lb;
  la.init(Cfg::A_KCONTIG ? g.A.s_mn : g.A.s_ki);
  lb.init(Cfg::B_KCONTIG ? g.B.s_mn : g.B.s_ki);
  const double* a_tile = Ab + (Cfg::A_KCONTIG ? m0 * g.A.s_mn : m0);
  const double* b_tile = Bb + (Cfg::B_KCONTIG ? n0 * g.B.s_mn : n0);
  const int64_t m_left = g.M - m0, n_left = g.N - n0;

#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // load-side k-tile cursor (runs STAGES-1 tiles ahead of the compute side)
  int64_t l_ko = kt0 / ktPerKo;
  int64_t l_ki = kt0 - l_ko * ktPerKo;
  int64_t c_ko = l_ko, c_ki = l_ki;  // compute-side cursor
  auto load_stage = [&](int stage) {
    const int64_t ki0 = l_ki * Cfg::BK;
    const int64_t k_left = g.Kin - ki0;
    double* as = As + stage * Cfg::A_STAGE;
    double* bs = Bs + stage * Cfg::B_STAGE;
    if (Cfg::A_KCONTIG)
      la.issue(as, a_tile + l_ko * g.A.s_ko + ki0, m_left, k_left, g.A.ptr);
    else
      la.issue(as, a_tile + l_ko * g.A.s_ko + ki0 * g.A.s_ki, k_left, m_left, g.A.ptr);
    if (Cfg::B_KCONTIG)
      lb.issue(bs, b_tile + l_ko * g.B.s_ko + ki0, n_left, k_left, g.B.ptr);
    else
      lb.issue(bs, b_tile + l_ko * g.B.s_ko + ki0 * g.B.s_ki, k_left, n_left, g.B.ptr);
    if (++l_ki == ktPerKo) {
      l_ki = 0;
      ++l_ko;
    }
  };

#pragma unroll
  for (int s = 0; s < Cfg::STAGES - 1; ++s) {
    if (kt0 + s < kt1) load_stage(s);
    cp_async_commit();
  }

  int stage = 0;
  int next_stage = Cfg::STAGES - 1;
  double afr[2][Cfg::FM], bfr[2][Cfg::FN];
  for (int64_t kt = kt0; kt < kt1; ++kt) {
    cp_async_wait<Cfg::STAGES - 2>();
    __syncthreads();
    const double* as = As + stage * Cfg::A_STAGE;
    const double* bs = Bs + stage * Cfg::B_STAGE;
    double sc[Cfg::FN];
    if (g.bscale != nullptr) {
      const double* srow = g.bscale + batch * g.s_scale_b + c_ko * g.s_scale_ko;
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        const int64_t n = n0 + wn0 + j * 8 + gq;
        sc[j] = (n < g.N) ? __ldg(srow + n) : 0.0;
      }
    }
    const double* arow = nullptr;
    int64_t a_kleft = 0;
    if (g.ascale != nullptr) {
      const int64_t ki0 = c_ki * Cfg::BK;
      arow = g.ascale + batch * g.s_ascale_b + c_ko * g.s_ascale_ko + ki0;
      a_kleft = g.Kin - ki0;
    }
    auto load_frags = [&](int buf, int kk) {
      double asc = 1.0;
      if (g.ascale != nullptr) asc = (kk + tq < a_kleft) ? __ldg(arow + kk + tq) : 0.0;
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int m = wm0 + i * 8 + gq;
        afr[buf][i] = Cfg::A_KCONTIG ? as[m * Cfg::LDA + kk + tq] : as[(kk + tq) * Cfg::LDA + m];
        if (g.ascale != nullptr) afr[buf][i] *= asc;
      }
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        const int n = wn0 + j * 8 + gq;
        bfr[buf][j] = Cfg::B_KCONTIG ? bs[n * Cfg::LDB + kk + tq] : bs[(kk + tq) * Cfg::LDB + n];
        if (g.bscale != nullptr) bfr[buf][j] *= sc[j];
      }
    };
    load_frags(0, 0);
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      if (ks + 1 < KSTEPS) load_frags((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j)
          dmma884(acc[i][j][0], acc[i][j][1], afr[ks & 1][i], bfr[ks & 1][j]);
      if (ks == 0) {
        // refill the stage consumed in the previous iteration while this
        // stage's DMMAs drain
        if (kt + Cfg::STAGES - 1 < kt1) load_stage(next_stage);
        cp_async_commit();
      }
    }
    if (++c_ki == ktPerKo) {
      c_ki = 0;
      ++c_ko;
    }
    stage = (stage + 1 == Cfg::STAGES) ? 0 : stage + 1;
    next_stage = (next_stage + 1 == Cfg::STAGES) ? 0 : next_stage + 1;
  }
  cp_async_wait<0>();
}

// Map a linear tile index to (tm, tn) -- lower triangle when symmetric.
__device__ __forceinline__ void bt_tile_coords(const BtGemmArgs& g, int64_t lin, int64_t& tm,
                                               int64_t& tn) {
  if (!g.symmetric) {
    tm = lin % g.tiles_m;
    tn = lin / g.tiles_m;
    return;
  }
  // lin enumerates (tm, tn) with tn <= tm: row tm holds tm+1 tiles
  int64_t r = static_cast<int64_t>((sqrt(8.0 * static_cast<double>(lin) + 1.0) - 1.0) * 0.5);
  while ((r + 1) * (r + 2) / 2 <= lin) ++r;
  while (r * (r + 1) / 2 > lin) --r;
  tm = r;
  tn = lin - r * (r + 1) / 2;
}

// Fast epilogue for an interior tile of a row-major C (sCn == 1, beta == 0,
// 16-byte aligned rows): row pointers formed once per fragment row, the two
// accumulators of a lane stored as one 16-byte st.global -- no per-element
// bounds checks or 64-bit address products (the generic path costs ~8
// integer instructions per element, a quarter of a K = 128 tile's issue).
// Returns false when the tile needs the generic path.
template <class Cfg>
__device__ __forceinline__ bool bt_store_tile_fast(const BtGemmArgs& g, double* Cb, int64_t m0,
                                                   int64_t n0, int wm0, int wn0, int gq, int tq,
                                                   double (&acc)[Cfg::FM][Cfg::FN][2]) {
  if (!(g.sCn == 1 && g.beta == 0.0 && (g.sCm & 1) == 0 && m0 + Cfg::BM <= g.M &&
        n0 + Cfg::BN <= g.N && (reinterpret_cast<uintptr_t>(Cb) & 15u) == 0))
    return false;
  double* base = Cb + (m0 + wm0 + gq) * g.sCm + (n0 + wn0 + 2 * tq);
  const int64_t row8 = 8 * g.sCm;
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i) {
    double* row = base + i * row8;
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
      *reinterpret_cast<double2*>(row + j * 8) =
          make_double2(g.alpha * acc[i][j][0], g.alpha * acc[i][j][1]);
  }
  return true;
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS) bt_gemm_kernel(BtGemmArgs g) {
  extern __shared__ __align__(16) double smem_dyn[];
  int64_t tm, tn;
  bt_tile_coords(g, blockIdx.x, tm, tn);
  const int64_t m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;
  const int64_t batch = blockIdx.z;
  const int64_t ktPerKo = (g.Kin + Cfg::BK - 1) / Cfg::BK;
  const int64_t KT = ktPerKo * g.Kout;
  const int64_t split = blockIdx.y;
  const int64_t kt0 = KT * split / g.splits, kt1 = KT * (split + 1) / g.splits;
  double acc[Cfg::FM][Cfg::FN][2];
  bt_gemm_mainloop<Cfg>(g, batch, m0, n0, kt0, kt1, acc, smem_dyn);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WM) * Cfg::TM;
  const int wn0 = (warp / Cfg::WM) * Cfg::TN;
  const bool direct = (g.splits == 1) && !g.symmetric;
  double* wsb = g.ws + (batch * g.splits + split) * g.M * g.N;
  double* Cb = g.C + batch * g.sCb;
  if (direct && bt_store_tile_fast<Cfg>(g, Cb, m0, n0, wm0, wn0, gq, tq, acc)) return;
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i) {
    const int64_t m = m0 + wm0 + i * 8 + gq;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t n = n0 + wn0 + j * 8 + 2 * tq + h;
        if (n >= g.N) continue;
        if (direct) {
          double* c = Cb + m * g.sCm + n * g.sCn;
          const double v = g.alpha * acc[i][j][h];
          *c = (g.beta == 0.0) ? v : v + g.beta * (*c);
        } else {
          wsb[m * g.N + n] = acc[i][j][h];
        }
      }
    }
  }
}

// Persistent variant for short reductions (few k-tiles per output tile, many
// tiles -- the 128-long mode products of the multilevel matvec, batched small
// GEMMs): each CTA walks its tiles t = blockIdx.x, += gridDim.x as ONE stream
// of (tile, k-tile) steps, so the cp.async stages of the next tile are in
// flight while the current tile finishes and stores its accumulators (the
// one-tile-per-CTA kernel drains and refills its pipeline at every tile).
// Non-symmetric, no split-K; alpha/beta and the operand scales as above.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS) bt_gemm_persist_kernel(BtGemmArgs g,
                                                                       int64_t batches) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* As = smem_dyn;
  double* Bs = smem_dyn + Cfg::STAGES * Cfg::A_STAGE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm0 = (warp % Cfg::WM) * Cfg::TM;
  const int wn0 = (warp / Cfg::WM) * Cfg::TN;
  const int64_t ktPerKo = (g.Kin + Cfg::BK - 1) / Cfg::BK;
  const int64_t KT = ktPerKo * g.Kout;
  const int64_t per_batch = g.tiles_m * g.tiles_n;
  const int64_t total_tiles = per_batch * batches;
  const int64_t my_tiles =
      blockIdx.x < total_tiles ? (total_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t steps = my_tiles * KT;
  constexpr int KSTEPS = Cfg::BK / 4;

  BtTileLoader<Cfg::ROWS_A, (Cfg::A_KCONTIG ? Cfg::BK : Cfg::BM), Cfg::LDA, Cfg::VEC, Cfg::THREADS>
      la;
  BtTileLoader<Cfg::ROWS_B, (Cfg::B_KCONTIG ? Cfg::BK : Cfg::BN), Cfg::LDB, Cfg::VEC, Cfg::THREADS>
      lb;
  la.init(Cfg::A_KCONTIG ? g.A.s_mn : g.A.s_ki);
  lb.init(Cfg::B_KCONTIG ? g.B.s_mn : g.B.s_ki);

  auto tile_of = [&](int64_t local, int64_t& b, int64_t& m0, int64_t& n0) {
    const int64_t t = blockIdx.x + local * gridDim.x;
    b = t / per_batch;
    const int64_t rem = t - b * per_batch;
    const int64_t tn = rem / g.tiles_m;
    m0 = (rem - tn * g.tiles_m) * Cfg::BM;
    n0 = tn * Cfg::BN;
  };

  // load-side cursor
  int64_t l_tile = 0, l_ko = 0, l_ki = 0;
  int64_t l_b = 0, l_m0 = 0, l_n0 = 0;
  if (my_tiles > 0) tile_of(0, l_b, l_m0, l_n0);
  auto load_stage = [&](int stage) {
    const double* Ab = g.A.ptr + l_b * g.A.s_b;
    const double* Bb = g.B.ptr + l_b * g.B.s_b;
    const double* a_tile = Ab + (Cfg::A_KCONTIG ? l_m0 * g.A.s_mn : l_m0);
    const double* b_tile = Bb + (Cfg::B_KCONTIG ? l_n0 * g.B.s_mn : l_n0);
    const int64_t ki0 = l_ki * Cfg::BK;
    const int64_t k_left = g.Kin - ki0;
    double* as = As + stage * Cfg::A_STAGE;
    double* bs = Bs + stage * Cfg::B_STAGE;
    if (Cfg::A_KCONTIG)
      la.issue(as, a_tile + l_ko * g.A.s_ko + ki0, g.M - l_m0, k_left, g.A.ptr);
    else
      la.issue(as, a_tile + l_ko * g.A.s_ko + ki0 * g.A.s_ki, k_left, g.M - l_m0, g.A.ptr);
    if (Cfg::B_KCONTIG)
      lb.issue(bs, b_tile + l_ko * g.B.s_ko + ki0, g.N - l_n0, k_left, g.B.ptr);
    else
      lb.issue(bs, b_tile + l_ko * g.B.s_ko + ki0 * g.B.s_ki, k_left, g.N - l_n0, g.B.ptr);
    if (++l_ki == ktPerKo) {
      l_ki = 0;
      if (++l_ko == g.Kout) {
        l_ko = 0;
        if (++l_tile < my_tiles) tile_of(l_tile, l_b, l_m0, l_n0);
      }
    }
  };

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < Cfg::STAGES - 1; ++s) {
    if (s < steps) load_stage(s);
    cp_async_commit();
  }
  // compute-side cursor
  int64_t c_tile = 0, c_ko = 0, c_ki = 0;
  int64_t c_b = 0, c_m0 = 0, c_n0 = 0;
  if (my_tiles > 0) tile_of(0, c_b, c_m0, c_n0);
  int stage = 0;
  int next_stage = Cfg::STAGES - 1;
  double afr[2][Cfg::FM], bfr[2][Cfg::FN];
  for (int64_t st = 0; st < steps; ++st) {
    cp_async_wait<Cfg::STAGES - 2>();
    __syncthreads();
    const double* as = As + stage * Cfg::A_STAGE;
    const double* bs = Bs + stage * Cfg::B_STAGE;
    double sc[Cfg::FN];
    if (g.bscale != nullptr) {
      const double* srow = g.bscale + c_b * g.s_scale_b + c_ko * g.s_scale_ko;
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        const int64_t n = c_n0 + wn0 + j * 8 + gq;
        sc[j] = (n < g.N) ? __ldg(srow + n) : 0.0;
      }
    }
    const double* arow = nullptr;
    int64_t a_kleft = 0;
    if (g.ascale != nullptr) {
      const int64_t ki0 = c_ki * Cfg::BK;
      arow = g.ascale + c_b * g.s_ascale_b + c_ko * g.s_ascale_ko + ki0;
      a_kleft = g.Kin - ki0;
    }
    auto load_frags = [&](int buf, int kk) {
      double asc = 1.0;
      if (g.ascale != nullptr) asc = (kk + tq < a_kleft) ? __ldg(arow + kk + tq) : 0.0;
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int m = wm0 + i * 8 + gq;
        afr[buf][i] = Cfg::A_KCONTIG ? as[m * Cfg::LDA + kk + tq] : as[(kk + tq) * Cfg::LDA + m];
        if (g.ascale != nullptr) afr[buf][i] *= asc;
      }
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        const int n = wn0 + j * 8 + gq;
        bfr[buf][j] = Cfg::B_KCONTIG ? bs[n * Cfg::LDB + kk + tq] : bs[(kk + tq) * Cfg::LDB + n];
        if (g.bscale != nullptr) bfr[buf][j] *= sc[j];
      }
    };
    load_frags(0, 0);
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      if (ks + 1 < KSTEPS) load_frags((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j)
          dmma884(acc[i][j][0], acc[i][j][1], afr[ks & 1][i], bfr[ks & 1][j]);
      if (ks == 0) {
        if (st + Cfg::STAGES - 1 < steps) load_stage(next_stage);
        cp_async_commit();
      }
    }
    stage = (stage + 1 == Cfg::STAGES) ? 0 : stage + 1;
    next_stage = (next_stage + 1 == Cfg::STAGES) ? 0 : next_stage + 1;
    if (++c_ki == ktPerKo) {
      c_ki = 0;
      if (++c_ko == g.Kout) {
        c_ko = 0;
        // tile done: store (the next tile's first stages are already in flight)
        double* Cb = g.C + c_b * g.sCb;
        if (bt_store_tile_fast<Cfg>(g, Cb, c_m0, c_n0, wm0, wn0, gq, tq, acc)) {
#pragma unroll
          for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
          if (++c_tile < my_tiles) tile_of(c_tile, c_b, c_m0, c_n0);
          continue;
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) {
          const int64_t m = c_m0 + wm0 + i * 8 + gq;
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int64_t n = c_n0 + wn0 + j * 8 + 2 * tq + h;
              if (m < g.M && n < g.N) {
                double* c = Cb + m * g.sCm + n * g.sCn;
                const double v = g.alpha * acc[i][j][h];
                *c = (g.beta == 0.0) ? v : v + g.beta * (*c);
              }
              acc[i][j][h] = 0.0;
            }
          }
        }
        if (++c_tile < my_tiles) tile_of(c_tile, c_b, c_m0, c_n0);
      }
    }
  }
  cp_async_wait<0>();
}

// Deterministic split-K reduction (fixed order over splits) + mirror for
// symmetric outputs + alpha/beta.
__global__ void bt_gemm_reduce_kernel(BtGemmArgs g, int64_t bm, int64_t bn);

// Host-side launcher: picks VEC, splits, tiles and launches one Cfg.
template <class Cfg>
int bt_gemm_launch(BtGemmArgs g, int64_t batch, cudaStream_t st, int want_splits);
