// Strided-batched FP64 DMMA GEMM (exported as bt_gemm_f64) + the shared
// split-K reduction.  Replaces the dgemm calls of the reference's
// mode products and Grams (tensor.py:90 `u @ unfold(t, mode)`,
// decomp.py:227 SVD-of-unfolding -> Gram SYRK) without unfolding copies.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "gemm.cuh"

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------

static thread_local char g_last_error[1024] = "";

void bt_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

extern "C" const char* bt_last_error(void) { return g_last_error; }

extern "C" int bt_version(void) { return BT_ABI_VERSION; }

static std::atomic<long long> g_launches{0};
void bt_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" int64_t bt_launch_count(void) { return g_launches.load(); }

int bt_num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// Stream-ordered scratch (cudaMallocAsync) stays in the device's default pool
// between calls: with the default release threshold of 0 every synchronise
// hands the freed block back to the driver, and the next cudaMallocAsync
// (~210 us) and the synchronise after cudaFreeAsync (~200 us) pay for it --
// 0.4 ms of a 1.3 ms C1 cp_als call.  Called once per device by the paths
// that take scratch that way (the small CP-ALS paths); torch's own caching
// allocator is not involved.
void bt_keep_async_pool() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool = nullptr;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess && pool != nullptr) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done[dev] = true;
}

// ---------------------------------------------------------------------------
// reduction
// ---------------------------------------------------------------------------

__global__ void bt_gemm_reduce_kernel(BtGemmArgs g, int64_t bm, int64_t bn) {
  const int64_t total = g.M * g.N;
  const int64_t batch = blockIdx.y;
  const double* wsb = g.ws + batch * g.splits * total;
  double* Cb = g.C + batch * g.sCb;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = idx / g.N, n = idx % g.N;
    int64_t src = idx;
    if (g.symmetric && (m / bm < n / bn || (m / bm == n / bn && m < n))) src = n * g.N + m;
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < g.splits; ++k) s += wsb[k * total + src];
    double* c = Cb + m * g.sCm + n * g.sCn;
    const double v = g.alpha * s;
    *c = (g.beta == 0.0) ? v : v + g.beta * (*c);
  }
}

// ---------------------------------------------------------------------------
// launch
// ---------------------------------------------------------------------------

// Split-K count for grids smaller than one wave (2 CTAs per SM for every
// config): the smallest split whose CTA count fills its last wave best --
// e.g. the C3 mode-1 SYRK (36 lower tiles) takes 8 splits = 288 CTAs (97% of
// the 296 slots), where "ceil(296 / 36) = 9" would spill 28 CTAs into a
// second, nearly empty wave.
static int bt_pick_splits(int64_t tiles, int64_t batch, int64_t KT) {
  const int64_t slots = 2 * bt_num_sms();
  const int64_t have = tiles * batch;
  if (have >= slots || KT < 8) return 1;
  int best = 1;
  double best_eff = static_cast<double>(have) / static_cast<double>(slots);
  // up to one split per slot: a rank's C5 mode-3 GEMM at 8 GPUs is a single
  // 128x64 output tile over a 16.8M-long reduction (a cap of 64 splits ran
  // it on 64 of the 296 slots: 8.4 TF/s)
  const int64_t smax = std::min<int64_t>(slots, KT / 4);
  for (int64_t s = 2; s <= smax; ++s) {
    const int64_t n = have * s;
    const int64_t waves = (n + slots - 1) / slots;
    const double eff = static_cast<double>(n) / static_cast<double>(waves * slots);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = static_cast<int>(s);
    }
  }
  return best;
}

template <class Cfg>
static void bt_gemm_geometry(BtGemmArgs& g, int64_t batch, int want_splits) {
  g.tiles_m = bt_cdiv(g.M, Cfg::BM);
  g.tiles_n = bt_cdiv(g.N, Cfg::BN);
  const int64_t tiles = g.symmetric ? g.tiles_m * (g.tiles_m + 1) / 2 : g.tiles_m * g.tiles_n;
  const int64_t KT = bt_cdiv(g.Kin, Cfg::BK) * g.Kout;
  g.splits = want_splits > 0 ? want_splits : bt_pick_splits(tiles, batch, KT);
  if (g.splits > KT) g.splits = static_cast<int>(std::max<int64_t>(KT, 1));
}

// resident CTAs per SM of the persistent kernel (cached per config)
template <class Cfg>
static int bt_persist_resident() {
  static int per_sm = -1;
  if (per_sm < 0) {
    cudaFuncSetAttribute(bt_gemm_persist_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM_BYTES);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bt_gemm_persist_kernel<Cfg>,
                                                      Cfg::THREADS, Cfg::SMEM_BYTES) != cudaSuccess)
      per_sm = 0;
  }
  return per_sm;
}

template <class Cfg>
int bt_gemm_launch(BtGemmArgs g, int64_t batch, cudaStream_t st, int want_splits) {
  bt_gemm_geometry<Cfg>(g, batch, want_splits);
  const int64_t tiles = g.symmetric ? g.tiles_m * (g.tiles_m + 1) / 2 : g.tiles_m * g.tiles_n;
  {
    // short reductions over many tiles: persistent CTAs with the stage
    // pipeline running across tile boundaries
    static const bool no_persist = getenv("BT_GEMM_PERSIST") && getenv("BT_GEMM_PERSIST")[0] == '0';
    const int64_t KT = bt_cdiv(g.Kin, Cfg::BK) * g.Kout;
    const int resident = (!no_persist && !g.symmetric && g.splits == 1 && KT <= 16)
                             ? bt_persist_resident<Cfg>() : 0;
    const int64_t slots = static_cast<int64_t>(resident) * bt_num_sms();
    if (resident > 0 && tiles * batch >= 3 * slots) {
      bt_gemm_persist_kernel<Cfg><<<static_cast<unsigned>(slots), Cfg::THREADS, Cfg::SMEM_BYTES,
                                    st>>>(g, batch);
      BT_LAUNCH_CHECK();
      return BT_OK;
    }
  }
  static bool attr_done = false;
  if (!attr_done) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(bt_gemm_kernel<Cfg>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES));
    attr_done = true;
  }
  BT_REQUIRE(tiles <= INT32_MAX && batch <= 65535 && g.splits <= 65535, BT_E_SHAPE,
             "gemm grid too large (tiles %lld batch %lld)", (long long)tiles, (long long)batch);
  dim3 grid(static_cast<unsigned>(tiles), g.splits, static_cast<unsigned>(batch));
  bt_gemm_kernel<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(g);
  BT_LAUNCH_CHECK();
  if (g.splits > 1 || g.symmetric) {
    const int64_t total = g.M * g.N;
    const int blocks = static_cast<int>(std::min<int64_t>(bt_cdiv(total, 256), 4096));
    bt_gemm_reduce_kernel<<<dim3(blocks, static_cast<unsigned>(batch)), 256, 0, st>>>(g, Cfg::BM,
                                                                                      Cfg::BN);
    BT_LAUNCH_CHECK();
  }
  return BT_OK;
}

// configurations ------------------------------------------------------------
// (tuned on B200 with tools/tune_gemm.py -- the alternatives tried are listed
// in profiles/r01_fp64_and_tuning.md; 2 CTAs per SM with 64x32 warp tiles win)
// wide: 128x64 CTA tile, 4 warps of 64x32, BK 16, 4 stages (~102 KB smem, 2 CTAs/SM)
template <bool AK, bool BKc, int V>
using CfgWide = GemmCfg<128, 64, 16, 2, 2, 4, AK, BKc, V>;
// narrow: 128x16 CTA tile for N <= 16 (Grams of R <= 16 factors, TTM r <= 16)
template <bool AK, bool BKc, int V>
using CfgNarrow = GemmCfg<128, 16, 16, 8, 1, 4, AK, BKc, V>;
// mid: 128x32 CTA tile for 16 < N <= 32 (TTM to r <= 32, e.g. C3's mode-2
// projection), 4 warps of 32x32
template <bool AK, bool BKc, int V>
using CfgMid = GemmCfg<128, 32, 16, 4, 1, 4, AK, BKc, V>;
// square: 128x128 for N > 64 and symmetric (SYRK) outputs, 8 warps of 64x32,
// 2 stages (~78 KB smem, 2 CTAs/SM)
template <bool AK, bool BKc, int V>
using CfgSquare = GemmCfg<128, 128, 16, 2, 4, 2, AK, BKc, V>;

enum BtTileClass { BT_TILE_WIDE = 0, BT_TILE_NARROW = 1, BT_TILE_SQUARE = 2, BT_TILE_MID = 3 };

template <template <bool, bool, int> class C>
static int bt_dispatch_layout(const BtGemmArgs& g, int64_t batch, cudaStream_t st, bool ak,
                              bool bk, int vec, int want_splits) {
  if (vec == 2) {
    if (ak && bk) return bt_gemm_launch<C<true, true, 2>>(g, batch, st, want_splits);
    if (ak && !bk) return bt_gemm_launch<C<true, false, 2>>(g, batch, st, want_splits);
    if (!ak && bk) return bt_gemm_launch<C<false, true, 2>>(g, batch, st, want_splits);
    return bt_gemm_launch<C<false, false, 2>>(g, batch, st, want_splits);
  }
  if (ak && bk) return bt_gemm_launch<C<true, true, 1>>(g, batch, st, want_splits);
  if (ak && !bk) return bt_gemm_launch<C<true, false, 1>>(g, batch, st, want_splits);
  if (!ak && bk) return bt_gemm_launch<C<false, true, 1>>(g, batch, st, want_splits);
  return bt_gemm_launch<C<false, false, 1>>(g, batch, st, want_splits);
}

static int bt_tile_class(const BtGemmArgs& g) {
  if (g.symmetric) return BT_TILE_SQUARE;
  static const char* force = getenv("BT_GEMM_FORCE");  // tuning switch (tools)
  if (force && force[0] == 'w' && g.N > 64) return BT_TILE_WIDE;
  if (g.N <= 16) return BT_TILE_NARROW;
  static const bool no_mid = getenv("BT_GEMM_NO_MID") != nullptr;  // A/B switch (tools)
  if (g.N <= 32 && !no_mid) return BT_TILE_MID;
  return g.N <= 64 ? BT_TILE_WIDE : BT_TILE_SQUARE;
}

static bool even_aligned(const double* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Normalise an argument set (swap to make N the small side, decide layouts
// and vector width) and run it.  Used by every internal GEMM-shaped call.
int bt_gemm_run(BtGemmArgs g, int64_t batch, cudaStream_t st, int want_splits, int64_t ws_elems) {
  BT_REQUIRE(g.M >= 0 && g.N >= 0 && g.Kin >= 0 && g.Kout >= 0 && batch >= 1, BT_E_SHAPE,
             "gemm: negative extent");
  if (g.M == 0 || g.N == 0) return BT_OK;
  if (g.Kin == 0 || g.Kout == 0) {
    // C = beta * C (alpha * empty sum)
    BtGemmArgs z = g;
    z.alpha = 0.0;
    z.Kin = 1;
    z.Kout = 1;
    g = z;
  }
  // make N the smaller extent (the CTA tile is tall); no swap with a B-scale
  if (!g.symmetric && g.bscale == nullptr && g.ascale == nullptr && g.N > g.M && g.N > 64) {
    BtGemmArgs s = g;
    s.M = g.N;
    s.N = g.M;
    s.A = g.B;
    s.B = g.A;
    s.sCm = g.sCn;
    s.sCn = g.sCm;
    g = s;
  }
  const bool ak = (g.A.s_ki == 1);
  const bool bk = (g.B.s_ki == 1);
  BT_REQUIRE(ak || g.A.s_mn == 1, BT_E_SHAPE, "gemm: A needs unit stride along m or k");
  BT_REQUIRE(bk || g.B.s_mn == 1, BT_E_SHAPE, "gemm: B needs unit stride along n or k");
  const int64_t a_row = ak ? g.A.s_mn : g.A.s_ki;
  const int64_t b_row = bk ? g.B.s_mn : g.B.s_ki;
  const bool v2 = even_aligned(g.A.ptr) && even_aligned(g.B.ptr) && (a_row % 2 == 0) &&
                  (b_row % 2 == 0) && (g.A.s_ko % 2 == 0) && (g.B.s_ko % 2 == 0) &&
                  (g.A.s_b % 2 == 0) && (g.B.s_b % 2 == 0);
  const int vec = v2 ? 2 : 1;
  int cls = bt_tile_class(g);
  // workspace check (computed with the same geometry the launcher will use)
  BtGemmArgs probe = g;
  if (cls == BT_TILE_SQUARE)
    bt_gemm_geometry<CfgSquare<true, true, 1>>(probe, batch, want_splits);
  else if (cls == BT_TILE_NARROW)
    bt_gemm_geometry<CfgNarrow<true, true, 1>>(probe, batch, want_splits);
  else if (cls == BT_TILE_MID)
    bt_gemm_geometry<CfgMid<true, true, 1>>(probe, batch, want_splits);
  else
    bt_gemm_geometry<CfgWide<true, true, 1>>(probe, batch, want_splits);
  const int64_t need = (probe.splits > 1 || g.symmetric) ? batch * probe.splits * g.M * g.N : 0;
  if (need > ws_elems) {
    BT_REQUIRE(!g.symmetric && ws_elems >= 0, BT_E_VALUE,
               "gemm: workspace too small (%lld < %lld doubles)", (long long)ws_elems,
               (long long)need);
    want_splits = 1;
  } else if (want_splits <= 0) {
    want_splits = probe.splits;
  }
  if (cls == BT_TILE_SQUARE)
    return bt_dispatch_layout<CfgSquare>(g, batch, st, ak, bk, vec, want_splits);
  if (cls == BT_TILE_NARROW)
    return bt_dispatch_layout<CfgNarrow>(g, batch, st, ak, bk, vec, want_splits);
  if (cls == BT_TILE_MID)
    return bt_dispatch_layout<CfgMid>(g, batch, st, ak, bk, vec, want_splits);
  return bt_dispatch_layout<CfgWide>(g, batch, st, ak, bk, vec, want_splits);
}

int64_t bt_gemm_ws_elems(BtGemmArgs g, int64_t batch) {
  if (!g.symmetric && g.bscale == nullptr && g.ascale == nullptr && g.N > g.M && g.N > 64)
    std::swap(g.M, g.N);
  int cls = bt_tile_class(g);
  if (cls == BT_TILE_SQUARE)
    bt_gemm_geometry<CfgSquare<true, true, 1>>(g, batch, 0);
  else if (cls == BT_TILE_NARROW)
    bt_gemm_geometry<CfgNarrow<true, true, 1>>(g, batch, 0);
  else if (cls == BT_TILE_MID)
    bt_gemm_geometry<CfgMid<true, true, 1>>(g, batch, 0);
  else
    bt_gemm_geometry<CfgWide<true, true, 1>>(g, batch, 0);
  return (g.splits > 1 || g.symmetric) ? batch * g.splits * g.M * g.N : 0;
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------

static BtGemmArgs bt_make_args(const bt_gemm_desc* d) {
  BtGemmArgs g;
  memset(&g, 0, sizeof(g));
  g.M = d->M;
  g.N = d->N;
  g.Kin = d->Kin;
  g.Kout = d->Kout;
  g.A = BtOperand{d->A, d->sAm, d->sAko, d->sAki, d->sAb};
  g.B = BtOperand{d->B, d->sBn, d->sBko, d->sBki, d->sBb};
  g.bscale = d->bscale;
  g.s_scale_ko = d->s_scale_ko;
  g.s_scale_b = d->s_scale_b;
  g.ascale = d->ascale;
  g.s_ascale_ko = d->s_ascale_ko;
  g.s_ascale_b = d->s_ascale_b;
  g.C = d->C;
  g.sCm = d->sCm;
  g.sCn = d->sCn;
  g.sCb = d->sCb;
  g.alpha = d->alpha;
  g.beta = d->beta;
  g.symmetric = d->symmetric;
  return g;
}

extern "C" int64_t bt_gemm_f64_ws_bytes(const bt_gemm_desc* d) {
  return bt_gemm_ws_elems(bt_make_args(d), d->batch < 1 ? 1 : d->batch) * 8;
}

extern "C" int bt_gemm_f64(const bt_gemm_desc* d, double* ws, int64_t ws_bytes, void* stream) {
  BT_NVTX("bt_gemm_f64");
  BT_REQUIRE(d != nullptr, BT_E_VALUE, "gemm: null descriptor");
  BT_REQUIRE(!d->symmetric || d->M == d->N, BT_E_SHAPE, "gemm: symmetric output must be square");
  BtGemmArgs g = bt_make_args(d);
  g.ws = ws;
  return bt_gemm_run(g, d->batch < 1 ? 1 : d->batch, bt_stream(stream), d->splits,
                     ws ? ws_bytes / 8 : 0);
}
