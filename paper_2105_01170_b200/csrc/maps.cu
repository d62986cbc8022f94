// K1 / K2: the isometric block gather T_E and its inverse M_E.
//
// Replaces blocks.py:395-449 (extract_blocks + mat_to_tensor: a Python loop
// over every grid cell with numpy slice compares) and blocks.py:363-381 /
// 452-462 (struct_expand / tensor_to_mat).  One CTA walks whole grid cells
// (grid-stride over cells), so the class id, representative location and
// weight are CTA-uniform and the inner loop is a pure vectorised stream:
//   gather : read every element of A once (HBM, evict-first), read the
//            class representative (L2, evict-last), compare, write the
//            weighted representative once into t.
//   scatter: read t (L2-resident slices), write every element of A once.
// Values are bit-identical to the reference: sqrt(eta) * a in the gather,
// t / sqrt(eta) in the scatter (both IEEE correctly rounded).
//
// Verification mirrors the reference exactly, including numpy's NaN
// propagation (np.max of a NaN-containing |diff| is NaN and `NaN > tol` is
// False, so such a cell passes): per cell we record "some |d| > tol" and
// "some d is NaN"; the cell is bad iff the first holds and the second does
// not.  The first bad cell in the reference's scan order wins (integer
// atomicMin on its order rank -- deterministic).
#include <algorithm>
#include <cstdlib>

#include "bt_common.cuh"

namespace {

constexpr int MAP_THREADS = 256;

__device__ __forceinline__ void cell_flags(double d, double tol, int& exceed, int& nan) {
  exceed |= (d > tol);
  nan |= (d != d);
}

// U independent vector accesses per thread per iteration: with one access in
// flight per thread the SM holds only ~32 KB of outstanding requests, short
// of what HBM3e latency x bandwidth needs (~50 KB/SM); U = 4 covers it.
constexpr int MAP_UNROLL = 4;

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// tuning overrides: BT_GATHER_U / BT_SCATTER_U in {1, 2, 4, 8}
int gather_unroll() {
  static const int u = env_int("BT_GATHER_U", 2);
  return u;
}
int scatter_unroll() {
  static const int u = env_int("BT_SCATTER_U", MAP_UNROLL);
  return u;
}



// incremental (row, vcol) walk over an m x nv block without divisions
struct CellWalk {
  int rr, cv, nv, drow, dcol;
  __device__ CellWalk(int start, int nv_) : nv(nv_) {
    rr = start / nv;
    cv = start % nv;
    drow = MAP_THREADS / nv;
    dcol = MAP_THREADS % nv;
  }
  __device__ __forceinline__ void next() {
    rr += drow;
    cv += dcol;
    if (cv >= nv) {
      cv -= nv;
      ++rr;
    }
  }
};

template <int V>
__device__ __forceinline__ void flag_diff(const double* x, const double* y, double tol,
                                          int& exceed, int& nan) {
#pragma unroll
  for (int e = 0; e < V; ++e) cell_flags(fabs(x[e] - y[e]), tol, exceed, nan);
}

template <int V>
__device__ __forceinline__ void load_v(const double* p, double* out, bool keep) {
  if (V == 2) {
    const double2 v = keep ? ld_keep2(p) : ld_stream2(p);
    out[0] = v.x;
    out[1] = v.y;
  } else {
    out[0] = keep ? ld_keep(p) : ld_stream(p);
  }
}

template <int V, int U>
__global__ void __launch_bounds__(MAP_THREADS)
    gather_kernel(const double* __restrict__ a, int64_t lda, bt_pattern_dev pat, double tol,
                  int weighted, double* __restrict__ t, int* __restrict__ flags) {
  const int64_t cells = pat.ell * pat.q;
  const int64_t m = pat.m, n = pat.n, p = pat.p;
  const int nv = static_cast<int>(n / V);
  const int64_t per = m * nv;
  __shared__ int red[2][MAP_THREADS / 32];
  for (int64_t cell = blockIdx.x; cell < cells; cell += gridDim.x) {
    const int64_t ci = cell / pat.q, cj = cell % pat.q;
    const int k = pat.cell_class[cell];
    const double* blk = a + ci * m * lda + cj * n;
    int exceed = 0, nan = 0;
    CellWalk w(threadIdx.x, nv);
    if (k < 0) {
      const double zero[V] = {};
      for (int64_t idx = threadIdx.x; idx < per; idx += U * MAP_THREADS) {
        double x[U][V];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ok[u] = idx + u * MAP_THREADS < per;
          if (ok[u]) load_v<V>(blk + (int64_t)w.rr * lda + w.cv * V, x[u], false);
          w.next();
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ok[u]) flag_diff<V>(x[u], zero, tol, exceed, nan);
      }
    } else {
      const int64_t rc = pat.rep_cell[k];
      const bool is_rep = (rc == cell);
      const double* ref = a + (rc / pat.q) * m * lda + (rc % pat.q) * n;
      const double wt = weighted ? sqrt(static_cast<double>(pat.eta[k])) : 1.0;
      double* tk = t + k * n;  // t[row][k][col] = t[row * p * n + k * n + col]
      for (int64_t idx = threadIdx.x; idx < per; idx += U * MAP_THREADS) {
        double x[U][V];
        int rrs[U], cvs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          rrs[u] = (idx + u * MAP_THREADS < per) ? w.rr : -1;
          cvs[u] = w.cv;
          w.next();
        }
        if (is_rep) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (rrs[u] >= 0) load_v<V>(blk + (int64_t)rrs[u] * lda + cvs[u] * V, x[u], true);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (rrs[u] < 0) continue;
            double* dst = tk + (int64_t)rrs[u] * p * n + cvs[u] * V;
            if (V == 2) {
              *reinterpret_cast<double2*>(dst) = make_double2(wt * x[u][0], wt * x[u][V - 1]);
            } else {
              dst[0] = wt * x[u][0];
            }
          }
        } else {
          double y[U][V];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (rrs[u] < 0) continue;
            const int64_t off = (int64_t)rrs[u] * lda + cvs[u] * V;
            load_v<V>(blk + off, x[u], false);
            load_v<V>(ref + off, y[u], true);
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (rrs[u] >= 0) flag_diff<V>(x[u], y[u], tol, exceed, nan);
        }
      }
    }
    exceed = __any_sync(0xffffffffu, exceed);
    nan = __any_sync(0xffffffffu, nan);
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = exceed;
      red[1][threadIdx.x >> 5] = nan;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int e = 0, nn = 0;
      for (int w2 = 0; w2 < MAP_THREADS / 32; ++w2) {
        e |= red[0][w2];
        nn |= red[1][w2];
      }
      flags[cell] = e | (nn << 1);
    }
    __syncthreads();
  }
}

// Split gather, check half: every non-representative cell against its class
// representative (uncovered cells against zero), U independent 16-byte loads
// in flight per operand per thread; representative cells are skipped (their
// flags are zero).  Same flag semantics as gather_kernel.
template <int V, int U>
__global__ void __launch_bounds__(MAP_THREADS)
    gather_check_kernel(const double* __restrict__ a, int64_t lda, bt_pattern_dev pat, double tol,
                        int* __restrict__ flags) {
  const int64_t cells = pat.ell * pat.q;
  const int64_t m = pat.m, n = pat.n;
  const int nv = static_cast<int>(n / V);
  const int64_t per = m * nv;
  __shared__ int red[2][MAP_THREADS / 32];
  for (int64_t cell = blockIdx.x; cell < cells; cell += gridDim.x) {
    const int k = pat.cell_class[cell];
    const int64_t rc = k >= 0 ? pat.rep_cell[k] : -1;
    if (rc == cell) {  // CTA-uniform
      if (threadIdx.x == 0) flags[cell] = 0;
      continue;
    }
    const double* blk = a + (cell / pat.q) * m * lda + (cell % pat.q) * n;
    const double* ref = k >= 0 ? a + (rc / pat.q) * m * lda + (rc % pat.q) * n : nullptr;
    int exceed = 0, nan = 0;
    CellWalk w(threadIdx.x, nv);
    for (int64_t idx = threadIdx.x; idx < per; idx += U * MAP_THREADS) {
      double x[U][V], y[U][V];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ok[u] = idx + u * MAP_THREADS < per;
        if (ok[u]) {
          const int64_t off = (int64_t)w.rr * lda + w.cv * V;
          load_v<V>(blk + off, x[u], false);
          if (ref) {
            load_v<V>(ref + off, y[u], true);
          } else {
#pragma unroll
            for (int e = 0; e < V; ++e) y[u][e] = 0.0;
          }
        }
        w.next();
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) flag_diff<V>(x[u], y[u], tol, exceed, nan);
    }
    exceed = __any_sync(0xffffffffu, exceed);
    nan = __any_sync(0xffffffffu, nan);
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = exceed;
      red[1][threadIdx.x >> 5] = nan;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int e = 0, nn = 0;
      for (int w2 = 0; w2 < MAP_THREADS / 32; ++w2) {
        e |= red[0][w2];
        nn |= red[1][w2];
      }
      flags[cell] = e | (nn << 1);
    }
    __syncthreads();
  }
}

// Split gather, tensor half: t[:, k, :] = w_k * (representative block of k).
template <int V>
__global__ void __launch_bounds__(MAP_THREADS)
    gather_rep_kernel(const double* __restrict__ a, int64_t lda, bt_pattern_dev pat, int weighted,
                      double* __restrict__ t) {
  const int64_t m = pat.m, n = pat.n, p = pat.p;
  const int64_t nv = n / V;
  const int64_t per = m * nv;
  const int64_t total = p * per;
  for (int64_t g = blockIdx.x * (int64_t)MAP_THREADS + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * MAP_THREADS) {
    const int64_t k = g / per, v = g - k * per;
    const int64_t r = v / nv, cv = v - r * nv;
    const int64_t rc = pat.rep_cell[k];
    const double wt = weighted ? sqrt(static_cast<double>(pat.eta[k])) : 1.0;
    const double* src = a + ((rc / pat.q) * m + r) * lda + (rc % pat.q) * n + cv * V;
    double* dst = t + r * p * n + k * n + cv * V;
    if (V == 2) {
      const double2 x = ld_stream2(src);
      *reinterpret_cast<double2*>(dst) = make_double2(wt * x.x, wt * x.y);
    } else {
      dst[0] = wt * ld_stream(src);
    }
  }
}

__global__ void gather_verdict(const int* __restrict__ flags, const int64_t* __restrict__ order,
                               int64_t cells, unsigned long long* __restrict__ first) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int f = flags[c];
    if ((f & 1) && !(f & 2)) atomicMin(first, static_cast<unsigned long long>(order[c]));
  }
}

// PH 0: every cell, a = t / sqrt(eta).  PH 1: class representative cells
// only.  PH 2: every other cell copies its class representative's block back
// out of A (L2-resident after PH 1) -- the same bits, no division in the
// 8.6 GB stream (measured 1.93 vs 2.03 ms on the 32768^2 stand-in; a
// row-major sweep of A was slower, 2.5 ms).
template <int V, int U, int PH>
__global__ void __launch_bounds__(MAP_THREADS)
    scatter_kernel(const double* __restrict__ t, int64_t t_sm, int64_t t_sp, int64_t t_sn,
                   bt_pattern_dev pat, double* __restrict__ a, int64_t lda) {
  const int64_t cells = (PH == 1) ? pat.p : pat.ell * pat.q;
  const int64_t m = pat.m, n = pat.n;
  const int nv = static_cast<int>(n / V);
  const int64_t per = m * nv;
  for (int64_t it = blockIdx.x; it < cells; it += gridDim.x) {
    const int64_t cell = (PH == 1) ? pat.rep_cell[it] : it;
    const int64_t ci = cell / pat.q, cj = cell % pat.q;
    const int k = (PH == 1) ? static_cast<int>(it) : pat.cell_class[cell];
    if (PH == 2 && k >= 0 && pat.rep_cell[k] == cell) continue;  // written by PH 1
    double* blk = a + ci * m * lda + cj * n;
    const double s = (k >= 0) ? sqrt(static_cast<double>(pat.eta[k])) : 1.0;
    const double* tk = t + (k >= 0 ? k : 0) * t_sp;
    const double* rep = nullptr;
    if (PH == 2 && k >= 0) {
      const int64_t rc = pat.rep_cell[k];
      rep = a + (rc / pat.q) * m * lda + (rc % pat.q) * n;
    }
    CellWalk w(threadIdx.x, nv);
    for (int64_t idx = threadIdx.x; idx < per; idx += U * MAP_THREADS) {
      double x[U][V];
      bool ok[U];
      int64_t off[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ok[u] = idx + u * MAP_THREADS < per;
        off[u] = (int64_t)w.rr * lda + w.cv * V;
        if (ok[u]) {
          if (k >= 0 && PH == 2) {
            load_v<V>(rep + off[u], x[u], true);
          } else if (k >= 0) {
            const double* src = tk + (int64_t)w.rr * t_sm + (int64_t)w.cv * V * t_sn;
            if (V == 2) {
              const double2 v = *reinterpret_cast<const double2*>(src);
              x[u][0] = v.x;
              x[u][V - 1] = v.y;
            } else {
              x[u][0] = src[0];
            }
          } else {
#pragma unroll
            for (int e = 0; e < V; ++e) x[u][e] = 0.0;
          }
        }
        w.next();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
        if (k >= 0 && PH != 2) {
#pragma unroll
          for (int e = 0; e < V; ++e) x[u][e] = x[u][e] / s;
        }
        if (V == 2) {
          st_stream2(blk + off[u], make_double2(x[u][0], x[u][V - 1]));
        } else {
          st_stream(blk + off[u], x[u][0]);
        }
      }
    }
  }
}

// Class-major second phase (needs class_ptr/class_cells): work item (k, c)
// holds chunk c of class k's representative block -- CHUNK vectors, VPT per
// thread -- in registers, read once from A (written by PH 1), and writes it
// into every other cell of the class.  The representative is read once per
// class instead of once per cell, so the write stream no longer evicts the
// 67 MB of representatives from L2 (ncu: 2.1 GB of DRAM re-reads in the
// cell-major pass on the 32768^2 stand-in).
template <int V, int VPT>
__global__ void __launch_bounds__(MAP_THREADS)
    scatter_class_kernel(bt_pattern_dev pat, double* __restrict__ a, int64_t lda, int64_t chunks) {
  constexpr int64_t CHUNK = (int64_t)MAP_THREADS * VPT;
  const int64_t n = pat.n;
  const int64_t nv = n / V;
  const int64_t per = pat.m * nv;
  for (int64_t item = blockIdx.x; item < pat.p * chunks; item += gridDim.x) {
    const int64_t k = item / chunks, c = item - k * chunks;
    const int64_t c0 = pat.class_ptr[k], c1 = pat.class_ptr[k + 1];
    if (c1 - c0 < 2) continue;  // only the representative itself
    const int64_t rc = pat.rep_cell[k];
    const double* rep = a + (rc / pat.q) * pat.m * lda + (rc % pat.q) * n;
    double x[VPT][V];
    int64_t off[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int64_t v = c * CHUNK + u * MAP_THREADS + threadIdx.x;
      off[u] = -1;
      if (v < per) {
        const int64_t r = v / nv, cv = v - r * nv;
        off[u] = r * lda + cv * V;
        load_v<V>(rep + off[u], x[u], false);
      }
    }
    for (int64_t e = c0; e < c1; ++e) {
      const int64_t cell = pat.class_cells[e];
      if (cell == rc) continue;
      double* blk = a + (cell / pat.q) * pat.m * lda + (cell % pat.q) * n;
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        if (off[u] < 0) continue;
        if (V == 2)
          st_stream2(blk + off[u], make_double2(x[u][0], x[u][V - 1]));
        else
          st_stream(blk + off[u], x[u][0]);
      }
    }
  }
}

// zero the uncovered cells (class -1) only
template <int V>
__global__ void __launch_bounds__(MAP_THREADS)
    zero_uncovered_kernel(bt_pattern_dev pat, double* __restrict__ a, int64_t lda) {
  const int64_t cells = pat.ell * pat.q;
  const int nv = static_cast<int>(pat.n / V);
  const int64_t per = pat.m * nv;
  for (int64_t cell = blockIdx.x; cell < cells; cell += gridDim.x) {
    if (pat.cell_class[cell] >= 0) continue;
    double* blk = a + (cell / pat.q) * pat.m * lda + (cell % pat.q) * pat.n;
    CellWalk w(threadIdx.x, nv);
    for (int64_t idx = threadIdx.x; idx < per; idx += MAP_THREADS) {
      if (V == 2)
        st_stream2(blk + (int64_t)w.rr * lda + w.cv * V, make_double2(0.0, 0.0));
      else
        st_stream(blk + (int64_t)w.rr * lda + w.cv, 0.0);
      w.next();
    }
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int grid_for(int64_t cells) {
  static const int mult = env_int("BT_MAP_GRID", 16);  // CTAs per SM (tuning override)
  return static_cast<int>(std::min<int64_t>(cells, static_cast<int64_t>(bt_num_sms()) * mult));
}

}  // namespace

extern "C" int64_t bt_gather_ws_bytes(const bt_pattern_dev* pat) {
  return pat->ell * pat->q * 4 + 16;
}

extern "C" int bt_gather_blocks_f64(const double* a, int64_t lda, const bt_pattern_dev* pat,
                                    double tol, int weighted, double* t, void* ws,
                                    int64_t* bad_order, void* stream) {
  BT_NVTX("bt_gather_blocks_f64");
  BT_REQUIRE(pat->m >= 1 && pat->n >= 1 && pat->ell >= 1 && pat->q >= 1, BT_E_SHAPE,
             "gather: pattern extents must be positive");
  BT_REQUIRE(lda >= pat->q * pat->n, BT_E_SHAPE, "gather: lda too small");
  BT_REQUIRE(pat->n <= (int64_t)1 << 30 && pat->m * pat->n < ((int64_t)1 << 40), BT_E_SHAPE,
             "gather: block too large");
  cudaStream_t st = bt_stream(stream);
  const int64_t cells = pat->ell * pat->q;
  int* flags = static_cast<int*>(ws);
  unsigned long long* first =
      reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + ((cells * 4 + 15) / 16) * 16);
  BT_CUDA_CHECK(cudaMemsetAsync(first, 0xff, 8, st));
  const bool v2 = (pat->n % 2 == 0) && (lda % 2 == 0) && aligned16(a) && aligned16(t) &&
                  ((pat->p * pat->n) % 2 == 0);
  const int gu = gather_unroll();
  const int split = env_int("BT_GATHER_SPLIT", 1);
  if (split) {
    // check pass (all cells but the representatives) + representative pass
    if (v2) {
      gather_check_kernel<2, 4><<<grid_for(cells), MAP_THREADS, 0, st>>>(a, lda, *pat, tol, flags);
      BT_LAUNCH_CHECK();
      if (pat->p > 0) {
        gather_rep_kernel<2><<<bt_num_sms() * 8, MAP_THREADS, 0, st>>>(a, lda, *pat, weighted, t);
        BT_LAUNCH_CHECK();
      }
    } else {
      gather_check_kernel<1, 4><<<grid_for(cells), MAP_THREADS, 0, st>>>(a, lda, *pat, tol, flags);
      BT_LAUNCH_CHECK();
      if (pat->p > 0) {
        gather_rep_kernel<1><<<bt_num_sms() * 8, MAP_THREADS, 0, st>>>(a, lda, *pat, weighted, t);
        BT_LAUNCH_CHECK();
      }
    }
  } else {
#define BT_GATHER(V_, U_) \
  gather_kernel<V_, U_><<<grid_for(cells), MAP_THREADS, 0, st>>>(a, lda, *pat, tol, weighted, t, flags)
  if (!v2)
    BT_GATHER(1, 2);
  else if (gu == 8)
    BT_GATHER(2, 8);
  else if (gu == 4)
    BT_GATHER(2, 4);
  else if (gu == 2)
    BT_GATHER(2, 2);
  else
    BT_GATHER(2, 1);
#undef BT_GATHER
  BT_LAUNCH_CHECK();
  }
  gather_verdict<<<static_cast<int>(std::min<int64_t>(bt_cdiv(cells, 256), 1024)), 256, 0, st>>>(
      flags, pat->cell_order, cells, first);
  BT_LAUNCH_CHECK();
  unsigned long long h = 0;
  BT_CUDA_CHECK(cudaMemcpyAsync(&h, first, 8, cudaMemcpyDeviceToHost, st));
  BT_CUDA_CHECK(cudaStreamSynchronize(st));
  if (h != ~0ull) {
    if (bad_order) *bad_order = static_cast<int64_t>(h);
    bt_set_error("pattern mismatch at scan rank %lld", (long long)h);
    return BT_E_PATTERN;
  }
  if (bad_order) *bad_order = -1;
  return BT_OK;
}

extern "C" int bt_scatter_blocks_f64(const double* t, int64_t t_sm, int64_t t_sp, int64_t t_sn,
                                     const bt_pattern_dev* pat, double* a, int64_t lda,
                                     void* stream) {
  BT_NVTX("bt_scatter_blocks_f64");
  BT_REQUIRE(pat->m >= 1 && pat->n >= 1 && pat->ell >= 1 && pat->q >= 1, BT_E_SHAPE,
             "scatter: pattern extents must be positive");
  BT_REQUIRE(lda >= pat->q * pat->n, BT_E_SHAPE, "scatter: lda too small");
  cudaStream_t st = bt_stream(stream);
  const int64_t cells = pat->ell * pat->q;
  const bool v2 = (pat->n % 2 == 0) && (lda % 2 == 0) && (t_sn == 1) && (t_sm % 2 == 0) &&
                  (t_sp % 2 == 0) && aligned16(a) && aligned16(t);
  const int su = scatter_unroll();
  // tuning: 0 one pass, 1 representatives + class-major copies, 2 cell-major copies
  const int two_phase = env_int("BT_SCATTER_PH", 1);
#define BT_SCATTER(V_, U_, PH_)                                                           \
  scatter_kernel<V_, U_, PH_><<<grid_for(PH_ == 1 ? pat->p : cells), MAP_THREADS, 0, st>>>( \
      t, t_sm, t_sp, t_sn, *pat, a, lda)
  if (two_phase == 1 && pat->p > 0 && pat->class_ptr && pat->class_cells) {
    // PH 1 (representatives, with the division), class-major copies, zeros
    constexpr int VPT = 8;
    const int64_t nvec = pat->m * (pat->n / (v2 ? 2 : 1));
    const int64_t chunks = bt_cdiv(nvec, (int64_t)MAP_THREADS * VPT);
    const int grid = static_cast<int>(
        std::min<int64_t>(pat->p * chunks, static_cast<int64_t>(bt_num_sms()) * 16));
    if (v2) {
      BT_SCATTER(2, 4, 1);
      BT_LAUNCH_CHECK();
      scatter_class_kernel<2, VPT><<<grid, MAP_THREADS, 0, st>>>(*pat, a, lda, chunks);
    } else {
      BT_SCATTER(1, 4, 1);
      BT_LAUNCH_CHECK();
      scatter_class_kernel<1, VPT><<<grid, MAP_THREADS, 0, st>>>(*pat, a, lda, chunks);
    }
    BT_LAUNCH_CHECK();
    if (pat->nnz < cells) {
      if (v2)
        zero_uncovered_kernel<2><<<grid_for(cells), MAP_THREADS, 0, st>>>(*pat, a, lda);
      else
        zero_uncovered_kernel<1><<<grid_for(cells), MAP_THREADS, 0, st>>>(*pat, a, lda);
      BT_LAUNCH_CHECK();
    }
    return BT_OK;
  }
  if (two_phase && pat->p > 0) {
    if (v2) {
      BT_SCATTER(2, 4, 1);
      BT_LAUNCH_CHECK();
      BT_SCATTER(2, 4, 2);
    } else {
      BT_SCATTER(1, 4, 1);
      BT_LAUNCH_CHECK();
      BT_SCATTER(1, 4, 2);
    }
  } else if (!v2) {
    BT_SCATTER(1, 4, 0);
  } else if (su == 2) {
    BT_SCATTER(2, 2, 0);
  } else {
    BT_SCATTER(2, 4, 0);
  }
#undef BT_SCATTER
  BT_LAUNCH_CHECK();
  return BT_OK;
}

// ---------------------------------------------------------------------------
// Representative blocks of detect_pattern (blocks.py:298-306 returns each
// class's first occurrence as a contiguous array): out[k] (m x n) = the
// block at cell cells[k] = i*q + j of a.  One launch for all classes, one
// CTA row per block row, 16-byte copies when the rows allow it.
// ---------------------------------------------------------------------------

__global__ void copy_cells_kernel(const double* __restrict__ a, int64_t lda,
                                  const int64_t* __restrict__ cells, int64_t p, int64_t q,
                                  int64_t m, int64_t n, double* __restrict__ out, int vec2) {
  const int64_t rows = p * m;
  for (int64_t rr = blockIdx.x; rr < rows; rr += gridDim.x) {
    const int64_t k = rr / m, r = rr - k * m;
    const int64_t c = cells[k];
    const int64_t i = c / q, j = c - i * q;
    const double* src = a + (i * m + r) * lda + j * n;
    double* dst = out + (k * m + r) * n;
    if (vec2) {
      const double2* s2 = reinterpret_cast<const double2*>(src);
      double2* d2 = reinterpret_cast<double2*>(dst);
      for (int64_t x = threadIdx.x; x < n / 2; x += blockDim.x) d2[x] = s2[x];
    } else {
      for (int64_t x = threadIdx.x; x < n; x += blockDim.x) dst[x] = src[x];
    }
  }
}

extern "C" int bt_copy_cells_f64(const double* a, int64_t lda, const int64_t* cells, int64_t p,
                                 int64_t q, int64_t m, int64_t n, double* out, void* stream) {
  BT_NVTX("bt_copy_cells_f64");
  BT_REQUIRE(p >= 0 && m >= 0 && n >= 0 && q >= 1, BT_E_SHAPE, "copy_cells: bad extents");
  if (p == 0 || m == 0 || n == 0) return BT_OK;
  const int vec2 = (n % 2 == 0) && (lda % 2 == 0) &&
                   (reinterpret_cast<uintptr_t>(a) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  const int threads = n >= 512 ? 256 : 128;
  const int64_t rows = p * m;
  copy_cells_kernel<<<static_cast<unsigned>(rows < 65535 ? rows : 65535), threads, 0,
                      bt_stream(stream)>>>(a, lda, cells, p, q, m, n, out, vec2);
  BT_LAUNCH_CHECK();
  return BT_OK;
}
