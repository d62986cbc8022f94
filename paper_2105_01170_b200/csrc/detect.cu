// Block-repeat detection (blocks.py:266-329 `detect_pattern`).
//
// The reference walks the ell x q block grid in Python, hashing each block's
// bytes (tol == 0) or scanning the class representatives (tol > 0).  Here
// one HBM pass computes, per grid cell, a 128-bit order-independent digest of
// the block's bytes (a sum of per-word multiply/xor-shift mixes and a sum of
// position-rotated words, both keyed by the word's position -- any reduction
// order gives the same bits) and the reference's
// skip predicate (`blk.any()` for tol == 0, `max|blk| <= tol` for tol > 0,
// with numpy's NaN semantics).  The host groups equal digests in row-major
// first-occurrence order; a second pass compares every cell with its class
// representative word for word (exact) or within tol, so a digest collision
// can never merge two different blocks.
#include <algorithm>

#include "bt_common.cuh"

namespace {

constexpr int DT = 256;
constexpr int DU = 4;  // independent loads in flight per thread

constexpr uint64_t kK1 = 0x9e3779b97f4a7c15ull, kK2 = 0xd1b54a32d192ed03ull;

template <int V>
__device__ __forceinline__ void load_vec(const double* p, double* out) {
  if (V == 2) {
    const double2 v = ld_stream2(p);
    out[0] = v.x;
    out[V - 1] = v.y;
  } else {
    out[0] = ld_stream(p);
  }
}

// acc += (a + ka) * (b + kb), 32 x 32 -> 64 bits with the 64-bit add: one
// IMAD.WIDE.U32 on the FMA pipe (NH hashing: a sum over positions of keyed
// word products; with keys that differ per position a changed word changes
// the sum unless its partner word + key is 0 mod 2^32)
__device__ __forceinline__ uint64_t nh(uint64_t acc, uint32_t a, uint32_t ka, uint32_t b,
                                       uint32_t kb) {
  return acc + static_cast<uint64_t>(a + ka) * static_cast<uint64_t>(b + kb);
}

// one access (V doubles) into the two sums; k1, k2: the access's keys
template <int V, bool EXACT>
__device__ __forceinline__ void digest_access(const double* x, uint64_t k1, uint64_t k2, double tol,
                                              uint64_t& a1, uint64_t& a2, uint32_t& any_bits,
                                              int& flag) {
  const uint32_t k1h = static_cast<uint32_t>(k1 >> 32), k1l = static_cast<uint32_t>(k1) ^ k1h;
  const uint32_t k2h = static_cast<uint32_t>(k2 >> 32), k2l = static_cast<uint32_t>(k2) ^ k2h;
  const uint64_t w0 = static_cast<uint64_t>(__double_as_longlong(x[0]));
  const uint32_t x0 = static_cast<uint32_t>(w0), x1 = static_cast<uint32_t>(w0 >> 32);
  if (V == 2) {
    const uint64_t w1 = static_cast<uint64_t>(__double_as_longlong(x[V - 1]));
    const uint32_t x2 = static_cast<uint32_t>(w1), x3 = static_cast<uint32_t>(w1 >> 32);
    a1 = nh(a1, x0, k1l, x1, k1h);
    a1 = nh(a1, x2, ~k1h, x3, ~k1l);
    a2 = nh(a2, x0, k2h, x3, k2l);
    a2 = nh(a2, x1, ~k2l, x2, ~k2h);
    if (EXACT) {
      any_bits |= ((x1 | x3) & 0x7fffffffu) | x0 | x2;  // not +0.0 / -0.0 (NaN counts, like np.any)
    } else {
      flag |= !(fabs(x[0]) <= tol);  // NaN or |x| > tol
      flag |= !(fabs(x[V - 1]) <= tol);
    }
  } else {
    a1 = nh(a1, x0, k1l, x1, k1h);
    a2 = nh(a2, x0, k2h, x1, k2l);
    if (EXACT)
      any_bits |= (x1 & 0x7fffffffu) | x0;
    else
      flag |= !(fabs(x[0]) <= tol);
  }
}

// per cell: h1, h2 (digest), nz (EXACT, i.e. tol == 0: any word not +-0.0;
// else max|x| > tol or NaN present).  V doubles per access; the two 64-bit
// keys of an access are linear in its position in the block (row-major), their
// high words are multiply-shift hashes of the position and the low words are
// xored with them.  Every sum is over positions, so any reduction order gives
// the same bits.  ~30 instructions per 16-byte access (the multiply/xor-shift
// + rotate digests it replaces took 87 and were ALU-pipe bound at 4.4 TB/s).
// DC0: DT is a multiple of the accesses per block row, so a thread keeps its
// column and walks rows.  32-bit walk indices (a block has < 2^31 accesses).
template <int V, bool EXACT, bool DC0>
__global__ void __launch_bounds__(DT, 4)
    block_digest_kernel(const double* __restrict__ a, int64_t lda, int64_t ell, int64_t q, int64_t m,
                        int64_t n, double tol, uint64_t* __restrict__ h1, uint64_t* __restrict__ h2,
                        int* __restrict__ nz) {
  __shared__ uint64_t s1[DT / 32], s2[DT / 32];
  __shared__ int sn[DT / 32];
  const int64_t cells = ell * q;
  const int nv = static_cast<int>(n / V);
  const int per = static_cast<int>(m) * nv;
  const int dr = DT / nv, dc = DT % nv;
  const int64_t row_step = static_cast<int64_t>(dr) * lda;
  for (int64_t cell = blockIdx.x; cell < cells; cell += gridDim.x) {
    const int64_t ci = cell / q, cj = cell % q;
    const double* blk = a + ci * m * lda + cj * n;
    uint64_t a1 = 0, a2 = 0;
    uint32_t any_bits = 0;
    int flag = 0;
    int r = threadIdx.x / nv, c = threadIdx.x % nv;
    const double* p = blk + static_cast<int64_t>(r) * lda + c * V;
    int idx0 = threadIdx.x;
    // full groups of DU accesses: no bounds tests, DU independent loads in flight
    for (; idx0 + (DU - 1) * DT < per; idx0 += DU * DT) {
      double x[DU][V];
#pragma unroll
      for (int u = 0; u < DU; ++u) {
        if (DC0) {
          load_vec<V>(p, x[u]);
          p += row_step;
        } else {
          load_vec<V>(blk + (int64_t)r * lda + c * V, x[u]);
          r += dr;
          c += dc;
          if (c >= nv) {
            c -= nv;
            ++r;
          }
        }
      }
      // one multiply pair per DU accesses; the per-access keys follow by adds
      const uint64_t kb1 = static_cast<uint64_t>(idx0) * kK1 + kK2;
      const uint64_t kb2 = static_cast<uint64_t>(idx0) * kK2 + kK1;
#pragma unroll
      for (int u = 0; u < DU; ++u)
        digest_access<V, EXACT>(x[u], kb1 + static_cast<uint64_t>(u) * (static_cast<uint64_t>(DT) * kK1),
                                kb2 + static_cast<uint64_t>(u) * (static_cast<uint64_t>(DT) * kK2), tol,
                                a1, a2, any_bits, flag);
    }
    for (; idx0 < per; idx0 += DT) {  // ragged tail
      double x[V];
      if (DC0) {
        load_vec<V>(p, x);
        p += row_step;
      } else {
        load_vec<V>(blk + (int64_t)r * lda + c * V, x);
        r += dr;
        c += dc;
        if (c >= nv) {
          c -= nv;
          ++r;
        }
      }
      digest_access<V, EXACT>(x, static_cast<uint64_t>(idx0) * kK1 + kK2,
                              static_cast<uint64_t>(idx0) * kK2 + kK1, tol, a1, a2, any_bits, flag);
    }
    if (EXACT) flag = any_bits != 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      flag |= __shfl_xor_sync(0xffffffffu, flag, o);
    }
    if ((threadIdx.x & 31) == 0) {
      s1[threadIdx.x >> 5] = a1;
      s2[threadIdx.x >> 5] = a2;
      sn[threadIdx.x >> 5] = flag;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t t1 = 0, t2 = 0;
      int f = 0;
      for (int w = 0; w < DT / 32; ++w) {
        t1 += s1[w];
        t2 += s2[w];
        f |= sn[w];
      }
      h1[cell] = t1;
      h2[cell] = t2;
      nz[cell] = f;
    }
    __syncthreads();
  }
}

// Grouping of equal digests on the device (the host lexsort + one round trip
// it replaces cost more than either HBM pass).  An open-addressing table of
// cell indices: a slot is owned by the first cell that claims it and stands
// for that cell's (h1, h2) key -- keys are read through the owner index from
// the read-only digest arrays, so no key is ever stored half-written; every
// kept cell with the owner's key lowers the slot's `first` by atomicMin, which
// makes the class leader the row-major first occurrence whatever the race
// order.  leader[cell] = that first cell (-1 for a skipped cell), cand[cell]
// = leader if another cell leads, else -1 (the match pass's input).
__device__ __forceinline__ uint32_t slot_hash(uint64_t k1, uint64_t k2) {
  uint64_t z = (k1 ^ (k2 >> 31) ^ (k2 << 33)) * 0xbf58476d1ce4e5b9ull;
  return static_cast<uint32_t>(z >> 32) ^ static_cast<uint32_t>(z);
}

__global__ void group_insert_kernel(const uint64_t* __restrict__ h1, const uint64_t* __restrict__ h2,
                                    const int* __restrict__ nz, int cells, uint32_t mask,
                                    int* owner, int* first, int* slot_of) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= cells) return;
  if (!nz[cell]) {
    slot_of[cell] = -1;
    return;
  }
  const uint64_t k1 = h1[cell], k2 = h2[cell];
  uint32_t s = slot_hash(k1, k2) & mask;
  for (;;) {
    int o = atomicCAS(&owner[s], -1, cell);
    if (o == -1) o = cell;
    if (o == cell || (h1[o] == k1 && h2[o] == k2)) break;
    s = (s + 1) & mask;
  }
  atomicMin(&first[s], cell);
  slot_of[cell] = static_cast<int>(s);
}

__global__ void group_leader_kernel(const int* __restrict__ slot_of, const int* __restrict__ first,
                                    int cells, int64_t* __restrict__ leader,
                                    int64_t* __restrict__ cand) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= cells) return;
  const int s = slot_of[cell];
  const int64_t l = s < 0 ? -1 : first[s];
  leader[cell] = l;
  cand[cell] = (l == cell) ? -1 : l;
}

uint32_t group_table_size(int64_t cells) {
  uint32_t t = 64;
  while (t < 2 * static_cast<uint64_t>(cells)) t <<= 1;
  return t;
}

// per cell with cand[cell] >= 0: eq[cell] = block(cell) matches block(cand)
// (exact: every 64-bit word equal; else max|d| <= tol, a NaN difference
// failing like numpy's `np.max(np.abs(blk - rep)) <= tol`)
template <int V>
__global__ void __launch_bounds__(DT)
    block_match_kernel(const double* __restrict__ a, int64_t lda, int64_t ell, int64_t q, int64_t m,
                       int64_t n, const int64_t* __restrict__ cand, double tol, int exact,
                       int* __restrict__ eq) {
  __shared__ int sb[DT / 32];
  const int64_t cells = ell * q;
  const int64_t nv = n / V;
  const int64_t per = m * nv;
  for (int64_t cell = blockIdx.x; cell < cells; cell += gridDim.x) {
    const int64_t rc = cand[cell];
    if (rc < 0) continue;  // CTA-uniform
    const double* blk = a + (cell / q) * m * lda + (cell % q) * n;
    const double* rep = a + (rc / q) * m * lda + (rc % q) * n;
    int bad = 0;
    int64_t r = threadIdx.x / nv, c = threadIdx.x % nv;
    const int64_t dr = DT / nv, dc = DT % nv;
    for (int64_t idx0 = threadIdx.x; idx0 < per; idx0 += DU * DT) {
      double x[DU][V], y[DU][V];
      bool ok[DU];
#pragma unroll
      for (int u = 0; u < DU; ++u) {
        ok[u] = idx0 + u * DT < per;
        if (ok[u]) {
          load_vec<V>(blk + r * lda + c * V, x[u]);
          if (V == 2) {
            const double2 v = ld_keep2(rep + r * lda + c * V);
            y[u][0] = v.x;
            y[u][V - 1] = v.y;
          } else {
            y[u][0] = ld_keep(rep + r * lda + c);
          }
        }
        r += dr;
        c += dc;
        if (c >= nv) {
          c -= nv;
          ++r;
        }
      }
#pragma unroll
      for (int u = 0; u < DU; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if (exact)
            bad |= __double_as_longlong(x[u][e]) != __double_as_longlong(y[u][e]);
          else
            bad |= !(fabs(x[u][e] - y[u][e]) <= tol);
        }
      }
    }
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = bad;
    __syncthreads();
    if (threadIdx.x == 0) {
      int b = 0;
      for (int w = 0; w < DT / 32; ++w) b |= sb[w];
      eq[cell] = !b;
    }
    __syncthreads();
  }
}

bool vec2_ok(const double* a, int64_t lda, int64_t n) {
  return (n % 2 == 0) && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15u) == 0);
}

int grid_cells(int64_t cells) {
  return static_cast<int>(std::min<int64_t>(cells, static_cast<int64_t>(bt_num_sms()) * 8));
}

}  // namespace

extern "C" int bt_block_digest_f64(const double* a, int64_t lda, int64_t ell, int64_t q, int64_t m,
                                   int64_t n, double tol, uint64_t* h1, uint64_t* h2, int* nz,
                                   void* stream) {
  BT_NVTX("bt_block_digest_f64");
  BT_REQUIRE(ell >= 1 && q >= 1 && m >= 1 && n >= 1, BT_E_SHAPE, "digest: empty grid");
  BT_REQUIRE(lda >= q * n, BT_E_SHAPE, "digest: lda too small");
  BT_REQUIRE(m * (n / (vec2_ok(a, lda, n) ? 2 : 1)) < ((int64_t)1 << 31), BT_E_SHAPE,
             "digest: block too large");
  cudaStream_t st = bt_stream(stream);
  const bool v2 = vec2_ok(a, lda, n);
  const int64_t nv = n / (v2 ? 2 : 1);
  const bool dc0 = nv <= DT && DT % nv == 0;
  const bool exact = tol == 0.0;
  // one wave of resident CTAs, each walking its share of the cells (a grid
  // above the resident count left a part-filled second wave: 1184 CTAs on
  // 6 x 148 slots ran as long as two full waves)
#define BT_DIGEST(V, E, D)                                                                        \
  do {                                                                                            \
    static int per_sm = 0;                                                                        \
    if (per_sm == 0) {                                                                            \
      BT_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(                                \
          &per_sm, block_digest_kernel<V, E, D>, DT, 0));                                         \
      if (per_sm < 1) per_sm = 1;                                                                 \
    }                                                                                             \
    const int grid = static_cast<int>(                                                            \
        std::min<int64_t>(ell * q, static_cast<int64_t>(bt_num_sms()) * per_sm));                 \
    block_digest_kernel<V, E, D><<<grid, DT, 0, st>>>(a, lda, ell, q, m, n, tol, h1, h2, nz);     \
  } while (0)
  if (v2) {
    if (exact) { if (dc0) BT_DIGEST(2, true, true); else BT_DIGEST(2, true, false); }
    else       { if (dc0) BT_DIGEST(2, false, true); else BT_DIGEST(2, false, false); }
  } else {
    if (exact) { if (dc0) BT_DIGEST(1, true, true); else BT_DIGEST(1, true, false); }
    else       { if (dc0) BT_DIGEST(1, false, true); else BT_DIGEST(1, false, false); }
  }
#undef BT_DIGEST
  BT_LAUNCH_CHECK();
  return BT_OK;
}

extern "C" int bt_block_match_f64(const double* a, int64_t lda, int64_t ell, int64_t q, int64_t m,
                                  int64_t n, const int64_t* cand, double tol, int exact, int* eq,
                                  void* stream) {
  BT_NVTX("bt_block_match_f64");
  BT_REQUIRE(ell >= 1 && q >= 1 && m >= 1 && n >= 1, BT_E_SHAPE, "match: empty grid");
  BT_REQUIRE(lda >= q * n, BT_E_SHAPE, "match: lda too small");
  if (vec2_ok(a, lda, n))
    block_match_kernel<2><<<grid_cells(ell * q), DT, 0, bt_stream(stream)>>>(a, lda, ell, q, m, n,
                                                                            cand, tol, exact, eq);
  else
    block_match_kernel<1><<<grid_cells(ell * q), DT, 0, bt_stream(stream)>>>(a, lda, ell, q, m, n,
                                                                            cand, tol, exact, eq);
  BT_LAUNCH_CHECK();
  return BT_OK;
}

extern "C" int64_t bt_block_group_ws_bytes(int64_t cells) {
  if (cells < 1 || cells >= (int64_t)0x3f000000) return -1;
  return (2 * static_cast<int64_t>(group_table_size(cells)) + cells) * 4;
}

extern "C" int bt_block_group(const uint64_t* h1, const uint64_t* h2, const int* nz, int64_t cells,
                              int64_t* leader, int64_t* cand, void* ws, int64_t ws_bytes,
                              void* stream) {
  BT_NVTX("bt_block_group");
  BT_REQUIRE(cells >= 1 && cells < (int64_t)0x3f000000, BT_E_SHAPE, "group: cell count out of range");
  BT_REQUIRE(ws != nullptr && ws_bytes >= bt_block_group_ws_bytes(cells), BT_E_SHAPE,
             "group: workspace too small");
  const uint32_t tsz = group_table_size(cells);
  cudaStream_t st = bt_stream(stream);
  int* owner = static_cast<int*>(ws);
  int* first = owner + tsz;
  int* slot_of = first + tsz;
  BT_CUDA_CHECK(cudaMemsetAsync(owner, 0xff, sizeof(int) * tsz, st));  // -1: free
  BT_CUDA_CHECK(cudaMemsetAsync(first, 0x7f, sizeof(int) * tsz, st));  // 0x7f7f7f7f > any cell index
  const int nc = static_cast<int>(cells);
  const unsigned blocks = static_cast<unsigned>(bt_cdiv(cells, 256));
  group_insert_kernel<<<blocks, 256, 0, st>>>(h1, h2, nz, nc, tsz - 1, owner, first, slot_of);
  BT_LAUNCH_CHECK();
  group_leader_kernel<<<blocks, 256, 0, st>>>(slot_of, first, nc, leader, cand);
  BT_LAUNCH_CHECK();
  return BT_OK;
}
