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

// one multiply + xor-shift per word and digest: the digest only has to make
// collisions rare (every grouping is verified bit for bit afterwards)
__device__ __forceinline__ uint64_t mix_lite(uint64_t z, uint64_t mul) {
  z = (z ^ (z >> 32)) * mul;
  return z ^ (z >> 29);
}

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

__device__ __forceinline__ uint64_t rotl64(uint64_t w, unsigned r) {
  return (w << r) | (w >> (64u - r));
}

// per cell: h1, h2 (digest), nz (EXACT, i.e. tol == 0: any word not +-0.0;
// else max|x| > tol or NaN present).  V doubles per access, keyed by the
// access's position in the block (row-major); the V words of an access share
// one multiply in h1.  32-bit walk indices (a block has < 2^31 accesses).
template <int V, bool EXACT>
__global__ void __launch_bounds__(DT)
    block_digest_kernel(const double* __restrict__ a, int64_t lda, int64_t ell, int64_t q, int64_t m,
                        int64_t n, double tol, uint64_t* __restrict__ h1, uint64_t* __restrict__ h2,
                        int* __restrict__ nz) {
  __shared__ uint64_t s1[DT / 32], s2[DT / 32];
  __shared__ int sn[DT / 32];
  const int64_t cells = ell * q;
  const int nv = static_cast<int>(n / V);
  const int per = static_cast<int>(m) * nv;
  const int dr = DT / nv, dc = DT % nv;
  for (int64_t cell = blockIdx.x; cell < cells; cell += gridDim.x) {
    const int64_t ci = cell / q, cj = cell % q;
    const double* blk = a + ci * m * lda + cj * n;
    uint64_t a1 = 0, a2 = 0;
    int flag = 0;
    int r = threadIdx.x / nv, c = threadIdx.x % nv;
    for (int idx0 = threadIdx.x; idx0 < per; idx0 += DU * DT) {
      double x[DU][V];
#pragma unroll
      for (int u = 0; u < DU; ++u) {  // DU independent loads in flight per thread
        if (idx0 + u * DT < per) load_vec<V>(blk + (int64_t)r * lda + c * V, x[u]);
        r += dr;
        c += dc;
        if (c >= nv) {
          c -= nv;
          ++r;
        }
      }
      const uint64_t kbase = static_cast<uint64_t>(idx0) * kK1;  // one multiply per DU accesses
#pragma unroll
      for (int u = 0; u < DU; ++u) {
        const int pos = idx0 + u * DT;
        if (pos >= per) continue;
        const uint64_t k1 = kbase + static_cast<uint64_t>(u) * (static_cast<uint64_t>(DT) * kK1);
        const uint64_t w0 = static_cast<uint64_t>(__double_as_longlong(x[u][0]));
        const uint64_t w1 = static_cast<uint64_t>(__double_as_longlong(x[u][V - 1]));
        const uint64_t z = (V == 2) ? (w0 ^ k1) + rotl64(w1 ^ kK2, 29) : (w0 ^ k1);
        a1 += mix_lite(z, 0xbf58476d1ce4e5b9ull);
        const unsigned rot = (static_cast<unsigned>(pos) & 63u) | 1u;
        a2 += rotl64(w0, rot) ^ k1;
        if (V == 2) a2 += rotl64(w1, rot ^ 62u) + k1;
        if (EXACT) {
          flag |= (w0 << 1) != 0;  // not +0.0 / -0.0 (NaN counts as nonzero, like np.any)
          if (V == 2) flag |= (w1 << 1) != 0;
        } else {
          flag |= !(fabs(x[u][0]) <= tol);  // NaN or |x| > tol
          if (V == 2) flag |= !(fabs(x[u][V - 1]) <= tol);
        }
      }
    }
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
  const int grid = grid_cells(ell * q);
  cudaStream_t st = bt_stream(stream);
  if (vec2_ok(a, lda, n)) {
    if (tol == 0.0)
      block_digest_kernel<2, true><<<grid, DT, 0, st>>>(a, lda, ell, q, m, n, tol, h1, h2, nz);
    else
      block_digest_kernel<2, false><<<grid, DT, 0, st>>>(a, lda, ell, q, m, n, tol, h1, h2, nz);
  } else {
    if (tol == 0.0)
      block_digest_kernel<1, true><<<grid, DT, 0, st>>>(a, lda, ell, q, m, n, tol, h1, h2, nz);
    else
      block_digest_kernel<1, false><<<grid, DT, 0, st>>>(a, lda, ell, q, m, n, tol, h1, h2, nz);
  }
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
