// bt200 -- shared device helpers and C-ABI error plumbing (sm_100a only).
//
// Status codes mirror the reference's exception classes (errors.py:11-32,
// exit-code classes cli.py:383-397); see include/bt200.h.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include "../../include/bt200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "bt200 is built for sm_100a only"
#endif

void bt_set_error(const char* fmt, ...);

#define BT_CUDA_CHECK(x)                                                                  \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      bt_set_error("%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_));       \
      return BT_E_CUDA;                                                                   \
    }                                                                                     \
  } while (0)

// every kernel launch site is followed by BT_LAUNCH_CHECK(), which also
// counts the launch (bt_launch_count(): evidence of native work per step)
void bt_count_launch();
#define BT_LAUNCH_CHECK()              \
  do {                                 \
    bt_count_launch();                 \
    BT_CUDA_CHECK(cudaGetLastError()); \
  } while (0)

#define BT_TRY(x)                  \
  do {                             \
    int s_ = (x);                  \
    if (s_ != BT_OK) return s_;    \
  } while (0)

#define BT_REQUIRE(cond, code, ...)     \
  do {                                  \
    if (!(cond)) {                      \
      bt_set_error(__VA_ARGS__);        \
      return code;                      \
    }                                   \
  } while (0)

// NVTX range around a C-ABI call (header-only NVTX3: a no-op unless a tool
// such as nsys / ncu is attached); names are the C-ABI entry points
struct BtNvtxRange {
  explicit BtNvtxRange(const char* name) { nvtxRangePushA(name); }
  ~BtNvtxRange() { nvtxRangePop(); }
  BtNvtxRange(const BtNvtxRange&) = delete;
  BtNvtxRange& operator=(const BtNvtxRange&) = delete;
};
#define BT_NVTX(name) BtNvtxRange bt_nvtx_range_(name)

static inline cudaStream_t bt_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static inline int64_t bt_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// device primitives
// ---------------------------------------------------------------------------

// FP64 tensor-core MMA.  On sm_100a every f64 mma.sync shape lowers to
// DMMA.8x8x4 in SASS, so m8n8k4 is the native primitive.
// Fragments (PTX ISA, mma.m8n8k4 .f64): lane = 4*g + t;
//   A(8x4, row): a = A[g][t];  B(4x8, col): b = B[t][g];
//   C(8x8): c0 = C[g][2t], c1 = C[g][2t+1].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero-fill of the bytes beyond src_bytes.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// mbarrier helpers (shared::cta)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void mbar_cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Streaming loads/stores for single-pass HBM traffic (L2 evict-first
// policy via createpolicy + cache_hint; L1 not allocated).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(p), "l"(l2_policy_evict_first()));
  return v;
}
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(l2_policy_evict_first()));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* p) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v)
               : "l"(p), "l"(l2_policy_evict_last()));
  return v;
}
__device__ __forceinline__ double2 ld_keep2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(l2_policy_evict_last()));
  return v;
}
__device__ __forceinline__ void st_stream(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v));
}
__device__ __forceinline__ void st_stream2(double* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Shared-memory leading dimension (in doubles) that is == 4 (mod 16): the
// 8x4 fragment reads of m8n8k4 (addr = t*ld + g or g*ld + t) then hit 16
// distinct 8-byte banks in each half-warp -- conflict free.
__host__ __device__ constexpr int bt_ld(int x) { return x + ((4 - (x % 16)) % 16 + 16) % 16; }

// number of SMs, cached per process (device 0 semantics of the caller's
// current device)
int bt_num_sms();

// keep cudaMallocAsync scratch cached in the device's default pool (gemm.cu)
void bt_keep_async_pool();
