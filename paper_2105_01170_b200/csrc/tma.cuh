// TMA (cp.async.bulk.tensor) helpers: host-side tensor-map encoding through
// the driver entry point (no libcuda link), device-side bulk tensor loads
// that complete on an mbarrier's transaction count.
#pragma once

#include <cuda.h>

#include "bt_common.cuh"

// Encode a 3-D tiled map of an fp64 C-order array (d2, d1, d0) -- d0
// fastest -- with box (b0, b1, b2) and 128-byte swizzle (b0 * 8 == 128).
// Out-of-range box elements are zero-filled by the hardware.  Returns BT_OK
// or BT_E_CUDA (message set).
int bt_tma_map_f64_3d(CUtensorMap* map, const double* base, int64_t d0, int64_t d1, int64_t d2,
                      int64_t stride1_elems, int64_t stride2_elems, int b0, int b1, int b2);

// 2-D map of an fp64 row-major (d1, d0) array, row stride stride1_elems,
// box (b0, b1), 128-byte swizzle (b0 * 8 == 128)
int bt_tma_map_f64_2d(CUtensorMap* map, const double* base, int64_t d0, int64_t d1,
                      int64_t stride1_elems, int b0, int b1);

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// box load of `map` at coordinates (c0, c1, c2) into smem `dst`; the bytes
// complete_tx on `bar`
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
