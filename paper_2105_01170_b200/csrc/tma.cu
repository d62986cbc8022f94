// Host side of tma.cuh: cuTensorMapEncodeTiled resolved once through
// cudaGetDriverEntryPoint (the library links only the static runtime).
#include <mutex>

#include "tma.cuh"

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}
}  // namespace

static int encode(CUtensorMap* map, const double* base, int rank, const cuuint64_t* dims,
                  const cuuint64_t* strides, const cuuint32_t* box) {
  EncodeFn fn = encode_fn();
  BT_REQUIRE(fn != nullptr, BT_E_CUDA, "TMA: cuTensorMapEncodeTiled unavailable");
  BT_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15u) == 0, BT_E_CUDA, "TMA: base not 16-byte aligned");
  for (int d = 0; d + 1 < rank; ++d)
    BT_REQUIRE(strides[d] % 16 == 0, BT_E_CUDA, "TMA: stride not a multiple of 16 bytes");
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BT_REQUIRE(r == CUDA_SUCCESS, BT_E_CUDA, "TMA: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BT_OK;
}

int bt_tma_map_f64_2d(CUtensorMap* map, const double* base, int64_t d0, int64_t d1,
                      int64_t stride1_elems, int b0, int b1) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d0), static_cast<cuuint64_t>(d1)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(stride1_elems * 8)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(b0), static_cast<cuuint32_t>(b1)};
  return encode(map, base, 2, dims, strides, box);
}

int bt_tma_map_f64_3d(CUtensorMap* map, const double* base, int64_t d0, int64_t d1, int64_t d2,
                      int64_t stride1_elems, int64_t stride2_elems, int b0, int b1, int b2) {
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d0), static_cast<cuuint64_t>(d1),
                              static_cast<cuuint64_t>(d2)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(stride1_elems * 8),
                                 static_cast<cuuint64_t>(stride2_elems * 8)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(b0), static_cast<cuuint32_t>(b1),
                             static_cast<cuuint32_t>(b2)};
  return encode(map, base, 3, dims, strides, box);
}
