// tmap.cpp -- TMA tensor maps for the SSAM streaming loaders.
#include "tmap.hpp"

#include <cstdlib>
#include <mutex>

namespace ssam_b200 {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static std::once_flag once;
  static EncodeFn fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}
// L2 fetch granularity for box rows.  Box rows start 16-byte aligned inside
// rows shared with neighbouring strips; SSAM_B200_L2PROMO (0/64/128/256)
// overrides the default for experiments.
CUtensorMapL2promotion l2_promotion() {
  static const CUtensorMapL2promotion v = [] {
    const char* e = std::getenv("SSAM_B200_L2PROMO");
    const int b = e ? std::atoi(e) : 128;
    return b >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
           : b >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
           : b >= 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                      : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  }();
  return v;
}
}  // namespace

cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, int elem_bytes, uint64_t cols,
                         uint64_t rows, uint64_t row_bytes, uint32_t box_cols,
                         uint32_t box_rows) {
  EncodeFn fn = encoder();
  if (!fn) return cudaErrorNotSupported;
  // 4- and 8-byte elements are moved as raw bits; zero fill is all-zero bits.
  const CUtensorMapDataType dt =
      elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_INT64;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace ssam_b200
