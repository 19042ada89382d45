// Host-side tensor-map encoders shared by the attention kernels.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace vp {

inline PFN_cuTensorMapEncodeTiled_v12000 encode3() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3D map over a [B, S, cols] bf16 activation: box {64 cols, rows, 1}
// (SWIZZLE_128B), or {32 cols, rows, 1} with SWIZZLE_64B when narrow.
inline bool make_tmap_bsc(CUtensorMap* map, const void* base, uint64_t cols, uint64_t S,
                          uint64_t B, uint32_t rows, bool narrow = false) {
  auto fn = encode3();
  if (!fn) return false;
  cuuint64_t dims[3] = {cols, S, B};
  cuuint64_t strides[2] = {cols * 2, S * cols * 2};
  cuuint32_t box[3] = {narrow ? 32u : 64u, rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            narrow ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3D map over a [B, S, cols] fp32 accumulator: box {32 cols (128 B), rows, 1}.
inline bool make_tmap_bsc_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t S,
                              uint64_t B, uint32_t rows) {
  auto fn = encode3();
  if (!fn) return false;
  cuuint64_t dims[3] = {cols, S, B};
  cuuint64_t strides[2] = {cols * 4, S * cols * 4};
  cuuint32_t box[3] = {32, rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace vp
