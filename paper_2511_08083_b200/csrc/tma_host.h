// Host-side TMA tensor-map encoding through the driver entry point (the
// library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <mutex>

namespace hk {

inline PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// A BNHD bf16 tensor [B][N][H][d] viewed as the 4-D map (d, H, N, B), box
// (64, 1, box_rows, 1), 128-byte swizzle: one box = box_rows x 128 B, the
// canonical SWIZZLE_128B K-major atom stacked along rows.
// Last CUresult from encode_bnhd (per thread), for error messages.
inline int& last_encode_result() {
  static thread_local int r = 0;
  return r;
}

inline bool encode_bnhd(CUtensorMap* map, const void* base, int B, int N, int H, int d, int box_rows) {
  auto fn = get_encode_fn();
  if (!fn) {
    last_encode_result() = -1;
    return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)H * d * 2, (cuuint64_t)N * H * d * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  last_encode_result() = (int)r;
  return r == CUDA_SUCCESS;
}

// An fp32 BNHD tensor [B][N][H][d] as the 4-D map (d, H, N, B), box (32, 1, 128, 1), 128-byte
// swizzle (32 fp32 = 128 B per box row): the fused backward's dQ accumulator (bulk reduce-add).
inline bool encode_bnhd_f32(CUtensorMap* map, const void* base, int B, int N, int H, int d) {
  auto fn = get_encode_fn();
  if (!fn) {
    last_encode_result() = -1;
    return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)d * 4, (cuuint64_t)H * d * 4, (cuuint64_t)N * H * d * 4};
  cuuint32_t box[4] = {32, 1, 128, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  last_encode_result() = (int)r;
  return r == CUDA_SUCCESS;
}

// A row-major bf16 matrix [rows][cols] viewed as the 2-D map (cols, rows), box
// (64, box_rows), 128-byte swizzle (K-major operand tiles for tcgen05).
inline bool encode_rowmajor(CUtensorMap* map, const void* base, int rows, int cols, int box_rows) {
  auto fn = get_encode_fn();
  if (!fn) {
    last_encode_result() = -1;
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  last_encode_result() = (int)r;
  return r == CUDA_SUCCESS;
}

}  // namespace hk
