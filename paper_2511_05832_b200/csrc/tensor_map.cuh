// Host-side TMA descriptor construction (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so libhla does not link libcuda directly).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace hla {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline hla_status get_encode_fn(EncodeTiledFn* fn) {
  static EncodeTiledFn cached = nullptr;
  if (!cached) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    HLA_REQUIRE(e == cudaSuccess && p != nullptr && q == cudaDriverEntryPointSuccess, HLA_ERR_CUDA,
                "cuTensorMapEncodeTiled unavailable: %s", cudaGetErrorString(e));
    cached = reinterpret_cast<EncodeTiledFn>(p);
  }
  *fn = cached;
  return HLA_OK;
}

// bf16 tensor [rows_total, heads, head_dim] viewed as 3-D (head_dim, heads, rows);
// box = (head_dim, 1, box_rows); swizzle = head_dim * 2 bytes (64 -> 128B, 32 -> 64B).
inline hla_status make_rows_map(CUtensorMap* map, const void* base, int64_t rows_total, int heads, int head_dim,
                                int box_rows) {
  EncodeTiledFn enc;
  hla_status st = get_encode_fn(&enc);
  if (st != HLA_OK) return st;
  cuuint64_t dims[3] = {(cuuint64_t)head_dim, (cuuint64_t)heads, (cuuint64_t)rows_total};
  cuuint64_t strides[2] = {(cuuint64_t)head_dim * 2, (cuuint64_t)heads * head_dim * 2};
  cuuint32_t box[3] = {(cuuint32_t)head_dim, 1, (cuuint32_t)box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMapSwizzle swz = head_dim * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                           : head_dim * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HLA_REQUIRE(r == CUDA_SUCCESS, HLA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HLA_OK;
}

// bf16 tensor [batch, grid_h * grid_w cells, heads, head_dim] viewed as 5-D (head_dim, heads,
// grid_w, grid_h, batch); box = (head_dim, 1, 8, 8, 1): one op moves an aligned 8 x 8 cell square
// of one head, 64 rows in raster order -- a 64-token segment of the tiled Hilbert order.
inline hla_status make_square_map(CUtensorMap* map, const void* base, int batch, int grid_h, int grid_w, int heads,
                                  int head_dim, int box_rows = 8) {
  EncodeTiledFn enc;
  hla_status st = get_encode_fn(&enc);
  if (st != HLA_OK) return st;
  const cuuint64_t row = (cuuint64_t)heads * head_dim * 2;
  cuuint64_t dims[5] = {(cuuint64_t)head_dim, (cuuint64_t)heads, (cuuint64_t)grid_w, (cuuint64_t)grid_h,
                        (cuuint64_t)batch};
  cuuint64_t strides[4] = {(cuuint64_t)head_dim * 2, row, row * grid_w, row * grid_w * grid_h};
  cuuint32_t box[5] = {(cuuint32_t)head_dim, 1, 8, (cuuint32_t)box_rows, 1};   // box_rows < 8: part of a square
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUtensorMapSwizzle swz = head_dim * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                           : head_dim * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HLA_REQUIRE(r == CUDA_SUCCESS, HLA_ERR_CUDA, "cuTensorMapEncodeTiled (square) failed (%d)", (int)r);
  return HLA_OK;
}

// bf16 tensor [rows_total, heads * head_dim] viewed as 2-D (heads*head_dim, rows) for
// .tile::gather4 loads of single token rows: box = (head_dim, box_h).
inline hla_status make_gather_map(CUtensorMap* map, const void* base, int64_t rows_total, int heads, int head_dim,
                                  int box_h = 1) {
  EncodeTiledFn enc;
  hla_status st = get_encode_fn(&enc);
  if (st != HLA_OK) return st;
  cuuint64_t dims[2] = {(cuuint64_t)heads * head_dim, (cuuint64_t)rows_total};
  cuuint64_t strides[1] = {(cuuint64_t)heads * head_dim * 2};
  cuuint32_t box[2] = {(cuuint32_t)head_dim, (cuuint32_t)box_h};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle swz = head_dim * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                           : head_dim * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HLA_REQUIRE(r == CUDA_SUCCESS, HLA_ERR_CUDA, "cuTensorMapEncodeTiled (gather) failed (%d)", (int)r);
  return HLA_OK;
}

// fp32 tensor [rows_total, heads, head_dim] as 3-D (head_dim, heads, rows); box =
// (box_cols, 1, box_rows), SWIZZLE_128B (box_cols * 4 == 128).
// box_cols 32 (128-B rows, 128B swizzle) or 16 (64-B rows, 64B swizzle)
inline hla_status make_f32_rows_map(CUtensorMap* map, const void* base, int64_t rows_total, int heads, int head_dim,
                                    int box_cols, int box_rows) {
  EncodeTiledFn enc;
  hla_status st = get_encode_fn(&enc);
  if (st != HLA_OK) return st;
  cuuint64_t dims[3] = {(cuuint64_t)head_dim, (cuuint64_t)heads, (cuuint64_t)rows_total};
  cuuint64_t strides[2] = {(cuuint64_t)head_dim * 4, (cuuint64_t)heads * head_dim * 4};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, 1, (cuuint32_t)box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HLA_REQUIRE(r == CUDA_SUCCESS, HLA_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (%d)", (int)r);
  return HLA_OK;
}

}  // namespace hla
