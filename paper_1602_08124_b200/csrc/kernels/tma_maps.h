// Tensor-map encoders shared by the conv kernels (driver entry points are
// resolved at run time through cudaGetDriverEntryPoint).
#pragma once
#include <cuda.h>

#include <cstdint>

namespace vdnnk {
bool encode_tiled(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                  const cuuint32_t* box, CUtensorMapSwizzle sw,
                  CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
// esz: element bytes (4 fp32, 2 bf16); one load = `pixels` rows of 128 bytes
bool encode_im2col(CUtensorMap* m, const void* base, int n, int h, int w, int c, int k, int stride, int pad,
                   int pixels, CUtensorMapSwizzle sw, int esz = 4);
// 2D [rows][cols] fp32 with 128-row x 32-col SWIZZLE_128B boxes (TMA-store epilogues)
bool encode_out(CUtensorMap* m, const void* base, int64_t rows, int cols);
}  // namespace vdnnk
