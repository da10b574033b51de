#pragma once
#include "common.cuh"

namespace sl {

// fp32 [rows, cols] (src_ld) -> bf16 (dst_ld), round-to-nearest-even.
void f32_to_bf16(int64_t rows, int64_t cols, const float* src, int64_t src_ld, __nv_bfloat16* dst,
                 int64_t dst_ld, cudaStream_t stream);

// dst[r * ld + col] = value for every row (the ones column of [X | 1]).
void fill_col_bf16(int64_t rows, int64_t col, __nv_bfloat16* dst, int64_t ld, float value,
                   cudaStream_t stream);

}  // namespace sl
