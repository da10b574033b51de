// Layout / precision conversion kernels for the BF16 path: fp32 row-major
// [rows, cols] (src_ld) -> bf16 [rows, cols] (dst_ld).  Vectorised 4-wide
// when both leading dimensions allow it; grid sized to the SM count.
#include "convert.h"
#include "profile.h"

namespace sl {
namespace {

// One warp per row (grid-stride over rows), lanes along the columns, 4 per
// lane when the layout allows: coalesced, no per-element 64-bit div / mod.
__global__ void f32_to_bf16_kernel(int64_t rows, int64_t cols, const float* __restrict__ src,
                                   int64_t src_ld, __nv_bfloat16* __restrict__ dst, int64_t dst_ld,
                                   bool vec) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const float* s = src + r * src_ld;
    __nv_bfloat16* d = dst + r * dst_ld;
    if (vec) {
      for (int64_t c = lane * 4; c < cols; c += 128) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(s + c));
        const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        *reinterpret_cast<uint2*>(d + c) =
            make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
      }
    } else {
      for (int64_t c = lane; c < cols; c += 32) d[c] = __float2bfloat16_rn(s[c]);
    }
  }
}

__global__ void fill_col_bf16_kernel(int64_t rows, int64_t col, __nv_bfloat16* dst, int64_t ld,
                                     __nv_bfloat16 v) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    dst[r * ld + col] = v;
}

}  // namespace

void fill_col_bf16(int64_t rows, int64_t col, __nv_bfloat16* dst, int64_t ld, float value,
                   cudaStream_t stream) {
  if (rows <= 0) return;
  fill_col_bf16_kernel<<<(int)std::min<int64_t>(ceil_div(rows, 256), 148 * 4), 256, 0, stream>>>(
      rows, col, dst, ld, __float2bfloat16_rn(value));
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void f32_to_bf16(int64_t rows, int64_t cols, const float* src, int64_t src_ld, __nv_bfloat16* dst,
                 int64_t dst_ld, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  const bool vec = (cols % 4 == 0) && (src_ld % 4 == 0) && (dst_ld % 4 == 0) &&
                   ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 8 == 0);
  const int grid = (int)std::min<int64_t>(ceil_div(rows, 8), 148 * 8);  // 8 rows (warps) per block
  f32_to_bf16_kernel<<<grid, 256, 0, stream>>>(rows, cols, src, src_ld, dst, dst_ld, vec);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace sl
