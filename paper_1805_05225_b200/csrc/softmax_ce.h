// Output projection + log_softmax + label-smoothed cross entropy (softmax_ce.cu).
#pragma once
#include "common.cuh"

namespace sl {

struct CeDims {
  int64_t rows, Dp, Vp;
  int nblk;  // 128-column softmax blocks per row
};
CeDims ce_dims(int B, int T, int D, int V);
size_t output_ce_workspace_bytes(int B, int T, int D, int V);
// x [B*T, D] fp32 (row r = b*T + t), targets [B*T], W [D, V], b [V]; loss_out a
// device scalar (mean over valid positions); dx [B*T, D], dW [D, V], db [V] may
// be null; bad_target (device int) is set when a valid position's id is out of range.
void output_ce(int B, int T, int D, int V, const float* x, const int32_t* targets, const int32_t* lens,
               const float* W, const float* b, float eps, float* loss_out, float* dx, float* dW, float* db,
               bool accumulate, void* workspace, int* bad_target, cudaStream_t stream);

// the same at the reference's precision: fp32 logits, split-bf16 tcgen05 GEMMs (x3)
size_t output_ce_f32_workspace_bytes(int B, int T, int D, int V);
void output_ce_f32(int B, int T, int D, int V, const float* x, const int32_t* targets, const int32_t* lens,
                   const float* W, const float* b, float eps, float* loss_out, float* dx, float* dW, float* db,
                   bool accumulate, void* workspace, int* bad_target, cudaStream_t stream);

}  // namespace sl
