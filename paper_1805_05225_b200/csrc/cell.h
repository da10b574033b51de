// Decoder cell step (K5) — see cell.cu.
#pragma once
#include "common.cuh"

namespace sl {

void cell_fwd(int B, int D, int H, const float* x, const float* h0, const float* c0,
              const float* W, const float* R, const float* b, float* h, float* c, float* saved,
              cudaStream_t stream);
void cell_bwd(int B, int D, int H, const float* x, const float* h0, const float* c0,
              const float* W, const float* R, const float* saved, const float* gh,
              const float* gc, float* dx, float* dh0, float* dc0, float* dW, float* dR,
              float* db, int accumulate, cudaStream_t stream);

}  // namespace sl
