// Fused global-norm clip + Adam over a flat fp32 parameter buffer (adam.cu).
#pragma once
#include "common.cuh"

namespace sl {

struct AdamHyper {
  float lr, beta1, beta2, eps;
  float grad_scale;  // applied to the gradient first (e.g. 1/N after a sum all-reduce)
  float clip_norm;   // <= 0: no clipping
  float inv_bc1, inv_bc2;  // 1 / (1 - beta^t), computed in double on the host
};

struct AdamScratch {  // device scratch, zeroed per step
  double sumsq;
  unsigned nonfinite;
  unsigned pad;
};

void adam_step(int64_t n, float* params, const float* grads, float* m, float* v, const AdamHyper& h,
               AdamScratch* scratch, float* norm_out, int32_t* nonfinite_out, cudaStream_t stream);

}  // namespace sl
