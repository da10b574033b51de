// Fused global-norm clip + Adam over a flat fp32 parameter buffer (adam.cu).
#pragma once
#include "common.cuh"

namespace sl {

struct AdamHyper {
  float lr, beta1, beta2, eps;
  float grad_scale;  // applied to the gradient first (e.g. 1/N after a sum all-reduce)
  float clip_norm;   // <= 0: no clipping
  int32_t step;      // > 0: this step number; 0: the device counter in the scratch + 1
};

struct AdamScratch {  // device scratch
  double sumsq;        // zeroed per step
  unsigned nonfinite;  // zeroed per step
  int32_t t;           // persistent step counter (zero when the scratch is created)
};

void adam_step(int64_t n, float* params, const float* grads, float* m, float* v, const AdamHyper& h,
               AdamScratch* scratch, float* norm_out, int32_t* nonfinite_out, cudaStream_t stream);

}  // namespace sl
