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

constexpr int kAdamMaxBlocks = 2048;
struct AdamScratch {  // device scratch (zero when created)
  double sumsq;        // zeroed per step; the fixed-order total of part[]
  unsigned nonfinite;  // zeroed per step
  int32_t t;           // persistent step counter (byte offset 12: optim.py reads it)
  unsigned ticket;     // blocks done with pass 1; the last one resets it
  unsigned pad;
  double part[kAdamMaxBlocks];  // per-block sums of squares (deterministic reduction)
};

void adam_step(int64_t n, float* params, const float* grads, float* m, float* v, const AdamHyper& h,
               AdamScratch* scratch, float* norm_out, int32_t* nonfinite_out, cudaStream_t stream);

}  // namespace sl
