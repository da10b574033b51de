// The reference's counter-based input dropout (dropout.cu).
#pragma once
#include <algorithm>

#include "common.cuh"

namespace sl {

void dropout_apply(int B, int T, int F, float rate, uint64_t key0, const int32_t* counter, int64_t counter_value,
                   const float* in, float* out, cudaStream_t st);

}  // namespace sl
