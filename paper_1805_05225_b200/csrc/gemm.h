// Internal GEMM entry points (row-major, see gemm_f32.cu / gemm_tc.cu).
#pragma once
#include "common.cuh"

namespace sl {

// FP32 SIMT GEMM: C = alpha*op(A)*op(B) + beta*C + bias.
void gemm_f32(bool transA, bool transB, int M, int N, int K, float alpha, const float* A,
              int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
              const float* bias, cudaStream_t stream);

}  // namespace sl
