/* seqloom_cuda_internal.h — test / benchmarking hooks of libseqloom_cuda.so.
 * Not part of the drop-in boundary (see seqloom_cuda.h); used by tests/ to
 * check individual kernels against torch references. */
#ifndef SEQLOOM_CUDA_INTERNAL_H_
#define SEQLOOM_CUDA_INTERNAL_H_
#include "seqloom_cuda.h"
#ifdef __cplusplus
extern "C" {
#endif
/* C[M,N] = alpha * op(A) op(B) + beta * C + bias on the BF16 tcgen05 GEMM.
 * A: a_mn ? [K, M] : [M, K] bf16 (lda);  B: b_mn ? [K, N] : [N, K] bf16 (ldb). */
int sl_debug_gemm_bf16(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
                       int64_t ldb, int b_mn, float* C, int64_t ldc, float alpha, float beta,
                       const float* bias, sl_stream_t stream);
/* Same GEMM with A [M,K] K-major, B [K,N] N-major and a bf16 output (K1's XW path). */
int sl_debug_gemm_bf16_out(int M, int N, int K, const void* A, int64_t lda, const void* B,
                           int64_t ldb, void* Cb, int64_t ldc, const float* bias, sl_stream_t stream);
/* C = op(A) op(B) + beta C (+ bias) on the fp32-class split-bf16 GEMM (gemm_f32x3.cu);
 * ws: sl_debug_gemm_f32x3_ws bytes. */
size_t sl_debug_gemm_f32x3_ws(int transA, int transB, int M, int N, int K);
int sl_debug_gemm_f32x3(int transA, int transB, int M, int N, int K, const float* A, int64_t lda, const float* B,
                        int64_t ldb, float beta, float* C, int64_t ldc, const float* bias, void* ws,
                        sl_stream_t stream);
/* Debug: record per-step globaltimer stamps of CTA `cta` of the recurrence
 * kernels into dev_buf[T][8] (NULL disables). */
int sl_debug_set_trace(unsigned long long* dev_buf, int cta);
/* Experiments only (results become wrong): 1 = skip the recurrence MMAs,
 * 2 = skip the recurrence epilogue math/stores. */
int sl_debug_set_flags(int flags);
#ifdef __cplusplus
}
#endif
#endif
