// Internal GEMM entry points (row-major, see gemm_f32.cu / gemm_tc.cu).
#pragma once
#include "common.cuh"

namespace sl {

// FP32 SIMT GEMM: C = alpha*op(A)*op(B) + beta*C + bias.
void gemm_f32(bool transA, bool transB, int M, int N, int K, float alpha, const float* A,
              int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
              const float* bias, cudaStream_t stream);

// fp32-accurate GEMM on the bf16 tensor cores via split-bf16 operands
// (gemm_f32x3.cu): C = op(A) op(B) + beta C + bias.  With ones_row_out, A must be
// stored [K, M] (transA) and the column sums of op(B) (= ones^T op(B)) are also
// written to ones_row_out (+ beta * previous) — the bias gradient for free.
size_t gemm_f32x3_workspace_bytes(bool transA, bool transB, int M, int N, int K, bool a_ones);
// The split image of a stored fp32 matrix S [rows, cols]: bf16 hi [rows, x3_img_ld]
// followed by bf16 lo [rows, x3_img_ld] (padding columns zero).  It does not depend on
// the role the matrix plays in a GEMM (A or B, transposed or not), so one split serves
// every product that reads S.
int64_t x3_img_ld(int cols);
size_t x3_img_elems(int rows, int cols);
void x3_split_img(const float* S, int64_t ld, int rows, int cols, __nv_bfloat16* img, cudaStream_t st);
// the same into a window of a caller's image: hi rows at img (stride img_ld), lo rows
// lo_off elements further on, img_cols (a multiple of 8) columns written per row —
// the columns past `cols` as 0, except ones_col (>= 0): 1 in hi, 0 in lo
void x3_split_into(const float* S, int64_t ld, int rows, int cols, int ones_col, __nv_bfloat16* img, int64_t img_ld,
                   int64_t img_cols, int64_t lo_off, cudaStream_t st);
// B split once for repeated GEMMs (e.g. a weight used every time step): the image of
// the stored B (x3_b_elems elements); gemm_f32x3_pb then splits only A per call (its
// scratch: gemm_f32x3_workspace_bytes of the same shape).
size_t x3_b_elems(bool transB, int N, int K);
void x3_split_b(bool transB, int N, int K, const float* B, int64_t ldb, __nv_bfloat16* B3, cudaStream_t st);
// the general form: each operand either fp32 (split here) or a pre-split image (A3 /
// B3 non-null: the fp32 pointer is then unused).  An image's hi part is at A3 with
// row stride a3_ld and its lo part a3_lo elements further on (0: the x3_split_img
// layout of the stored operand).  With ones_row_out and a pre-split A (stored [K, M]),
// the image must hold the ones column at column M (x3_split_into ones_col = M).
void gemm_f32x3_ex(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda,
                   const __nv_bfloat16* A3, const float* B, int64_t ldb, const __nv_bfloat16* B3, float beta,
                   float* C, int64_t ldc, const float* bias, float* ones_row_out, int64_t ld_ones, void* ws,
                   cudaStream_t st, int64_t a3_ld = 0, int64_t a3_lo = 0, int64_t b3_ld = 0, int64_t b3_lo = 0);
// Split-K partial products for a consumer that sums them itself (fixed order z =
// 0..n-1, the order the reduction kernel uses): op(A) op(B) = sum_z p[z*stride + r*ld + c]
// (no bias / beta).  Saves the reduction launch and its round trip for the small
// per-step products whose consumer is an elementwise kernel anyway.
struct X3Parts {
  const float* p;
  int n;
  int64_t stride, ld;
};
__device__ __forceinline__ float x3_parts_sum(const X3Parts& q, int64_t r, int64_t c) {
  // the first 8 partials' loads all in flight before the (in-order) adds; a partial
  // past n contributes an exact +0
  const float* p = q.p + r * q.ld + c;
  float v[8];
#pragma unroll
  for (int z = 0; z < 8; ++z) v[z] = z < q.n ? __ldg(p + z * q.stride) : 0.f;
  float s = 0.f;
#pragma unroll
  for (int z = 0; z < 8; ++z) s += v[z];
  for (int z = 8; z < q.n; ++z) s += __ldg(p + z * q.stride);
  return s;
}
size_t gemm_f32x3_parts_workspace_bytes(bool transA, bool transB, int M, int N, int K);
X3Parts gemm_f32x3_parts(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda,
                         const __nv_bfloat16* A3, const float* B, int64_t ldb, const __nv_bfloat16* B3, void* ws,
                         cudaStream_t st, int64_t a3_ld = 0, int64_t a3_lo = 0, int64_t b3_ld = 0, int64_t b3_lo = 0);
// C = op(A) op(B) + bias (fp32, single pass) and, per row and 128-column block, the
// online-softmax statistics of C (TcGemm::sm_part) — the output layer's logits; falls
// back to the plain GEMM (returns false, no statistics) where the shape needs split-K
// or chunked accumulation
bool gemm_f32x3_softmax_stats(int M, int N, int K, const float* A, int64_t lda, const float* B, int64_t ldb,
                              float* C, int64_t ldc, const float* bias, float4* sm_part, int sm_ld,
                              const int32_t* targets, void* ws, cudaStream_t st,
                              const __nv_bfloat16* A3 = nullptr, int64_t a3_ld = 0, int64_t a3_lo = 0,
                              const __nv_bfloat16* B3 = nullptr, int64_t b3_ld = 0, int64_t b3_lo = 0);
// both operands pre-split (images of the stored A and B)
void gemm_f32x3_pab(bool transA, bool transB, int M, int N, int K, const __nv_bfloat16* A3,
                    const __nv_bfloat16* B3, float beta, float* C, int64_t ldc, const float* bias, void* ws,
                    cudaStream_t st);
void gemm_f32x3_pb(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda,
                   const __nv_bfloat16* B3, float beta, float* C, int64_t ldc, const float* bias, void* ws,
                   cudaStream_t st, float* ones_row_out = nullptr, int64_t ld_ones = 0);
void gemm_f32x3(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda, const float* B,
                int64_t ldb, float beta, float* C, int64_t ldc, const float* bias, float* ones_row_out,
                int64_t ld_ones, void* ws, cudaStream_t st);

}  // namespace sl

namespace sl {

// BF16 tcgen05 GEMM (gemm_tc.cu): C[M,N] = alpha * op(A) op(B) + beta * C + bias[N], fp32 C.
//   a_mn = false: A stored [M, K] (lda);  a_mn = true: A stored [K, M] (lda)
//   b_mn = false: B stored [N, K] (ldb);  b_mn = true: B stored [K, N] (ldb)
// lda / ldb must be multiples of 8 elements, base pointers 16 B aligned.
struct TcGemm {
  int M, N, K;
  const __nv_bfloat16* A;
  int64_t lda;
  bool a_mn;
  const __nv_bfloat16* B;
  int64_t ldb;
  bool b_mn;
  float* C;
  int64_t ldc;
  float alpha, beta;
  const float* bias;
  // optional: rows >= m_split are written to C2 (row - m_split) instead of C
  // (used to emit db = colsum(DZ) from the ones-column of [X | 1]^T . DZ)
  int m_split = 1 << 30;
  float* C2 = nullptr;
  int64_t ldc2 = 0;
  // optional: write the result as bf16 here (ld = ldc) instead of fp32 C
  __nv_bfloat16* Cb = nullptr;
  // optional (with Cb, pair GEMM only): per row and 128-column block, the online
  // softmax statistics of the (bf16-rounded) outputs — float4 {max, sum exp(z -
  // max), sum z, z[target] if the block holds the row's target else 0} at
  // sm_part[row * sm_ld + col / 128] (softmax_ce.cu)
  float4* sm_part = nullptr;
  int sm_ld = 0;
  const int32_t* sm_targets = nullptr;
  // optional (pair GEMM only): split K into ksplit ranges; range z writes its plain
  // partial product (alpha = 1, no bias / beta / C2) to C + z * split_stride (fp32) or,
  // with Cb, to Cb + z * split_stride (bf16)
  int ksplit = 1;
  int64_t split_stride = 0;
  // optional (pair GEMM, fp32 C only): accumulate K in chunks of kchunk 64-wide blocks —
  // each chunk in a fresh TMEM accumulator, the chunk sums added in fp32 registers by the
  // epilogue (round-to-nearest) — so the tensor core's accumulation error stays at the
  // one-chunk level for any K (gemm_f32x3.cu)
  int kchunk = 0;
  // optional (pair GEMM, fp32 C): fp32-class "x3" mode — A / B above are the bf16 hi
  // parts and these the lo parts (same shape and ld) of split fp32 operands; the GEMM
  // computes A_hi B_hi + A_lo B_hi + A_hi B_lo (gemm_f32x3.cu)
  const __nv_bfloat16* A_lo = nullptr;
  const __nv_bfloat16* B_lo = nullptr;
};
// number of K splits the pair GEMM would use to fill the SMs for this shape
int gemm_tc2_ksplit(int M, int N, int K);
void gemm_bf16_tc(const TcGemm& g, cudaStream_t stream);
// CTA-pair variant (gemm_tc2.cu, M = 256 tiles); gemm_bf16_tc dispatches to it
// when the operands allow (gemm_bf16_tc2_ok) unless SL_GEMM_1CTA is set.
bool gemm_bf16_tc2_ok(const TcGemm& g);
void gemm_bf16_tc2(const TcGemm& g, cudaStream_t stream);
// small-M GEMM on warp-level mma.sync (small_gemm.cu): C[M,N] = A[M,K] op(B) (+ bias),
// A row-major; b_kn: B [K, N] row-major, else B [N, K] row-major; fp32 C, no split
void small_gemm_bf16(int M, int N, int K, const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* B, int64_t ldb,
                     bool b_kn, float* C, int64_t ldc, const float* bias, cudaStream_t st);
// debug: per-CTA timeline stamps of the pair GEMM into buf (null: off)
void gemm_tc2_set_trace(unsigned long long* buf);

}  // namespace sl
