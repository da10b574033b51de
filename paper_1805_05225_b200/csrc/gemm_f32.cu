// FP32-exact GEMM used by the SL_PREC_FP32 path (the 1e-4 parity mode) for the
// hoisted input projection (K1) and the hoisted weight/input-gradient GEMMs
// (K4).  It replaces the reference's per-step Eigen products
// (tape.cpp:1103, 1174-1203) with ONE product over all B*T rows.
//
// Row-major: C[M,N] = alpha * op(A) * op(B) + beta * C + bias[N]
//   op(A) = A [M,K] (lda)   or A^T with A stored [K,M]
//   op(B) = B [K,N] (ldb)   or B^T with B stored [N,K]
// Classic 128x128x16 register-tiled SIMT kernel: 256 threads, 8x8 outputs
// per thread, double-buffered shared tiles stored K-major so the inner loop
// reads float4 fragments of both operands.
#include "gemm.h"
#include "profile.h"

namespace sl {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, TM = 8, TN = 8, NT = 256;

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_f32_kernel(int M, int N, int K, float alpha,
                                                      const float* __restrict__ A, int64_t lda,
                                                      const float* __restrict__ B, int64_t ldb,
                                                      float beta, float* __restrict__ C,
                                                      int64_t ldc,
                                                      const float* __restrict__ bias) {
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tr = tid / 16, tc = tid % 16;  // 16x16 thread grid, 8x8 each

  auto load = [&](int buf, int k0) {
    // A tile: BM x BK = 2048 elems, 8 per thread
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int e = tid + i * NT;
      int mm, kk;
      if (TA) {  // stored [K, M]: consecutive threads along M
        mm = e % BM;
        kk = e / BM;
      } else {  // stored [M, K]: consecutive threads along K
        kk = e % BK;
        mm = e / BK;
      }
      int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < K) v = TA ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk];
      As[buf][kk][mm] = v;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int e = tid + i * NT;
      int nn, kk;
      if (TB) {  // stored [N, K]
        kk = e % BK;
        nn = e / BK;
      } else {  // stored [K, N]
        nn = e % BN;
        kk = e / BN;
      }
      int gn = n0 + nn, gk = k0 + kk;
      float v = 0.f;
      if (gn < N && gk < K) v = TB ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn];
      Bs[buf][kk][nn] = v;
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  const int nk = (K + BK - 1) / BK;
  load(0, 0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) load(cur ^ 1, (kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
      float4 a0 = *reinterpret_cast<const float4*>(&As[cur][kk][tr * 4]);
      float4 a1 = *reinterpret_cast<const float4*>(&As[cur][kk][64 + tr * 4]);
      float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][kk][tc * 4]);
      float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][kk][64 + tc * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int gm = m0 + (i < 4 ? tr * 4 + i : 64 + tr * 4 + (i - 4));
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int gn = n0 + (j < 4 ? tc * 4 + j : 64 + tc * 4 + (j - 4));
      if (gn >= N) continue;
      float v = alpha * acc[i][j];
      if (bias) v += bias[gn];
      float* c = C + (int64_t)gm * ldc + gn;
      *c = beta == 0.f ? v : v + beta * *c;
    }
  }
}

}  // namespace

void gemm_f32(bool transA, bool transB, int M, int N, int K, float alpha, const float* A,
              int64_t lda, const float* B, int64_t ldb, float beta, float* C, int64_t ldc,
              const float* bias, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM));
#define SL_GEMM_LAUNCH(ta, tb) \
  gemm_f32_kernel<ta, tb><<<grid, NT, 0, stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, bias)
  if (!transA && !transB) SL_GEMM_LAUNCH(false, false);
  else if (!transA && transB) SL_GEMM_LAUNCH(false, true);
  else if (transA && !transB) SL_GEMM_LAUNCH(true, false);
  else SL_GEMM_LAUNCH(true, true);
#undef SL_GEMM_LAUNCH
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace sl
