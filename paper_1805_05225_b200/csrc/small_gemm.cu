// Small-M BF16 GEMM for the decoder's per-step projections (s_tr = s W_s and its
// adjoint d s = d s_tr W_s^T: M = batch rows, N = K = 1000): warp-level
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate) from shared-memory tiles.  These
// 0.5 GFLOP GEMMs are bound by fixed costs, not by the tensor pipe: the tcgen05
// pair GEMM spends ~10 us on launch, TMEM / barrier setup and a split-K partial
// epilogue; this kernel has no setup, no split and writes the final fp32 result
// once (128 CTAs of 128 threads; a double-buffered cp.async pipeline over 256-wide K
// tiles — the K loop is latency-bound: few, wide K steps beat many narrow ones:
// 6.3-6.6 us per call against 6.7-7.6 us for 3 x 128-wide, 7.6-7.8 us for 4 x 128-wide
// and 8.1-8.3 us for 6 x 32-wide stages; 3 x 256-wide is no faster).
//   C[M, N] = A[M, K] op(B) (+ bias[N]);  A row-major (lda);
//   b_kn: B stored [K, N] row-major (ldb), else B stored [N, K] row-major (ldb).
// K, lda, ldb multiples of 8 (16 B rows); N arbitrary; fp32 C (ldc).
#include "gemm.h"
#include "profile.h"

namespace sl {
namespace {

constexpr int BM = 32, BN = 64, BK = 256, kThreads = 128;
constexpr int APAD = BK + 8;  // smem row pitch (elements) of the A and [N][K] B tiles: conflict-free ldmatrix
constexpr int BPAD = BN + 8;  // smem row pitch of the [K][N] B tile

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  // 16 B global -> shared, zero-filled when !valid (src-size 0); L2 only (.cg)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kStages = 2;  // K tiles in flight: the K loop is latency-, not compute-bound
constexpr int kAVec = BM * BK / 8 / kThreads;                         // 16 B vectors per thread per A tile
constexpr int kBVec = BN * BK / 8 / kThreads;                         // ... per B tile
constexpr int kSA = BM * APAD, kSBkn = BK * BPAD, kSBnk = BN * APAD;  // elements per stage
template <bool B_KN>
constexpr size_t smem_bytes() { return (size_t)kStages * (kSA + (B_KN ? kSBkn : kSBnk)) * 2; }

template <bool B_KN>
__global__ void __launch_bounds__(kThreads) small_gemm_kernel(int M, int N, int K, const __nv_bfloat16* __restrict__ A,
                                                              int64_t lda, const __nv_bfloat16* __restrict__ Bm,
                                                              int64_t ldb, float* __restrict__ C, int64_t ldc,
                                                              const float* __restrict__ bias) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  constexpr int kSB = B_KN ? kSBkn : kSBnk;
  auto sa = reinterpret_cast<__nv_bfloat16 (*)[kSA]>(smem_raw);
  auto sb = reinterpret_cast<__nv_bfloat16 (*)[kSB]>(smem_raw + (size_t)kStages * kSA * 2);
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  // one K tile: A 32 x 32 (one 16 B vector per thread), B 64 x 32 (two per thread), zero-filled
  // outside the matrix (N must then be a multiple of 8 for [K][N] B: 16 B never straddles N)
  auto issue = [&](int kt, int buf) {
    const int k0 = kt * BK;
#pragma unroll
    for (int v = 0; v < kAVec; ++v) {
      const int i = tid + v * kThreads;
      const int r = i / (BK / 8), c = (i % (BK / 8)) * 8, gr = m0 + r, gk = k0 + c;
      const bool ok = gr < M && gk < K;
      cp_async16(&sa[buf][r * APAD + c], ok ? A + (int64_t)gr * lda + gk : A, ok);
    }
#pragma unroll
    for (int v = 0; v < kBVec; ++v) {
      const int i = tid + v * kThreads;
      if constexpr (B_KN) {
        const int r = i / (BN / 8), c = (i % (BN / 8)) * 8, gk = k0 + r, gn = n0 + c;
        const bool ok = gk < K && gn < N;
        cp_async16(&sb[buf][r * BPAD + c], ok ? Bm + (int64_t)gk * ldb + gn : Bm, ok);
      } else {
        const int r = i / (BK / 8), c = (i % (BK / 8)) * 8, gn = n0 + r, gk = k0 + c;
        const bool ok = gn < N && gk < K;
        cp_async16(&sb[buf][r * APAD + c], ok ? Bm + (int64_t)gn * ldb + gk : Bm, ok);
      }
    }
  };
  float acc[2][2][4];  // [m16 tile][n8 tile][4]: the warp owns rows 0..31, columns 16 warp .. +16
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.f;
  const int nkt = (K + BK - 1) / BK;
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < nkt) issue(st, st);
    cp_async_commit();
  }
  for (int kt = 0; kt < nkt; ++kt) {
    const int buf = kt % kStages;
    cp_async_wait<kStages - 2>();  // tile kt landed (this thread's copies) ...
    __syncthreads();               // ... and everyone's; the slot refilled below was read last iteration
    if (kt + kStages - 1 < nkt) issue(kt + kStages - 1, (kt + kStages - 1) % kStages);
    cp_async_commit();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 16) {
      uint32_t af[2][4], bf[2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {  // A 16 x 16 fragments (rows 16 i .., k kk ..)
        const __nv_bfloat16* p = &sa[buf][(16 * i + (lane % 16)) * APAD + kk + (lane / 16) * 8];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(af[i][0]), "=r"(af[i][1]), "=r"(af[i][2]), "=r"(af[i][3])
                     : "r"(smem_addr(p)));
      }
      if constexpr (B_KN) {  // B 16 x 8 fragments from [K][N] rows (transposed load)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const __nv_bfloat16* p = &sb[buf][(kk + (lane % 16)) * BPAD + warp * 16 + j * 8];
          asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                       : "=r"(bf[j][0]), "=r"(bf[j][1])
                       : "r"(smem_addr(p)));
        }
      } else {  // from [N][K] rows
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const __nv_bfloat16* p = &sb[buf][(warp * 16 + j * 8 + (lane % 8)) * APAD + kk + ((lane / 8) % 2) * 8];
          asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
                       : "=r"(bf[j][0]), "=r"(bf[j][1])
                       : "r"(smem_addr(p)));
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          asm volatile(
              "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
              "{%8, %9}, {%0, %1, %2, %3};"
              : "+f"(acc[i][j][0]), "+f"(acc[i][j][1]), "+f"(acc[i][j][2]), "+f"(acc[i][j][3])
              : "r"(af[i][0]), "r"(af[i][1]), "r"(af[i][2]), "r"(af[i][3]), "r"(bf[j][0]), "r"(bf[j][1]));
    }
  }
  cp_async_wait<0>();
  // C fragment: c0, c1 at (row g, cols 2t, 2t+1), c2, c3 at (row g + 8, ...)
  const int g = lane / 4, t = lane % 4;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = n0 + warp * 16 + j * 8 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = m0 + 16 * i + g + 8 * h;
        if (row >= M) continue;
        float v0 = acc[i][j][2 * h], v1 = acc[i][j][2 * h + 1];
        if (bias) {
          if (col < N) v0 += bias[col];
          if (col + 1 < N) v1 += bias[col + 1];
        }
        float* dst = C + (int64_t)row * ldc + col;
        if (col + 1 < N && ((ldc % 2) == 0)) {
          *reinterpret_cast<float2*>(dst) = make_float2(v0, v1);
        } else {
          if (col < N) dst[0] = v0;
          if (col + 1 < N) dst[1] = v1;
        }
      }
    }
}

}  // namespace

void small_gemm_bf16(int M, int N, int K, const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* B, int64_t ldb,
                     bool b_kn, float* C, int64_t ldc, const float* bias, cudaStream_t st) {
  SL_REQUIRE(K % 8 == 0 && lda % 8 == 0 && ldb % 8 == 0 && ((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0 &&
                 (!b_kn || N % 8 == 0),
             SL_ERR_INVALID_ARGUMENT,
             "small_gemm_bf16: K, lda, ldb (and N for a [K, N] B) multiples of 8, 16 B aligned operands");
  if (M <= 0 || N <= 0) return;
  static bool configured = false;  // > 48 KB dynamic shared memory needs the opt-in, once per process
  if (!configured) {
    SL_CUDA_TRY(cudaFuncSetAttribute(small_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_bytes<true>()));
    SL_CUDA_TRY(cudaFuncSetAttribute(small_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_bytes<false>()));
    configured = true;
  }
  const dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM));
  if (b_kn)
    small_gemm_kernel<true><<<grid, kThreads, smem_bytes<true>(), st>>>(M, N, K, A, lda, B, ldb, C, ldc, bias);
  else
    small_gemm_kernel<false><<<grid, kThreads, smem_bytes<false>(), st>>>(M, N, K, A, lda, B, ldb, C, ldc, bias);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace sl
