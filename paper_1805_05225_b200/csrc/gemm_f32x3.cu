// fp32-accurate GEMM on the bf16 tensor cores (split-bf16, "3 x bf16"):
//   x = x_hi + x_lo with x_hi = bf16(x), x_lo = bf16(x - x_hi)  (|x_lo| <= 2^-9 |x|)
//   A B ~= A_hi B_hi + A_lo B_hi + A_hi B_lo          (dropped A_lo B_lo ~ 2^-18)
// Each operand is split once into its image (hi and lo bf16 matrices of the stored
// shape); the pair GEMM's x3 mode (gemm_tc2.cu) loads A_hi, A_lo, B_hi, B_lo per
// 64-wide K block and issues the three products into one fp32 TMEM accumulator —
// relative error ~1e-5, i.e. fp32-class for the tolerances the reference's fp32 CPU
// path is held to, at tensor-core speed.
#include <algorithm>

#include "convert.h"
#include "gemm.h"
#include "profile.h"

namespace sl {
namespace {

__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// S [rows, cols] (ld) -> hi rows at D (stride dld) and lo rows lo_off elements further
// on; the first dcols (a multiple of 8) columns of each row are written, columns >= cols
// as 0 except ones_col (if >= 0): 1 (hi) / 0 (lo).  Eight columns per thread (16 B
// stores), grid-stride over rows.
template <bool V4, bool A16>
__global__ void split2_kernel(const float* __restrict__ S, int64_t ld, int rows, int cols, int ones_col,
                              __nv_bfloat16* __restrict__ D, int64_t dld, int64_t dcols, int64_t lo_off) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= dcols) return;
  __nv_bfloat16* lo_base = D + lo_off;
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {  // (grid y is capped at 65535)
    const float* src = S + (int64_t)r * ld;
    float x[8];
    if (V4 && c + 8 <= cols) {
      const float4 q0 = __ldg(reinterpret_cast<const float4*>(src + c));
      const float4 q1 = __ldg(reinterpret_cast<const float4*>(src + c + 4));
      x[0] = q0.x, x[1] = q0.y, x[2] = q0.z, x[3] = q0.w, x[4] = q1.x, x[5] = q1.y, x[6] = q1.z, x[7] = q1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t cc = c + i;
        x[i] = cc < cols ? src[cc] : 0.f;
      }
    }
    __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split_bf16(x[i], h[i], l[i]);
    if (ones_col >= c && ones_col < c + 8) {
      h[ones_col - c] = __float2bfloat16_rn(1.f);
      l[ones_col - c] = __float2bfloat16_rn(0.f);
    }
    if (A16) {
      *reinterpret_cast<uint4*>(D + (int64_t)r * dld + c) = *reinterpret_cast<const uint4*>(h);
      *reinterpret_cast<uint4*>(lo_base + (int64_t)r * dld + c) = *reinterpret_cast<const uint4*>(l);
    } else {  // a window at an unaligned column offset
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (c + i < dcols) D[(int64_t)r * dld + c + i] = h[i], lo_base[(int64_t)r * dld + c + i] = l[i];
    }
  }
}

// C[m, n] = sum_z P[z][m, n] (fixed order: deterministic) + bias[n] + beta C[m, n]; rows >= m_split -> C2
__global__ void splitk_reduce_kernel(const float* __restrict__ P, int S, int64_t pstride, int64_t pld, int M, int N,
                                     float beta, float* C, int64_t ldc, const float* __restrict__ bias, int m_split,
                                     float* C2, int64_t ldc2) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  for (int m = blockIdx.y; m < M; m += gridDim.y) {  // (grid y is capped at 65535)
  const float* src = P + (int64_t)m * pld + n;
  float s = 0.f;
#pragma unroll 4
  for (int z = 0; z < S; ++z) s += __ldg(src + z * pstride);
  if (bias) s += bias[n];
  float* dst = m >= m_split ? C2 + (int64_t)(m - m_split) * ldc2 + n : C + (int64_t)m * ldc + n;
  if (beta != 0.f) s += beta * *dst;
  *dst = s;
  }
}

// the same for 4 consecutive columns per thread (16 B aligned), the first 8 partials'
// loads in flight before the in-order adds
__global__ void splitk_reduce4_kernel(const float* __restrict__ P, int S, int64_t pstride, int64_t pld, int M, int N,
                                      float beta, float* C, int64_t ldc, const float* __restrict__ bias, int m_split,
                                      float* C2, int64_t ldc2) {
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (n >= N) return;
  for (int m = blockIdx.y; m < M; m += gridDim.y) {
    const float* src = P + (int64_t)m * pld + n;
    float4 v[8];
#pragma unroll
    for (int z = 0; z < 8; ++z)
      v[z] = z < S ? __ldg(reinterpret_cast<const float4*>(src + z * pstride)) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int z = 0; z < 8; ++z) s.x += v[z].x, s.y += v[z].y, s.z += v[z].z, s.w += v[z].w;
    for (int z = 8; z < S; ++z) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(src + z * pstride));
      s.x += t.x, s.y += t.y, s.z += t.z, s.w += t.w;
    }
    if (bias) {
      const float4 b = *reinterpret_cast<const float4*>(bias + n);
      s.x += b.x, s.y += b.y, s.z += b.z, s.w += b.w;
    }
    float* dst = m >= m_split ? C2 + (int64_t)(m - m_split) * ldc2 + n : C + (int64_t)m * ldc + n;
    if (beta != 0.f) {
      const float4 o = *reinterpret_cast<const float4*>(dst);
      s.x += beta * o.x, s.y += beta * o.y, s.z += beta * o.z, s.w += beta * o.w;
    }
    *reinterpret_cast<float4*>(dst) = s;
  }
}

constexpr int kX3ChunkBlocks = 16;  // K blocks (of 64, three products each) per tensor-core accumulation chunk

int sm_count_x3() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 148;
  }
  return n;
}

struct X3Dims {
  int64_t a_rows, a_cols, b_rows, b_cols;  // stored operands (a_cols includes the ones column)
  int ksplit;
  int64_t p_ld, p_stride;  // split-K partials [ksplit][M (+1)][p_ld] fp32
};

X3Dims x3_dims(bool transA, bool transB, int M, int N, int K, bool a_ones) {
  X3Dims d;
  const int Mt = M + (a_ones ? 1 : 0);
  // A stored [M, K] (op(A) = A) or [K, M (+ ones column)] (op(A) = A^T); B stored [K, N] or [N, K]
  if (!transA) d.a_rows = M, d.a_cols = K;
  else d.a_rows = K, d.a_cols = Mt;
  if (!transB) d.b_rows = K, d.b_cols = N;
  else d.b_rows = N, d.b_cols = K;
  // The tensor core's fp32 accumulation is not round-to-nearest: its error grows
  // linearly with the number of accumulated K steps (measured, scripts/x3_accuracy.py:
  // ~3e-5 relative at K = 4096, ~1e-4 at 20000, ~3e-4 at 60000 products deep).  The
  // GEMM therefore accumulates K in chunks of kX3ChunkBlocks 64-wide blocks, each in a
  // fresh TMEM accumulator, and sums the chunks in fp32 registers (round-to-nearest)
  // in its epilogue (TcGemm::kchunk): the error stays at the one-chunk level for any K.
  // Split-K (fp32 partials + a fixed-order reduction) only for outputs with fewer
  // 256 x 256 tiles than CTA pairs (e.g. the decoder's per-step M = batch products):
  // enough K ranges to occupy the pairs, >= 2 K blocks each.
  {
    const int tiles = (int)(ceil_div(Mt, 256) * ceil_div(N, 256));
    const int pairs = std::max(1, sm_count_x3() / 2);
    const int nk = (int)ceil_div(K, 64);
    int ks = 1;
    if (tiles < pairs) ks = std::max(1, std::min(pairs / tiles, nk / 2));
    d.ksplit = (int)ceil_div(nk, ceil_div(nk, ks));  // the count the pair GEMM runs (no empty ranges)
  }
  d.p_ld = round_up(N, 4);
  d.p_stride = round_up((int64_t)Mt * d.p_ld, 64);
  return d;
}

void split_into(const float* S, int64_t ld, int rows, int cols, int ones_col, __nv_bfloat16* D, int64_t dld,
                int64_t dcols, int64_t lo_off, cudaStream_t st) {
  if (rows <= 0) return;
  const dim3 grid((unsigned)ceil_div(dcols, 8 * 128), (unsigned)std::min(rows, 65535));
  const bool v4 = (ld % 4) == 0 && ((uintptr_t)S & 15) == 0;
  const bool a16 = dcols % 8 == 0 && dld % 8 == 0 && lo_off % 8 == 0 && ((uintptr_t)D & 15) == 0;
  if (v4 && a16) split2_kernel<true, true><<<grid, 128, 0, st>>>(S, ld, rows, cols, ones_col, D, dld, dcols, lo_off);
  else if (a16) split2_kernel<false, true><<<grid, 128, 0, st>>>(S, ld, rows, cols, ones_col, D, dld, dcols, lo_off);
  else split2_kernel<false, false><<<grid, 128, 0, st>>>(S, ld, rows, cols, ones_col, D, dld, dcols, lo_off);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}
void split_img(const float* S, int64_t ld, int rows, int cols, int ones_col, __nv_bfloat16* D, cudaStream_t st) {
  const int64_t dld = x3_img_ld(cols + (ones_col >= 0 ? 1 : 0));
  split_into(S, ld, rows, cols, ones_col, D, dld, dld, (int64_t)rows * dld, st);
}

}  // namespace

int64_t x3_img_ld(int cols) { return round_up((int64_t)cols, 64); }
size_t x3_img_elems(int rows, int cols) { return (size_t)2 * rows * x3_img_ld(cols); }
void x3_split_img(const float* S, int64_t ld, int rows, int cols, __nv_bfloat16* img, cudaStream_t st) {
  split_img(S, ld, rows, cols, -1, img, st);
}
void x3_split_into(const float* S, int64_t ld, int rows, int cols, int ones_col, __nv_bfloat16* img, int64_t img_ld,
                   int64_t img_cols, int64_t lo_off, cudaStream_t st) {
  split_into(S, ld, rows, cols, ones_col, img, img_ld, img_cols, lo_off, st);
}

size_t gemm_f32x3_workspace_bytes(bool transA, bool transB, int M, int N, int K, bool a_ones) {
  const X3Dims d = x3_dims(transA, transB, M, N, K, a_ones);
  return round_up(x3_img_elems((int)d.a_rows, (int)d.a_cols) * 2, 256) +
         round_up(x3_img_elems((int)d.b_rows, (int)d.b_cols) * 2, 256) +
         (d.ksplit > 1 ? (size_t)d.ksplit * d.p_stride * 4 : 0);
}

size_t x3_b_elems(bool transB, int N, int K) {
  return transB ? x3_img_elems(N, K) : x3_img_elems(K, N);
}

void x3_split_b(bool transB, int N, int K, const float* B, int64_t ldb, __nv_bfloat16* B3, cudaStream_t st) {
  if (!transB) split_img(B, ldb, K, N, -1, B3, st);
  else split_img(B, ldb, N, K, -1, B3, st);
}

namespace {
// the GEMM over split operands: each image from the caller (a_pre / b_pre) or split
// here into the scratch
void x3_core(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda,
             const __nv_bfloat16* a_pre, const float* B, int64_t ldb, const __nv_bfloat16* b_pre, float beta,
             float* C, int64_t ldc, const float* bias, float* ones_row_out, int64_t ld_ones, void* ws,
             cudaStream_t st, int64_t a3_ld = 0, int64_t a3_lo = 0, int64_t b3_ld = 0, int64_t b3_lo = 0,
             X3Parts* parts = nullptr, const TcGemm* smx = nullptr) {
  if (M <= 0 || N <= 0) return;
  const bool a_ones = ones_row_out != nullptr;
  SL_REQUIRE(!a_ones || transA, SL_ERR_INVALID_ARGUMENT, "gemm_f32x3: ones row needs A stored [K, M]");

  const X3Dims d = x3_dims(transA, transB, M, N, K, a_ones);
  char* w = static_cast<char*>(ws);
  const __nv_bfloat16* a3 = a_pre;
  if (!a3) {
    auto* a3w = reinterpret_cast<__nv_bfloat16*>(w);
    split_img(A, lda, (int)d.a_rows, transA ? M : K, a_ones ? M : -1, a3w, st);
    a3 = a3w;
  }
  w += round_up(x3_img_elems((int)d.a_rows, (int)d.a_cols) * 2, 256);
  const __nv_bfloat16* b3 = b_pre;
  if (!b3) {
    auto* b3w = reinterpret_cast<__nv_bfloat16*>(w);
    split_img(B, ldb, (int)d.b_rows, (int)d.b_cols, -1, b3w, st);
    b3 = b3w;
  }
  w += round_up(x3_img_elems((int)d.b_rows, (int)d.b_cols) * 2, 256);
  // (a caller's image may carry its own stride and lo offset)
  const int64_t a_ld = a_pre && a3_ld ? a3_ld : x3_img_ld((int)d.a_cols);
  const int64_t b_ld = b_pre && b3_ld ? b3_ld : x3_img_ld((int)d.b_cols);
  TcGemm g{M + (a_ones ? 1 : 0), N, K, a3, a_ld, transA, b3, b_ld, !transB, C, ldc, 1.f, beta, bias};
  g.A_lo = a3 + (a_pre && a3_lo ? a3_lo : d.a_rows * a_ld);
  g.B_lo = b3 + (b_pre && b3_lo ? b3_lo : d.b_rows * b_ld);
  {  // chunked accumulation only where one work unit's K range is longer than a chunk
    const int64_t nk = ceil_div(K, 64);
    if (ceil_div(nk, d.ksplit) > kX3ChunkBlocks) g.kchunk = kX3ChunkBlocks;
  }
  if (smx) {  // softmax statistics in the epilogue (single pass only: the caller checked)
    g.sm_part = smx->sm_part;
    g.sm_ld = smx->sm_ld;
    g.sm_targets = smx->sm_targets;
  }
  if (parts) {  // the partials for the caller's consumer (ksplit may be 1)
    SL_REQUIRE(!a_ones && beta == 0.f && !bias, SL_ERR_INVALID_ARGUMENT, "gemm_f32x3: partials are plain products");
    float* part = reinterpret_cast<float*>(w);
    g.C = part;
    g.ldc = d.p_ld;
    g.ksplit = d.ksplit;
    g.split_stride = d.p_stride;
    gemm_bf16_tc(g, st);
    *parts = X3Parts{part, d.ksplit, d.p_stride, d.p_ld};
    return;
  }
  if (d.ksplit > 1) {  // small output: split K over the idle SMs, then a fixed-order reduction
    float* part = reinterpret_cast<float*>(w);
    g.C = part;
    g.ldc = d.p_ld;
    g.beta = 0.f;
    g.bias = nullptr;
    g.ksplit = d.ksplit;
    g.split_stride = d.p_stride;
    gemm_bf16_tc(g, st);
    const int Mt = M + (a_ones ? 1 : 0);
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    const bool v4 = N % 4 == 0 && d.p_ld % 4 == 0 && d.p_stride % 4 == 0 && ldc % 4 == 0 && al16(part) && al16(C) &&
                    (!bias || al16(bias)) && (!a_ones || (ld_ones % 4 == 0 && al16(ones_row_out)));
    if (v4)
      splitk_reduce4_kernel<<<dim3((unsigned)ceil_div(N / 4, 256), (unsigned)std::min(Mt, 65535)), 256, 0, st>>>(
          part, d.ksplit, d.p_stride, d.p_ld, Mt, N, beta, C, ldc, bias, a_ones ? M : (1 << 30), ones_row_out,
          ld_ones);
    else
      splitk_reduce_kernel<<<dim3((unsigned)ceil_div(N, 256), (unsigned)std::min(Mt, 65535)), 256, 0, st>>>(
          part, d.ksplit, d.p_stride, d.p_ld, Mt, N, beta, C, ldc, bias, a_ones ? M : (1 << 30), ones_row_out,
          ld_ones);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
    return;
  }
  if (a_ones) {
    g.m_split = M;
    g.C2 = ones_row_out;
    g.ldc2 = ld_ones;
  }
  gemm_bf16_tc(g, st);
}
}  // namespace

void gemm_f32x3(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda, const float* B,
                int64_t ldb, float beta, float* C, int64_t ldc, const float* bias, float* ones_row_out,
                int64_t ld_ones, void* ws, cudaStream_t st) {
  x3_core(transA, transB, M, N, K, A, lda, nullptr, B, ldb, nullptr, beta, C, ldc, bias, ones_row_out, ld_ones, ws,
          st);
}

void gemm_f32x3_pb(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda,
                   const __nv_bfloat16* B3, float beta, float* C, int64_t ldc, const float* bias, void* ws,
                   cudaStream_t st, float* ones_row_out, int64_t ld_ones) {
  x3_core(transA, transB, M, N, K, A, lda, nullptr, nullptr, 0, B3, beta, C, ldc, bias, ones_row_out, ld_ones, ws,
          st);
}

void gemm_f32x3_ex(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda,
                   const __nv_bfloat16* A3, const float* B, int64_t ldb, const __nv_bfloat16* B3, float beta,
                   float* C, int64_t ldc, const float* bias, float* ones_row_out, int64_t ld_ones, void* ws,
                   cudaStream_t st, int64_t a3_ld, int64_t a3_lo, int64_t b3_ld, int64_t b3_lo) {
  x3_core(transA, transB, M, N, K, A, lda, A3, B, ldb, B3, beta, C, ldc, bias, ones_row_out, ld_ones, ws, st, a3_ld,
          a3_lo, b3_ld, b3_lo);
}

size_t gemm_f32x3_parts_workspace_bytes(bool transA, bool transB, int M, int N, int K) {
  const X3Dims d = x3_dims(transA, transB, M, N, K, false);
  return round_up(x3_img_elems((int)d.a_rows, (int)d.a_cols) * 2, 256) +
         round_up(x3_img_elems((int)d.b_rows, (int)d.b_cols) * 2, 256) + (size_t)d.ksplit * d.p_stride * 4;
}

X3Parts gemm_f32x3_parts(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda,
                         const __nv_bfloat16* A3, const float* B, int64_t ldb, const __nv_bfloat16* B3, void* ws,
                         cudaStream_t st, int64_t a3_ld, int64_t a3_lo, int64_t b3_ld, int64_t b3_lo) {
  X3Parts q{nullptr, 0, 0, 0};
  x3_core(transA, transB, M, N, K, A, lda, A3, B, ldb, B3, 0.f, nullptr, 0, nullptr, nullptr, 0, ws, st, a3_ld,
          a3_lo, b3_ld, b3_lo, &q);
  return q;
}

bool gemm_f32x3_softmax_stats(int M, int N, int K, const float* A, int64_t lda, const float* B, int64_t ldb,
                              float* C, int64_t ldc, const float* bias, float4* sm_part, int sm_ld,
                              const int32_t* targets, void* ws, cudaStream_t st, const __nv_bfloat16* A3,
                              int64_t a3_ld, int64_t a3_lo, const __nv_bfloat16* B3, int64_t b3_ld, int64_t b3_lo) {
  const X3Dims d = x3_dims(false, false, M, N, K, false);
  const bool single = d.ksplit == 1 && ceil_div(K, 64) <= kX3ChunkBlocks;
  TcGemm sm{};
  sm.sm_part = sm_part;
  sm.sm_ld = sm_ld;
  sm.sm_targets = targets;
  x3_core(false, false, M, N, K, A, lda, A3, B, ldb, B3, 0.f, C, ldc, bias, nullptr, 0, ws, st, a3_ld, a3_lo, b3_ld,
          b3_lo, nullptr, single ? &sm : nullptr);
  return single;
}

void gemm_f32x3_pab(bool transA, bool transB, int M, int N, int K, const __nv_bfloat16* A3,
                    const __nv_bfloat16* B3, float beta, float* C, int64_t ldc, const float* bias, void* ws,
                    cudaStream_t st) {
  x3_core(transA, transB, M, N, K, nullptr, 0, A3, nullptr, 0, B3, beta, C, ldc, bias, nullptr, 0, ws, st);
}

}  // namespace sl
