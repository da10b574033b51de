// fp32-accurate GEMM on the bf16 tensor cores (split-bf16, "3 x bf16"):
//   x = x_hi + x_lo with x_hi = bf16(x), x_lo = bf16(x - x_hi)  (|x_lo| <= 2^-9 |x|)
//   A B ~= A_hi B_hi + A_lo B_hi + A_hi B_lo          (dropped A_lo B_lo ~ 2^-18)
// computed as ONE tcgen05 GEMM over a K dimension tripled by concatenation,
//   [A_hi | A_lo | A_hi] . [B_hi ; B_hi ; B_lo]
// with fp32 accumulation in TMEM — relative error ~1e-5, i.e. fp32-class for
// the tolerances the reference's fp32 CPU path is held to, at tensor-core
// speed.  Used where a small fp32 GEMM would otherwise leave most SMs idle on
// the SIMT path (the attention step's s W_s projections: M = batch).
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

// S [rows, cols] (ld) -> three copies along the K dimension (k_cols: K = cols, else K = rows),
// each copy padded to Kp with zeros; copy i holds hi unless lo_mask bit i is set.
// ones_col >= 0 (K = rows only): that column is 1 (hi) / 0 (lo) for k < K.
// One CTA row per (extended) source row, two contiguous columns per thread.
__global__ void split3_kernel(const float* __restrict__ S, int64_t ld, int rows, int cols, bool k_cols, int Kp,
                              int lo_mask, int ones_col, __nv_bfloat16* __restrict__ D, int64_t dld, int rows_ext) {
  for (int r = blockIdx.y; r < rows_ext; r += gridDim.y) {  // (grid y is capped at 65535)
  const int cols_ext = k_cols ? Kp : cols + (ones_col >= 0 ? 1 : 0);
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (c >= cols_ext) continue;
  float x[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int cc = c + i;
    x[i] = 0.f;
    if (r < rows && cc < cols) x[i] = S[(int64_t)r * ld + cc];
    else if (r < rows && cc == ones_col) x[i] = 1.f;
  }
  __nv_bfloat16 hi[2], lo[2];
  split_bf16(x[0], hi[0], lo[0]);
  split_bf16(x[1], hi[1], lo[1]);
  const bool pair = c + 1 < cols_ext;
#pragma unroll
  for (int copy = 0; copy < 3; ++copy) {
    const bool use_lo = (lo_mask >> copy) & 1;
    __nv_bfloat16* dst = k_cols ? D + (int64_t)r * dld + copy * Kp + c : D + (int64_t)(copy * Kp + r) * dld + c;
    if (pair) {
      __nv_bfloat162 v;
      v.x = use_lo ? lo[0] : hi[0];
      v.y = use_lo ? lo[1] : hi[1];
      *reinterpret_cast<__nv_bfloat162*>(dst) = v;
    } else {
      *dst = use_lo ? lo[0] : hi[0];
    }
  }
  }
}

// The same split, 8 contiguous columns per thread: two 16 B loads, three 16 B stores
// (every row and the ld's 16 B aligned, cols_ext % 8 == 0 handled by the caller).
__global__ void split3_v8_kernel(const float* __restrict__ S, int64_t ld, int rows, int cols, bool k_cols, int Kp,
                                 int lo_mask, int ones_col, __nv_bfloat16* __restrict__ D, int64_t dld,
                                 int rows_ext, int cols_ext) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= cols_ext) return;
  for (int r = blockIdx.y; r < rows_ext; r += gridDim.y) {
    float x[8];
    if (r < rows && c + 8 <= cols) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(S + (int64_t)r * ld + c));
      const float4 b = __ldg(reinterpret_cast<const float4*>(S + (int64_t)r * ld + c + 4));
      x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int cc = c + i;
        x[i] = (r < rows && cc < cols) ? S[(int64_t)r * ld + cc] : (r < rows && cc == ones_col) ? 1.f : 0.f;
      }
    }
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat16 h0, l0, h1, l1;
      split_bf16(x[2 * i], h0, l0);
      split_bf16(x[2 * i + 1], h1, l1);
      __nv_bfloat162 hh, ll;
      hh.x = h0, hh.y = h1, ll.x = l0, ll.y = l1;
      hi[i] = *reinterpret_cast<uint32_t*>(&hh);
      lo[i] = *reinterpret_cast<uint32_t*>(&ll);
    }
    const uint4 vh = make_uint4(hi[0], hi[1], hi[2], hi[3]), vl = make_uint4(lo[0], lo[1], lo[2], lo[3]);
#pragma unroll
    for (int copy = 0; copy < 3; ++copy) {
      __nv_bfloat16* dst = k_cols ? D + (int64_t)r * dld + copy * Kp + c : D + (int64_t)(copy * Kp + r) * dld + c;
      *reinterpret_cast<uint4*>(dst) = ((lo_mask >> copy) & 1) ? vl : vh;
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

constexpr int kX3ChunkBlocks = 48;  // K blocks (of 64) per tensor-core accumulation chunk

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
  int Kp;
  int64_t a_rows, a_ld, b_rows, b_ld;  // stored bf16 operands
  int ksplit;
  int64_t p_ld, p_stride;  // split-K partials [ksplit][M (+1)][p_ld] fp32
};

X3Dims x3_dims(bool transA, bool transB, int M, int N, int K, bool a_ones) {
  X3Dims d;
  d.Kp = (int)round_up(K, 8);
  // A: op(A) = A [M, K] -> K along columns; op(A) = A^T (A stored [K, M]) -> K along rows
  if (!transA) d.a_rows = M, d.a_ld = 3 * (int64_t)d.Kp;
  else d.a_rows = 3 * (int64_t)d.Kp, d.a_ld = round_up(M + (a_ones ? 1 : 0), 64);
  // B: op(B) = B stored [K, N] -> K along rows; op(B) = B^T (B stored [N, K]) -> K along columns
  if (!transB) d.b_rows = 3 * (int64_t)d.Kp, d.b_ld = round_up(N, 64);
  else d.b_rows = N, d.b_ld = 3 * (int64_t)d.Kp;
  const int Mt = M + (a_ones ? 1 : 0);
  // The tensor core's fp32 accumulation is not round-to-nearest: its error grows
  // linearly with the number of accumulated K steps (measured, scripts/x3_accuracy.py:
  // ~3e-5 relative at K = 4096, ~1e-4 at 20000, ~3e-4 at 60000).  The GEMM therefore
  // accumulates K in chunks of kX3ChunkBlocks 64-wide blocks, each in a fresh TMEM
  // accumulator, and sums the chunks in fp32 registers (round-to-nearest) in its
  // epilogue (TcGemm::kchunk): the error stays at the one-chunk level for any K.
  // Split-K (fp32 partials + a fixed-order reduction) only for outputs with fewer
  // 256 x 256 tiles than CTA pairs (e.g. the decoder's per-step M = batch products):
  // enough K ranges to occupy the pairs, >= 4 K blocks each.
  {
    const int tiles = (int)(ceil_div(Mt, 256) * ceil_div(N, 256));
    const int pairs = std::max(1, sm_count_x3() / 2);
    const int nk = (int)ceil_div(3 * (int64_t)d.Kp, 64);
    int ks = 1;
    if (tiles < pairs) ks = std::max(1, std::min(pairs / tiles, nk / 4));
    d.ksplit = (int)ceil_div(nk, ceil_div(nk, ks));  // the count the pair GEMM runs (no empty ranges)
  }
  d.p_ld = round_up(N, 4);
  d.p_stride = round_up((int64_t)Mt * d.p_ld, 64);
  return d;
}

void split3(const float* S, int64_t ld, int rows, int cols, bool k_cols, int Kp, int lo_mask, int ones_col,
            __nv_bfloat16* D, int64_t dld, cudaStream_t st) {
  const int rows_ext = k_cols ? rows : Kp;
  const int cols_ext = k_cols ? Kp : cols + (ones_col >= 0 ? 1 : 0);
  // (the image's row padding up to the next multiple of 8 columns is written as zeros)
  const int cols_v8 = (int)round_up(cols_ext, 8);
  const bool v8 = cols_v8 <= (k_cols ? Kp : dld) && (ld % 4) == 0 && (dld % 8) == 0 && (Kp % 8) == 0 &&
                  ((uintptr_t)S & 15) == 0 && ((uintptr_t)D & 15) == 0;
  if (v8) {
    const dim3 grid((unsigned)ceil_div(cols_v8, 8 * 128), (unsigned)std::min(rows_ext, 65535));
    split3_v8_kernel<<<grid, 128, 0, st>>>(S, ld, rows, cols, k_cols, Kp, lo_mask, ones_col, D, dld, rows_ext,
                                            cols_v8);
  } else {
    const dim3 grid((unsigned)ceil_div(cols_ext, 256), (unsigned)std::min(rows_ext, 65535));
    split3_kernel<<<grid, 128, 0, st>>>(S, ld, rows, cols, k_cols, Kp, lo_mask, ones_col, D, dld, rows_ext);
  }
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace

size_t gemm_f32x3_workspace_bytes(bool transA, bool transB, int M, int N, int K, bool a_ones) {
  const X3Dims d = x3_dims(transA, transB, M, N, K, a_ones);
  return (size_t)round_up(d.a_rows * d.a_ld * 2, 256) + (size_t)round_up(d.b_rows * d.b_ld * 2, 256) +
         (d.ksplit > 1 ? (size_t)d.ksplit * d.p_stride * 4 : 0);
}

size_t x3_b_elems(bool transB, int N, int K) {
  const X3Dims d = x3_dims(false, transB, 1, N, K, false);
  return (size_t)(d.b_rows * d.b_ld);
}

void x3_split_b(bool transB, int N, int K, const float* B, int64_t ldb, __nv_bfloat16* B3, cudaStream_t st) {
  const X3Dims d = x3_dims(false, transB, 1, N, K, false);
  if (!transB) split3(B, ldb, K, N, false, d.Kp, 0b100, -1, B3, d.b_ld, st);
  else split3(B, ldb, N, K, true, d.Kp, 0b100, -1, B3, d.b_ld, st);
}

namespace {
// the GEMM over split operands: a3 from the scratch, b3 split here or presplit
void x3_core(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda, const float* B,
             int64_t ldb, const __nv_bfloat16* b_pre, float beta, float* C, int64_t ldc, const float* bias,
             float* ones_row_out, int64_t ld_ones, void* ws, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  const bool a_ones = ones_row_out != nullptr;
  SL_REQUIRE(!a_ones || transA, SL_ERR_INVALID_ARGUMENT, "gemm_f32x3: ones row needs A stored [K, M]");
  const X3Dims d = x3_dims(transA, transB, M, N, K, a_ones);
  auto* a3 = static_cast<__nv_bfloat16*>(ws);
  char* after_a = static_cast<char*>(ws) + round_up(d.a_rows * d.a_ld * 2, 256);
  const __nv_bfloat16* b3 = b_pre;
  // A copies: hi, lo, hi (lo_mask 0b010); B copies: hi, hi, lo (0b100)
  if (!transA) split3(A, lda, M, K, true, d.Kp, 0b010, -1, a3, d.a_ld, st);
  else split3(A, lda, K, M, false, d.Kp, 0b010, a_ones ? M : -1, a3, d.a_ld, st);
  if (!b3) {
    auto* b3w = reinterpret_cast<__nv_bfloat16*>(after_a);
    if (!transB) split3(B, ldb, K, N, false, d.Kp, 0b100, -1, b3w, d.b_ld, st);
    else split3(B, ldb, N, K, true, d.Kp, 0b100, -1, b3w, d.b_ld, st);
    b3 = b3w;
  }
  TcGemm g{M + (a_ones ? 1 : 0), N, 3 * d.Kp, a3, d.a_ld, transA, b3, d.b_ld, !transB, C, ldc, 1.f, beta, bias};
  {  // chunked accumulation only where one work unit's K range is longer than a chunk
    const int64_t nk = ceil_div(3 * (int64_t)d.Kp, 64);
    if (ceil_div(nk, d.ksplit) > kX3ChunkBlocks) g.kchunk = kX3ChunkBlocks;
  }
  if (d.ksplit > 1) {  // small output: split K over the idle SMs, then a fixed-order reduction
    float* part = reinterpret_cast<float*>(after_a + round_up(d.b_rows * d.b_ld * 2, 256));
    g.C = part;
    g.ldc = d.p_ld;
    g.beta = 0.f;
    g.bias = nullptr;
    g.ksplit = d.ksplit;  // gemm_tc2_ksplit already returns a count without empty units
    g.split_stride = d.p_stride;
    gemm_bf16_tc(g, st);
    const int Mt = M + (a_ones ? 1 : 0);
    splitk_reduce_kernel<<<dim3((unsigned)ceil_div(N, 256), (unsigned)std::min(Mt, 65535)), 256, 0, st>>>(
        part, d.ksplit, d.p_stride, d.p_ld, Mt, N, beta, C, ldc, bias, a_ones ? M : (1 << 30), ones_row_out, ld_ones);
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
  x3_core(transA, transB, M, N, K, A, lda, B, ldb, nullptr, beta, C, ldc, bias, ones_row_out, ld_ones, ws, st);
}

void gemm_f32x3_pb(bool transA, bool transB, int M, int N, int K, const float* A, int64_t lda,
                   const __nv_bfloat16* B3, float beta, float* C, int64_t ldc, const float* bias, void* ws,
                   cudaStream_t st, float* ones_row_out, int64_t ld_ones) {
  x3_core(transA, transB, M, N, K, A, lda, nullptr, 0, B3, beta, C, ldc, bias, ones_row_out, ld_ones, ws, st);
}

}  // namespace sl
