// Output layer of the Listing-1 decoder: logits = x W + b,
// log_softmax, label-smoothed cross entropy averaged over the valid target
// positions, and its gradients — reference compiler.cpp:651-663 (Softmax layer
// = add(matmul(x, W), b) -> log_softmax), tape.cpp:879-924 (log_softmax and
// its adjoint) and tape.cpp:1224-1298 (ce_label_smoothing and its adjoint).
//
// Per valid row r with target y (lp = z - lse):
//   loss_r = -(1 - eps) lp_y - eps / V sum_j lp_j = lse - (1 - eps) z_y - eps / V sum_j z_j
//   dz_rj  = (softmax(z)_j - eps / V - (1 - eps) [j == y]) / n_valid
// (the composition of the two adjoints with upstream gradient 1).
//
// B200 plan (one training call, no fp32 logits in HBM):
//   1. K-GEMM  Z = X W + b on the CTA-pair tensor-core GEMM, bf16 Z, with the
//      online-softmax statistics of every 128-column block fused into the
//      epilogue (max, sum exp, sum z, z_y);
//   2. one warp per row folds the block statistics into lse / loss and turns
//      the row of Z into dZ in place (bf16);
//   3. dX = dZ W^T and [dW; db] = [X | 1]^T dZ on the same GEMM.
#include <algorithm>
#include <cmath>

#include "convert.h"
#include "gemm.h"
#include "profile.h"
#include "softmax_ce.h"

namespace sl {
namespace {

struct CeScratch {
  double loss_sum;
  int n_valid;
  int pad;
};

__global__ void ce_count_kernel(const int32_t* lens, int B, int T, CeScratch* sc) {
  int n = 0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) n += max(0, min(lens[b], T));
#pragma unroll
  for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  __shared__ int part[32];
  if (threadIdx.x % 32 == 0) part[threadIdx.x / 32] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) tot += part[w];
    sc->n_valid = tot;
    sc->loss_sum = 0.0;
  }
}

// one warp per row: fold the block statistics, accumulate the loss, Z -> dZ in place
__global__ void __launch_bounds__(256) ce_rows_kernel(__nv_bfloat16* __restrict__ Z, int64_t ldz, int rows, int T,
                                                      int V, const float4* __restrict__ part, int nblk,
                                                      const int32_t* __restrict__ targets,
                                                      const int32_t* __restrict__ lens, float eps, CeScratch* sc,
                                                      int* bad_target) {
  const int lane = threadIdx.x % 32;
  const int row = blockIdx.x * 8 + threadIdx.x / 32;
  if (row >= rows) return;
  const int b = row / T, t = row % T;
  const bool valid = t < lens[b];
  __nv_bfloat16* z = Z + (int64_t)row * ldz;
  if (!valid) {  // masked position (tape.cpp:1256-1262): no loss, zero gradient
    for (int j = lane * 8; j < V; j += 256)
      if (j + 8 <= V) *reinterpret_cast<uint4*>(z + j) = make_uint4(0u, 0u, 0u, 0u);
      else
        for (int k = j; k < V; ++k) z[k] = __float2bfloat16_rn(0.f);
    return;
  }
  const int y = targets[row];
  if (y < 0 || y >= V) {  // reference: IndexError naming the layer (tape.cpp:1265-1268)
    // poison the step: a NaN loss and NaN dZ row make every gradient non-finite, so
    // the fused optimizer step skips the update (the reference raises before it)
    if (lane == 0) {
      atomicMax(bad_target, 1);
      atomicAdd(&sc->loss_sum, (double)__int_as_float(0x7fc00000));
    }
    const __nv_bfloat16 nan = __float2bfloat16_rn(__int_as_float(0x7fc00000));
    for (int j = lane; j < V; j += 32) z[j] = nan;
    return;
  }
  float m = -INFINITY;
  for (int k = lane; k < nblk; k += 32) m = fmaxf(m, part[(int64_t)row * nblk + k].x);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f, tz = 0.f, zy = 0.f;
  for (int k = lane; k < nblk; k += 32) {
    const float4 q = part[(int64_t)row * nblk + k];
    s += q.y * exp2f((q.x - m) * 1.4426950408889634f);
    tz += q.z;
    zy += q.w;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    tz += __shfl_xor_sync(0xffffffffu, tz, o);
    zy += __shfl_xor_sync(0xffffffffu, zy, o);
  }
  const float lse = m + logf(s);
  if (lane == 0)
    atomicAdd(&sc->loss_sum, (double)lse - (1.0 - (double)eps) * (double)zy - (double)eps / V * (double)tz);
  const float inv_n = 1.f / (float)max(sc->n_valid, 1);
  const float base = -eps / (float)V;
  for (int j = lane * 8; j < V; j += 256) {
    if (j + 8 <= V) {
      uint4 w = *reinterpret_cast<const uint4*>(z + j);
      uint32_t* ww = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ww[k]));
        float g0 = exp2f((f.x - lse) * 1.4426950408889634f) + base;
        float g1 = exp2f((f.y - lse) * 1.4426950408889634f) + base;
        if (j + 2 * k == y) g0 -= 1.f - eps;
        if (j + 2 * k + 1 == y) g1 -= 1.f - eps;
        const __nv_bfloat162 o = __floats2bfloat162_rn(g0 * inv_n, g1 * inv_n);
        ww[k] = *reinterpret_cast<const uint32_t*>(&o);
      }
      *reinterpret_cast<uint4*>(z + j) = w;
    } else {
      for (int k = j; k < V; ++k) {
        float g = exp2f((__bfloat162float(z[k]) - lse) * 1.4426950408889634f) + base;
        if (k == y) g -= 1.f - eps;
        z[k] = __float2bfloat16_rn(g * inv_n);
      }
    }
  }
}

// fp32-class variant (SL_PREC_FP32): one warp per row of fp32 logits Z: an online
// (max, sum exp) pass with sum z and z_y, lse = m + log(s), then Z -> dZ in place.
// Reference arithmetic: expf / logf (tape.cpp:879-924, 1224-1298).
// dZ goes to its split-bf16 image (gemm.h x3_split_img layout: hi [rows, ldi], then
// lo; the padding columns zero), which both gradient GEMMs read — dZ is never
// written as fp32 and never split separately.
__device__ __forceinline__ void dz_store1(__nv_bfloat16* hi, __nv_bfloat16* lo, int64_t off, float g) {
  const __nv_bfloat16 h = __float2bfloat16_rn(g);
  hi[off] = h;
  lo[off] = __float2bfloat16_rn(g - __bfloat162float(h));
}

__global__ void __launch_bounds__(256) ce_rows_f32_kernel(const float* __restrict__ Z, int64_t ldz, int rows, int T,
                                                          int V, const int32_t* __restrict__ targets,
                                                          const int32_t* __restrict__ lens, float eps, CeScratch* sc,
                                                          int* bad_target, __nv_bfloat16* __restrict__ dzi,
                                                          int64_t ldi) {
  const int lane = threadIdx.x % 32;
  const int row = blockIdx.x * 8 + threadIdx.x / 32;
  if (row >= rows) return;
  const int b = row / T, t = row % T;
  const float* z = Z + (int64_t)row * ldz;
  __nv_bfloat16* hi = dzi + (int64_t)row * ldi;
  __nv_bfloat16* lo = dzi + ((int64_t)rows + row) * ldi;
  const bool vec = (V % 8) == 0 && (ldz % 4) == 0 && (ldi % 8) == 0;
  for (int j = V + lane; j < ldi; j += 32) dz_store1(hi, lo, j, 0.f);  // padding
  if (t >= lens[b]) {  // masked position (tape.cpp:1256-1262): no loss, zero gradient
    for (int j = lane; j < V; j += 32) dz_store1(hi, lo, j, 0.f);
    return;
  }
  const int y = targets[row];
  if (y < 0 || y >= V) {  // reference IndexError: poison the step (see ce_rows_kernel)
    if (lane == 0) {
      atomicMax(bad_target, 1);
      atomicAdd(&sc->loss_sum, (double)__int_as_float(0x7fc00000));
    }
    for (int j = lane; j < V; j += 32) dz_store1(hi, lo, j, __int_as_float(0x7fc00000));
    return;
  }
  float m = -INFINITY, s = 0.f, tz = 0.f;
  auto fold = [&](float v) {
    if (v > m) {
      s = s * expf(m - v) + 1.f;
      m = v;
    } else {
      s += expf(v - m);
    }
    tz += v;
  };
  if (vec) {
    for (int j = lane * 4; j < V; j += 128) {
      const float4 q = *reinterpret_cast<const float4*>(z + j);
      fold(q.x), fold(q.y), fold(q.z), fold(q.w);
    }
  } else {
    for (int j = lane; j < V; j += 32) fold(z[j]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - mm));
    m = mm;
    tz += __shfl_xor_sync(0xffffffffu, tz, o);
  }
  const float zy = z[y];
  const float lse = m + logf(s);
  if (lane == 0)
    atomicAdd(&sc->loss_sum, (double)lse - (1.0 - (double)eps) * (double)zy - (double)eps / V * (double)tz);
  const float inv_n = 1.f / (float)max(sc->n_valid, 1);
  const float base = -eps / (float)V;
  __syncwarp();
  if (vec) {  // 8 columns per lane: 16 B image stores
    for (int j = lane * 8; j < V; j += 256) {
      const float4 q0 = *reinterpret_cast<const float4*>(z + j), q1 = *reinterpret_cast<const float4*>(z + j + 4);
      const float q[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float g = expf(q[k] - lse) + base;
        if (j + k == y) g -= 1.f - eps;
        g *= inv_n;
        h[k] = __float2bfloat16_rn(g);
        l[k] = __float2bfloat16_rn(g - __bfloat162float(h[k]));
      }
      *reinterpret_cast<uint4*>(hi + j) = *reinterpret_cast<const uint4*>(h);
      *reinterpret_cast<uint4*>(lo + j) = *reinterpret_cast<const uint4*>(l);
    }
  } else {
    for (int j = lane; j < V; j += 32) {
      float g = expf(z[j] - lse) + base;
      if (j == y) g -= 1.f - eps;
      dz_store1(hi, lo, j, g * inv_n);
    }
  }
}

// The same with the row statistics folded in from the logits GEMM's epilogue
// (per 128-column block: max, sum exp(z - max), sum z, z_y): one pass over the row
// of Z (read Z, write dZ's image) instead of two.
__global__ void __launch_bounds__(256) ce_rows_f32_stats_kernel(const float* __restrict__ Z, int64_t ldz, int rows,
                                                                int T, int V, const int32_t* __restrict__ targets,
                                                                const int32_t* __restrict__ lens, float eps,
                                                                CeScratch* sc, int* bad_target,
                                                                const float4* __restrict__ part, int nblk,
                                                                __nv_bfloat16* __restrict__ dzi, int64_t ldi) {
  const int lane = threadIdx.x % 32;
  const int row = blockIdx.x * 8 + threadIdx.x / 32;
  if (row >= rows) return;
  const int b = row / T, t = row % T;
  const float* z = Z + (int64_t)row * ldz;
  __nv_bfloat16* hi = dzi + (int64_t)row * ldi;
  __nv_bfloat16* lo = dzi + ((int64_t)rows + row) * ldi;
  for (int j = V + lane; j < ldi; j += 32) dz_store1(hi, lo, j, 0.f);  // padding
  if (t >= lens[b]) {  // masked position (tape.cpp:1256-1262): no loss, zero gradient
    for (int j = lane; j < V; j += 32) dz_store1(hi, lo, j, 0.f);
    return;
  }
  const int y = targets[row];
  if (y < 0 || y >= V) {  // reference IndexError: poison the step (see ce_rows_kernel)
    if (lane == 0) {
      atomicMax(bad_target, 1);
      atomicAdd(&sc->loss_sum, (double)__int_as_float(0x7fc00000));
    }
    for (int j = lane; j < V; j += 32) dz_store1(hi, lo, j, __int_as_float(0x7fc00000));
    return;
  }
  float m = -INFINITY, ss = 0.f, tz = 0.f, zy = 0.f;
  for (int k = lane; k < nblk; k += 32) {
    const float4 q = part[(int64_t)row * nblk + k];
    const float mn = fmaxf(m, q.x);
    ss = (m == -INFINITY ? 0.f : ss * expf(m - mn)) + (q.x == -INFINITY ? 0.f : q.y * expf(q.x - mn));
    m = mn;
    tz += q.z;
    if (y / 128 == k) zy = q.w;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, ss, o);
    const float mm = fmaxf(m, m2);
    ss = (m == -INFINITY ? 0.f : ss * expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - mm));
    m = mm;
    tz += __shfl_xor_sync(0xffffffffu, tz, o);
    zy += __shfl_xor_sync(0xffffffffu, zy, o);
  }
  const float lse = m + logf(ss);
  if (lane == 0)
    atomicAdd(&sc->loss_sum, (double)lse - (1.0 - (double)eps) * (double)zy - (double)eps / V * (double)tz);
  const float inv_n = 1.f / (float)max(sc->n_valid, 1);
  const float base = -eps / (float)V;
  if ((V % 8) == 0 && (ldz % 4) == 0 && (ldi % 8) == 0) {  // 8 columns per lane: 16 B image stores
    for (int j = lane * 8; j < V; j += 256) {
      const float4 q0 = *reinterpret_cast<const float4*>(z + j), q1 = *reinterpret_cast<const float4*>(z + j + 4);
      const float q[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float g = expf(q[k] - lse) + base;
        if (j + k == y) g -= 1.f - eps;
        g *= inv_n;
        h[k] = __float2bfloat16_rn(g);
        l[k] = __float2bfloat16_rn(g - __bfloat162float(h[k]));
      }
      *reinterpret_cast<uint4*>(hi + j) = *reinterpret_cast<const uint4*>(h);
      *reinterpret_cast<uint4*>(lo + j) = *reinterpret_cast<const uint4*>(l);
    }
  } else {
    for (int j = lane; j < V; j += 32) {
      float g = expf(z[j] - lse) + base;
      if (j == y) g -= 1.f - eps;
      dz_store1(hi, lo, j, g * inv_n);
    }
  }
}

__global__ void ce_finalize_kernel(const CeScratch* sc, float* loss_out) {
  *loss_out = (float)(sc->loss_sum / (double)max(sc->n_valid, 1));
}

}  // namespace

CeDims ce_dims(int B, int T, int D, int V) {
  CeDims c;
  c.rows = (int64_t)B * T;
  c.Dp = round_up(D + 1, 64);  // + a ones column: db from the dW GEMM
  c.Vp = round_up(V, 64);
  c.nblk = (int)ceil_div(V, 128);
  return c;
}

size_t output_ce_workspace_bytes(int B, int T, int D, int V) {
  const CeDims c = ce_dims(B, T, D, V);
  auto al = [](size_t x) { return round_up((int64_t)x, 256); };
  return al(c.rows * c.Dp * 2) + al((size_t)D * c.Vp * 2) + al(c.rows * c.Vp * 2) +
         al(c.rows * c.nblk * sizeof(float4)) + al(sizeof(CeScratch)) + al(sizeof(int));
}

void output_ce(int B, int T, int D, int V, const float* x, const int32_t* targets, const int32_t* lens,
               const float* W, const float* b, float eps, float* loss_out, float* dx, float* dW, float* db,
               bool accumulate, void* workspace, int* bad_target, cudaStream_t stream) {
  const CeDims c = ce_dims(B, T, D, V);
  char* w = static_cast<char*>(workspace);
  auto take = [&](size_t bytes) {
    char* p = w;
    w += round_up((int64_t)bytes, 256);
    return p;
  };
  auto* xb = reinterpret_cast<__nv_bfloat16*>(take(c.rows * c.Dp * 2));
  auto* wb = reinterpret_cast<__nv_bfloat16*>(take((size_t)D * c.Vp * 2));
  auto* zb = reinterpret_cast<__nv_bfloat16*>(take(c.rows * c.Vp * 2));
  auto* part = reinterpret_cast<float4*>(take(c.rows * c.nblk * sizeof(float4)));
  auto* sc = reinterpret_cast<CeScratch*>(take(sizeof(CeScratch)));
  SL_CUDA_TRY(cudaMemsetAsync(bad_target, 0, sizeof(int), stream));
  // bf16 operands: [X | 1] and W (gemm operands are 16 B aligned rows)
  f32_to_bf16(c.rows, D, x, D, xb, c.Dp, stream);
  fill_col_bf16(c.rows, D, xb, c.Dp, 1.f, stream);
  f32_to_bf16(D, V, W, V, wb, c.Vp, stream);
  ce_count_kernel<<<1, 256, 0, stream>>>(lens, B, T, sc);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch(3);
  const double f = 2.0 * c.rows * D * (double)V;
  {  // 1. Z = X W + b (bf16) with the fused online-softmax statistics
    Phase ph(stream, "k7_logits_gemm", f);
    TcGemm g{(int)c.rows, V, D, xb, c.Dp, false, wb, c.Vp, true, nullptr, c.Vp, 1.f, 0.f, b};
    g.Cb = zb;
    g.sm_part = part;
    g.sm_ld = c.nblk;
    g.sm_targets = targets;
    gemm_bf16_tc(g, stream);
  }
  {  // 2. loss and Z -> dZ in place
    Phase ph(stream, "k7_softmax_ce", 0.0, 4.0 * c.rows * V);
    ce_rows_kernel<<<(unsigned)ceil_div(c.rows, 8), 256, 0, stream>>>(zb, c.Vp, (int)c.rows, T, V, part, c.nblk,
                                                                       targets, lens, eps, sc, bad_target);
    SL_CUDA_TRY(cudaGetLastError());
    ce_finalize_kernel<<<1, 1, 0, stream>>>(sc, loss_out);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch(2);
  }
  const float beta = accumulate ? 1.f : 0.f;
  if (dx) {  // 3a. dX = dZ W^T
    Phase ph(stream, "k7_dx_gemm", f);
    TcGemm g{(int)c.rows, D, V, zb, c.Vp, false, wb, c.Vp, false, dx, D, 1.f, beta, nullptr};
    gemm_bf16_tc(g, stream);
  }
  if (dW || db) {  // 3b. [dW; db] = [X | 1]^T dZ
    Phase ph(stream, "k7_dw_gemm", f);
    TcGemm g{D + 1, V, (int)c.rows, xb, c.Dp, true, zb, c.Vp, true, dW, V, 1.f, beta, nullptr};
    g.m_split = D;
    g.C2 = db;
    g.ldc2 = V;
    if (!db) g.M = D;
    gemm_bf16_tc(g, stream);
  }
}

size_t output_ce_f32_workspace_bytes(int B, int T, int D, int V) {
  const int64_t rows = (int64_t)B * T;
  const size_t x3 = std::max({gemm_f32x3_workspace_bytes(false, false, (int)rows, V, D, false),   // logits
                              gemm_f32x3_workspace_bytes(false, true, (int)rows, D, V, false),    // dX
                              gemm_f32x3_workspace_bytes(true, false, D, V, (int)rows, true)});   // [dW; db]
  return (size_t)round_up(rows * V * 4, 256) + (size_t)round_up(x3_img_elems((int)rows, V) * 2, 256) +
         (size_t)round_up(rows * ceil_div(V, 128) * sizeof(float4), 256) + (size_t)round_up(sizeof(CeScratch), 256) +
         (size_t)round_up(x3_img_elems((int)rows, D + 1) * 2, 256) + (size_t)round_up(x3_img_elems(D, V) * 2, 256) + x3;
}

void output_ce_f32(int B, int T, int D, int V, const float* x, const int32_t* targets, const int32_t* lens,
                   const float* W, const float* b, float eps, float* loss_out, float* dx, float* dW, float* db,
                   bool accumulate, void* workspace, int* bad_target, cudaStream_t stream) {
  const int64_t rows = (int64_t)B * T;
  char* w = static_cast<char*>(workspace);
  float* z = reinterpret_cast<float*>(w);
  w += round_up(rows * V * 4, 256);
  auto* dzi = reinterpret_cast<__nv_bfloat16*>(w);  // the split image of dZ
  w += round_up(x3_img_elems((int)rows, V) * 2, 256);
  const int nblk = (int)ceil_div(V, 128);
  auto* smp = reinterpret_cast<float4*>(w);  // per (row, 128-column block) softmax statistics
  w += round_up(rows * nblk * sizeof(float4), 256);
  auto* sc = reinterpret_cast<CeScratch*>(w);
  w += round_up(sizeof(CeScratch), 256);
  // x (ones column at D: the d b row) and W split once, each image read by two GEMMs
  auto* xi = reinterpret_cast<__nv_bfloat16*>(w);
  const int64_t xl = x3_img_ld(D + 1);
  w += round_up(x3_img_elems((int)rows, D + 1) * 2, 256);
  auto* wi = reinterpret_cast<__nv_bfloat16*>(w);
  const int64_t wl = x3_img_ld(V);
  w += round_up(x3_img_elems(D, V) * 2, 256);
  void* gws = w;
  x3_split_into(x, D, (int)rows, D, D, xi, xl, xl, rows * xl, stream);
  x3_split_img(W, V, D, V, wi, stream);
  SL_CUDA_TRY(cudaMemsetAsync(bad_target, 0, sizeof(int), stream));
  ce_count_kernel<<<1, 256, 0, stream>>>(lens, B, T, sc);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
  const double f = 2.0 * rows * D * (double)V;
  bool stats = false;
  {
    Phase ph(stream, "k7_logits_gemm", f);
    // (an out-of-range target only fails to match a column in the statistics; the CE
    // kernel still sees the raw id and poisons the step)
    stats = gemm_f32x3_softmax_stats((int)rows, V, D, nullptr, 0, nullptr, 0, z, V, b, smp, nblk, targets, gws,
                                     stream, xi, xl, rows * xl, wi, wl, (int64_t)D * wl);
  }
  {
    Phase ph(stream, "k7_softmax_ce", 0.0, 12.0 * rows * V);
    if (stats)
      ce_rows_f32_stats_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, stream>>>(
          z, V, (int)rows, T, V, targets, lens, eps, sc, bad_target, smp, nblk, dzi, x3_img_ld(V));
    else
      ce_rows_f32_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, stream>>>(z, V, (int)rows, T, V, targets, lens, eps,
                                                                           sc, bad_target, dzi, x3_img_ld(V));
    SL_CUDA_TRY(cudaGetLastError());
    ce_finalize_kernel<<<1, 1, 0, stream>>>(sc, loss_out);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch(2);
  }
  const float beta = accumulate ? 1.f : 0.f;
  if (dx) {
    Phase ph(stream, "k7_dx_gemm", f);
    gemm_f32x3_ex(false, true, (int)rows, D, V, nullptr, 0, dzi, nullptr, 0, wi, beta, dx, D, nullptr, nullptr, 0,
                  gws, stream, 0, 0, wl, (int64_t)D * wl);
  }
  if (dW) {
    Phase ph(stream, "k7_dw_gemm", f);
    gemm_f32x3_ex(true, false, D, V, (int)rows, nullptr, 0, xi, nullptr, 0, dzi, beta, dW, V, nullptr, db, V, gws,
                  stream, xl, rows * xl);
  } else if (db) {
    SL_REQUIRE(false, SL_ERR_INVALID_ARGUMENT, "output_ce (fp32): db needs dW");
  }
}

}  // namespace sl
