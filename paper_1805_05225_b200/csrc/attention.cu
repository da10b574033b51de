// The decoder's MLP attention step, forward and backward, as
// the reference's Listing-1 subnet wires it (models.cpp:107-154, evaluated by
// compiler.cpp:616-639):
//   s_tr  = s W_s + b_s                                  [B, K]
//   e     = tanh(enc_ctx + accum W_fb + b_fb + s_tr) v + b_v   [B, Ts]
//   a     = softmax over the valid source positions       (tape.cpp:926-985)
//   accum'= accum + a
//   att   = sum_j a_j enc_j                               (tape.cpp:987-1072)
// The step streams its [Ts, K] energy inputs and [Ts, E] encoder states once
// (forward) / twice with their gradients (backward), with the tanh / softmax /
// weighted sum fused into those passes; the small projections (s_tr and its
// gradients) run on the tensor cores as fp32-accurate split-bf16 GEMMs
// (gemm_f32x3.cu).  fp32 data: the step is bandwidth-bound, not tensor-bound.
#include <algorithm>

#include "attention.h"
#include "fastmath.cuh"
#include "gemm.h"
#include "profile.h"

namespace sl {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Decomposition: every kernel runs one CTA per (batch row, chunk of kJC source
// positions) or (batch row, slice of encoder columns) — ~1000 CTAs, so loads of
// one CTA overlap the tanh / reduction work of the others on the same SM (one
// CTA per batch row left 256 CTAs on 148 SMs, half of them alone, at ~25% of
// HBM).  Inside a CTA every thread owns VK key columns (VE encoder columns) and
// walks the chunk's positions with per-position partial sums in registers, so
// every load is an independent coalesced 16 B vector; the per-position dot
// products finish in one block reduction.  VK = 4 / VE = 8 when K % 4 == 0 /
// E % 8 == 0 and the rows stay 16 B aligned, else scalar columns.
constexpr int kJC = 16;        // source positions per CTA (d_a pass)
constexpr int kJE = 8;         // source positions per CTA (tanh passes: more CTAs resident per SM)
constexpr int kCtxThreads = 64;  // context kernel: 64 threads x VE columns per CTA ...
constexpr int kCtxGroups = 4;    // ... times 4 groups splitting the source positions

__device__ __forceinline__ int round_up_dev(int x, int m) { return (x + m - 1) / m * m; }

template <int W>
struct Vec {
  float f[W];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < W; ++i) f[i] = 0.f;
  }
  __device__ __forceinline__ void load(const float* p) {  // read-only data
    if constexpr (W % 8 == 0) {  // 256-bit loads (32 B aligned rows): half the load instructions
#pragma unroll
      for (int i = 0; i < W; i += 8)
        asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=f"(f[i]), "=f"(f[i + 1]), "=f"(f[i + 2]), "=f"(f[i + 3]), "=f"(f[i + 4]), "=f"(f[i + 5]),
                       "=f"(f[i + 6]), "=f"(f[i + 7])
                     : "l"(p + i));
    } else if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W; i += 4) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(p) + i / 4);
        f[i] = q.x, f[i + 1] = q.y, f[i + 2] = q.z, f[i + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < W; ++i) f[i] = __ldg(p + i);
    }
  }
  __device__ __forceinline__ void load_plain(const float* p) {  // data this kernel also writes
    if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W; i += 4) {
        const float4 q = reinterpret_cast<const float4*>(p)[i / 4];
        f[i] = q.x, f[i + 1] = q.y, f[i + 2] = q.z, f[i + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < W; ++i) f[i] = p[i];
    }
  }
  __device__ __forceinline__ void store(float* p) const {
    if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W; i += 4)
        reinterpret_cast<float4*>(p)[i / 4] = make_float4(f[i], f[i + 1], f[i + 2], f[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < W; ++i) p[i] = f[i];
    }
  }
  __device__ __forceinline__ void atomic_add(float* p) const {
    if constexpr (W % 4 == 0) {
#pragma unroll
      for (int i = 0; i < W; i += 4)
        atomicAdd(reinterpret_cast<float4*>(p) + i / 4, make_float4(f[i], f[i + 1], f[i + 2], f[i + 3]));
    } else {
#pragma unroll
      for (int i = 0; i < W; ++i) atomicAdd(p + i, f[i]);
    }
  }
};

// tanh(x) = 1 - 2 / (1 + e^{2x}): two MUFU ops, absolute error ~1e-7 (the
// energies and their adjoint only see tanh through sums, so an absolute bound
// is the one that matters); clamped so e^{2x} stays finite
__device__ __forceinline__ float tanh_fast(float x) {
  x = fminf(fmaxf(x, -15.f), 15.f);
  return 1.f - __fdividef(2.f, 1.f + __expf(2.f * x));
}

// sum over the block of per-thread partials part[0..n): result to out[0..n)
template <int kJC>
__device__ __forceinline__ void block_reduce_chunk(const float (&part)[kJC], int n, float* red /*[kWarps][kJC]*/,
                                                   float* out) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // transpose-reduce: after each round a lane holds sums over twice the lanes for half the positions
  float v[kJC];
#pragma unroll
  for (int j = 0; j < kJC; ++j) v[j] = part[j];
#pragma unroll
  for (int w = kJC / 2, o = 16; w >= 1; w /= 2, o /= 2) {
    const bool upper = lane & o;
#pragma unroll
    for (int j = 0; j < w; ++j) {
      const float send = upper ? v[j] : v[j + w];
      const float keep = upper ? v[j + w] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  float t = v[0];
#pragma unroll
  for (int o = 32 / kJC / 2; o >= 1; o /= 2) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane % (32 / kJC) == 0) {  // the position index is spelled by the lane's high bits
    int j = 0;
#pragma unroll
    for (int w = kJC / 2, o = 16; w >= 1; w /= 2, o /= 2)
      if (lane & o) j += w;
    red[warp * kJC + j] = t;
  }
  __syncthreads();
  if (threadIdx.x < n) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[w * kJC + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

template <int VK>
__device__ __forceinline__ void load_cols(const AttnArgs& p, int b, int k, Vec<VK>& c, Vec<VK>& w, Vec<VK>& v) {
  Vec<VK> bf;
  c.load(p.s_tr + (size_t)b * p.K + k);
  bf.load(p.b_fb + k);
#pragma unroll
  for (int i = 0; i < VK; ++i) c.f[i] += bf.f[i];
  w.load(p.W_fb + k);
  v.load(p.v + k);
}

// e[b, j] (without b_v) for the CTA's chunk of valid positions:
// e_j = <v, tanh(enc_ctx_j + accum_j W_fb + b_fb + s_tr)>  (compiler.cpp:616-639)
template <int VK>
__global__ void __launch_bounds__(kThreads, 3) attn_energy_kernel(AttnArgs p, float* __restrict__ e_out) {
  __shared__ float red[kWarps * kJE];
  const int b = blockIdx.y, j0 = blockIdx.x * kJE, K = p.K, Ts = p.Ts;
  const int nT = min(kJE, Ts - j0);  // the chunk's positions (no dependency on the length)
  // the chunk's energy inputs and column constants are loaded first, so the latency of
  // the length lookup hides under them
  const int kf = threadIdx.x * VK;
  Vec<VK> c0, w0, v0, x0[kJE];
  float acc[kJE], part[kJE];
  if (kf < K) {
    load_cols(p, b, kf, c0, w0, v0);
#pragma unroll
    for (int j = 0; j < kJE; ++j)
      if (j < nT) x0[j].load(p.enc_ctx + ((size_t)b * Ts + j0 + j) * K + kf);
  }
#pragma unroll
  for (int j = 0; j < kJE; ++j) {
    part[j] = 0.f;
    acc[j] = j < nT ? __ldg(p.accum + (size_t)b * Ts + j0 + j) : 0.f;
  }
  const int len = min(max(p.lens[b], 0), Ts);
  const int n = min(kJE, len - j0);
  if (n <= 0) return;
  auto cols = [&](const Vec<VK>& c, const Vec<VK>& w, const Vec<VK>& v, const Vec<VK>(&x)[kJE]) {
#pragma unroll
    for (int j = 0; j < kJE; ++j) {
      if (j < n) {
        if constexpr (VK % 2 == 0) {  // paired-fp32 math, two columns per instruction
          using namespace fm;
          float2 s2v = s2(0.f);
#pragma unroll
          for (int i = 0; i < VK; i += 2) {
            const float2 t = tanh2(fma2(s2(acc[j]), make_float2(w.f[i], w.f[i + 1]),
                                        add2(make_float2(x[j].f[i], x[j].f[i + 1]), make_float2(c.f[i], c.f[i + 1]))));
            s2v = fma2(make_float2(v.f[i], v.f[i + 1]), t, s2v);
          }
          part[j] += s2v.x + s2v.y;
        } else {
#pragma unroll
          for (int i = 0; i < VK; ++i) part[j] += v.f[i] * tanh_fast(x[j].f[i] + acc[j] * w.f[i] + c.f[i]);
        }
      }
    }
  };
  if (kf < K) cols(c0, w0, v0, x0);
  for (int k = kf + kThreads * VK; k < K; k += kThreads * VK) {
    Vec<VK> c, w, v, x[kJE];
    load_cols(p, b, k, c, w, v);
#pragma unroll
    for (int j = 0; j < kJE; ++j)
      if (j < n) x[j].load(p.enc_ctx + ((size_t)b * Ts + j0 + j) * K + k);
    cols(c, w, v, x);
  }
  block_reduce_chunk(part, n, red, e_out + (size_t)b * Ts + j0);
}

// masked softmax of row b (tape.cpp:952-960) into a_sh[0..Ts) — warp 0
__device__ __forceinline__ void row_softmax(const AttnArgs& p, const float* e, int b, int len, float* a_sh) {
  const int lane = threadIdx.x % 32, Ts = p.Ts;
  const float bv = *p.b_v;
  float m = -INFINITY;
  for (int j = lane; j < len; j += 32) m = fmaxf(m, e[(size_t)b * Ts + j] + bv);
  m = warp_max(m);
  float z = 0.f;
  for (int j = lane; j < len; j += 32) z += expf(e[(size_t)b * Ts + j] + bv - m);
  z = warp_sum(z);
  for (int j = lane; j < Ts; j += 32) a_sh[j] = j < len ? expf(e[(size_t)b * Ts + j] + bv - m) / z : 0.f;
}

// softmax (recomputed per CTA from the Ts energies) and the context slice
// att[b, x0:x1) = sum_j a_j enc[b, j, x0:x1)  (tape.cpp:1005-1014); CTA 0 of
// the row also writes a and accum'.  kCtxGroups thread groups split the
// positions (interleaved) for more loads in flight per SM and add their
// partial sums in a fixed order through shared memory (deterministic).
template <int VE>
__global__ void __launch_bounds__(kCtxThreads * kCtxGroups) attn_context_kernel(AttnArgs p, const float* __restrict__ e) {
  extern __shared__ float a_sh[];  // [Ts] then [kCtxGroups - 1][kCtxThreads * VE] partials
  const int b = blockIdx.y, Ts = p.Ts, E = p.E;
  const int ct = threadIdx.x % kCtxThreads, grp = threadIdx.x / kCtxThreads;
  const int x = (blockIdx.x * kCtxThreads + ct) * VE;
  constexpr int G = kCtxGroups;
  // the first 4 encoder rows of the thread's group do not depend on the softmax: their
  // loads go out before it (a_j = 0 past the length masks them)
  Vec<VE> pre[4];
  const bool use_pre = x < E && grp + 3 * G < Ts;
  if (use_pre) {
#pragma unroll
    for (int i = 0; i < 4; ++i) pre[i].load(p.enc + ((size_t)b * Ts + grp + i * G) * E + x);
  }
  const int len = min(max(p.lens[b], 0), Ts);
  if (threadIdx.x < 32) row_softmax(p, e, b, len, a_sh);
  __syncthreads();
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < Ts; j += kCtxThreads * kCtxGroups) {
      p.a[(size_t)b * Ts + j] = a_sh[j];
      p.accum_out[(size_t)b * Ts + j] = p.accum[(size_t)b * Ts + j] + a_sh[j];
    }
  float* part = a_sh + round_up_dev(Ts, 8);
  Vec<VE> s;
  s.zero();
  if (x < E) {
    int j = grp;
    if (use_pre) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float aj = a_sh[grp + i * G];
#pragma unroll
        for (int w = 0; w < VE; ++w) s.f[w] += aj * pre[i].f[w];
      }
      j = grp + 4 * G;
    }
    for (; j + 3 * G < len; j += 4 * G) {  // 4 independent loads in flight per thread
      Vec<VE> q[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) q[i].load(p.enc + ((size_t)b * Ts + j + i * G) * E + x);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float aj = a_sh[j + i * G];
#pragma unroll
        for (int w = 0; w < VE; ++w) s.f[w] += aj * q[i].f[w];
      }
    }
    for (; j < len; j += G) {
      Vec<VE> q;
      q.load(p.enc + ((size_t)b * Ts + j) * E + x);
      const float aj = a_sh[j];
#pragma unroll
      for (int w = 0; w < VE; ++w) s.f[w] += aj * q.f[w];
    }
    if (grp > 0) s.store(part + ((grp - 1) * kCtxThreads + ct) * VE);
  }
  __syncthreads();
  if (grp == 0 && x < E) {
#pragma unroll
    for (int g = 1; g < kCtxGroups; ++g) {
      Vec<VE> o;
      o.load_plain(part + ((g - 1) * kCtxThreads + ct) * VE);
#pragma unroll
      for (int w = 0; w < VE; ++w) s.f[w] += o.f[w];
    }
    s.store(p.att + (size_t)b * E + x);
#pragma unroll
    for (int c = 0; c < 2; ++c)
      if (p.att_copy[c]) s.store(p.att_copy[c] + (size_t)b * p.att_copy_ld[c] + x);
    if (p.att_img) {  // att's split image rows (hi, lo)
      __nv_bfloat16* dst = p.att_img + (size_t)b * p.att_img_ld + x;
#pragma unroll
      for (int w = 0; w < VE; ++w) {
        const __nv_bfloat16 h = __float2bfloat16_rn(s.f[w]);
        dst[w] = h;
        dst[p.att_img_lo + w] = __float2bfloat16_rn(s.f[w] - __bfloat162float(h));
      }
    }
  }
}

// backward 1: d_a[b, j] = <d_att_b, enc_bj> (valid j; tape.cpp:1031-1041) and
// d enc_bj = a_j d_att_b (every j of the chunk: zero at padded positions)
template <int VE>
__global__ void __launch_bounds__(kThreads, 2) attn_bwd_da_kernel(AttnArgs p, float* __restrict__ d_a) {
  __shared__ float red[kWarps * kJC];
  const int b = blockIdx.y, j0 = blockIdx.x * kJC, Ts = p.Ts, E = p.E;
  const int n = min(kJC, Ts - j0);
  float part[kJC], aj[kJC];
  if (p.defer && E <= kThreads * VE) {
    // deferred mode (the decoder's loop): only the dot products — every encoder row of
    // the chunk is loaded at once (no dependency on the row's length; 2 CTAs per SM so
    // the registers hold them), the length only masks the sums
    const int x = threadIdx.x * VE;
    Vec<VE> g;
    constexpr int kHalf = kJC / 2;
    const int len = min(max(p.lens[b], 0), Ts);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two batches of kJC / 2 rows in flight
      Vec<VE> q[kHalf];
      if (x < E) {
        if (h == 0) g.load(p.d_att + (size_t)b * E + x);
#pragma unroll
        for (int j = 0; j < kHalf; ++j)
          if (h * kHalf + j < n) q[j].load(p.enc + ((size_t)b * Ts + j0 + h * kHalf + j) * E + x);
      }
#pragma unroll
      for (int j = 0; j < kHalf; ++j) {
        const int jj = h * kHalf + j;
        part[jj] = 0.f;
        if (x < E && jj < n && j0 + jj < len) {
#pragma unroll
          for (int w = 0; w < VE; ++w) part[jj] += g.f[w] * q[j].f[w];
        }
      }
    }
    block_reduce_chunk(part, n, red, d_a + (size_t)b * Ts + j0);
    return;
  }
  const int len = min(max(p.lens[b], 0), Ts);
#pragma unroll
  for (int j = 0; j < kJC; ++j) {
    part[j] = 0.f;
    aj[j] = j < n ? __ldg(p.a_saved + (size_t)b * Ts + j0 + j) : 0.f;
  }
  for (int x = threadIdx.x * VE; x < E; x += kThreads * VE) {
    Vec<VE> g;
    g.load(p.d_att + (size_t)b * E + x);
#pragma unroll
    for (int j = 0; j < kJC; ++j) {
      if (j < n) {
        const size_t off = ((size_t)b * Ts + j0 + j) * E + x;
        if (!p.defer) {
          Vec<VE> o;
          if (p.accumulate) o.load_plain(p.d_enc + off);
          else o.zero();
#pragma unroll
          for (int w = 0; w < VE; ++w) o.f[w] += aj[j] * g.f[w];
          o.store(p.d_enc + off);
        }
        if (j0 + j < len) {
          Vec<VE> q;
          q.load(p.enc + off);
#pragma unroll
          for (int w = 0; w < VE; ++w) part[j] += g.f[w] * q.f[w];
        }
      }
    }
  }
  block_reduce_chunk(part, n, red, d_a + (size_t)b * Ts + j0);
}

// backward 2: softmax adjoint of the row (tape.cpp:966-978; + d accum', masked),
// then through tanh for the chunk: d e_in[j, k] = d_e_j v_k (1 - u^2) -> d enc_ctx,
// d accum_j = d accum'_j + <d e_in[j], W_fb>, and the column sums d s_tr[b] /
// d b_fb / d W_fb / d v (per-thread over the chunk, then vector atomics)
template <int VK, bool DEFER>
__global__ void __launch_bounds__(kThreads, DEFER ? 3 : 2) attn_bwd_de_kernel(AttnArgs p, const float* __restrict__ d_a) {
  __shared__ float red[kWarps * kJE];
  __shared__ float de_sh[kJE], sum_sh[kJE];
  const int b = blockIdx.y, j0 = blockIdx.x * kJE, Ts = p.Ts, K = p.K;
  const int n = min(kJE, Ts - j0);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // The chunk's energy inputs and column constants do not depend on the row's length
  // or on d a: their loads go out first, so the latency of the dependent prologue
  // below (length -> softmax-adjoint dot -> de) hides under them.
  const int k_first = threadIdx.x * VK;
  Vec<VK> c0, w0, v0, x0[kJE];
  float acc[kJE];
  if (k_first < K) {
    load_cols(p, b, k_first, c0, w0, v0);
#pragma unroll
    for (int j = 0; j < kJE; ++j)
      if (j < n) x0[j].load(p.enc_ctx + ((size_t)b * Ts + j0 + j) * K + k_first);
  }
#pragma unroll
  for (int j = 0; j < kJE; ++j) acc[j] = j < n ? __ldg(p.accum + (size_t)b * Ts + j0 + j) : 0.f;
  const int len = min(max(p.lens[b], 0), Ts);
  const float* da_b = d_a + (size_t)b * Ts;
  const float* a_b = p.a_saved + (size_t)b * Ts;
  const float* up_b = p.d_accum_out ? p.d_accum_out + (size_t)b * Ts : nullptr;
  if (warp == 0) {
    float dot = 0.f;
    for (int j = lane; j < len; j += 32) dot += (da_b[j] + (up_b ? up_b[j] : 0.f)) * a_b[j];
    dot = warp_sum(dot);
    float dbv = 0.f;
    if (lane < kJE) {
      const int jj = j0 + lane;
      const float d = (lane < n && jj < len) ? a_b[jj] * (da_b[jj] + (up_b ? up_b[jj] : 0.f) - dot) : 0.f;
      de_sh[lane] = d;
      dbv = d;
      if (p.de_out && lane < n) p.de_out[(size_t)b * Ts + jj] = d;
    }
    dbv = warp_sum(dbv);
    if (lane == 0 && dbv != 0.f && !p.defer) atomicAdd(p.d_b_v, dbv);
  }
  __syncthreads();
  float part[kJE], de[kJE];
#pragma unroll
  for (int j = 0; j < kJE; ++j) {
    part[j] = 0.f;
    de[j] = de_sh[j];
  }
  const int nv = max(0, min(n, len - j0));  // valid positions of the chunk
  auto cols = [&](int k, const Vec<VK>& c, const Vec<VK>& w, const Vec<VK>& v, const Vec<VK>(&x)[kJE]) {
    if constexpr (VK % 2 == 0 && DEFER) {
      {  // only d s_tr and d accum: paired-fp32 math (two columns per instruction)
        using namespace fm;
        float2 ds2[VK / 2];
#pragma unroll
        for (int i = 0; i < VK / 2; ++i) ds2[i] = s2(0.f);
#pragma unroll
        for (int j = 0; j < kJE; ++j) {
          if (j < nv) {
            float2 pj = s2(0.f);
#pragma unroll
            for (int i = 0; i < VK / 2; ++i) {
              const float2 w2 = make_float2(w.f[2 * i], w.f[2 * i + 1]);
              const float2 c2 = make_float2(c.f[2 * i], c.f[2 * i + 1]);
              const float2 v2 = make_float2(v.f[2 * i], v.f[2 * i + 1]);
              const float2 x2 = make_float2(x[j].f[2 * i], x[j].f[2 * i + 1]);
              const float2 u = tanh2(fma2(s2(acc[j]), w2, add2(x2, c2)));
              const float2 gk = mul2(mul2(s2(de[j]), v2), fma2(make_float2(-u.x, -u.y), u, s2(1.f)));
              ds2[i] = add2(ds2[i], gk);
              pj = fma2(gk, w2, pj);
            }
            part[j] += pj.x + pj.y;
          }
        }
        // this chunk's d s_tr partial (every chunk writes, zeros past the length): summed
        // in chunk order by attn_ds_sum_split_kernel — deterministic, no atomics
        Vec<VK> ds;
#pragma unroll
        for (int i = 0; i < VK / 2; ++i) ds.f[2 * i] = ds2[i].x, ds.f[2 * i + 1] = ds2[i].y;
        ds.store(p.ds_part + ((size_t)blockIdx.x * p.B + b) * K + k);
        return;
      }
    }
    Vec<VK> ds, dwf, dv;
    ds.zero(), dwf.zero(), dv.zero();
#pragma unroll
    for (int j = 0; j < kJE; ++j) {
      if (j < n) {
        const size_t off = ((size_t)b * Ts + j0 + j) * K + k;
        Vec<VK> gk;
        if (j < nv) {
#pragma unroll
          for (int i = 0; i < VK; ++i) {
            const float u = tanh_fast(x[j].f[i] + acc[j] * w.f[i] + c.f[i]);
            gk.f[i] = de[j] * v.f[i] * (1.f - u * u);
            ds.f[i] += gk.f[i];
            dwf.f[i] += acc[j] * gk.f[i];
            dv.f[i] += u * de[j];
            part[j] += gk.f[i] * w.f[i];
          }
        } else {
          gk.zero();
        }
        if (!p.defer) {
          if (p.accumulate) {
            Vec<VK> o;
            o.load_plain(p.d_enc_ctx + off);
#pragma unroll
            for (int i = 0; i < VK; ++i) gk.f[i] += o.f[i];
          }
          gk.store(p.d_enc_ctx + off);
        }
      }
    }
    if (nv > 0) {
      ds.atomic_add(p.d_s_tr + (size_t)b * K + k);
      if (!p.defer) {
        ds.atomic_add(p.d_b_fb + k);
        dwf.atomic_add(p.d_W_fb + k);
        dv.atomic_add(p.d_v + k);
      }
    }
  };
  if (k_first < K) cols(k_first, c0, w0, v0, x0);
  for (int k = k_first + kThreads * VK; k < K; k += kThreads * VK) {
    Vec<VK> c, w, v, x[kJE];
    load_cols(p, b, k, c, w, v);
#pragma unroll
    for (int j = 0; j < kJE; ++j)
      if (j < nv) x[j].load(p.enc_ctx + ((size_t)b * Ts + j0 + j) * K + k);
    cols(k, c, w, v, x);
  }
  block_reduce_chunk(part, n, red, sum_sh);
  __syncthreads();
  if (threadIdx.x < n) {
    const int jj = j0 + threadIdx.x;
    const float up = (jj < len && up_b) ? up_b[jj] : 0.f;
    float* ga = p.d_accum + (size_t)b * Ts + jj;
    *ga = (p.accumulate && !p.d_accum_fresh ? *ga : 0.f) + up + (jj < len ? sum_sh[threadIdx.x] : 0.f);
  }
}

// d s_tr = sum over the source chunks (in order) of the tanh pass's partials, written
// as fp32 (the deferred d W_s GEMM's operand) and as its split image (the per-step
// d s = d s_tr W_s^T GEMM's A operand: hi [B, ld], lo lo_off further on)
__global__ void attn_ds_sum_split_kernel(const float* __restrict__ part, int nchunk, int B, int K, float* out,
                                         __nv_bfloat16* img, int64_t ld, int64_t lo_off) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * ld) return;
  const int b = (int)(i / ld), k = (int)(i % ld);
  float v = 0.f;
  if (k < K) {
    for (int c = 0; c < nchunk; ++c) v += __ldg(part + ((size_t)c * B + b) * K + k);
    out[(size_t)b * K + k] = v;
  }
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  img[i] = h;
  img[lo_off + i] = __float2bfloat16_rn(v - __bfloat162float(h));
}

// the same for 4 consecutive k per thread (K % 4 == 0, ld % 4 == 0)
__global__ void attn_ds_sum_split4_kernel(const float* __restrict__ part, int nchunk, int B, int K, float* out,
                                          __nv_bfloat16* img, int64_t ld, int64_t lo_off) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= (int64_t)B * ld) return;
  const int b = (int)(i / ld), k = (int)(i % ld);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (k < K) {
    for (int c = 0; c < nchunk; ++c) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(part + ((size_t)c * B + b) * K + k));
      v.x += t.x, v.y += t.y, v.z += t.z, v.w += t.w;
    }
    *reinterpret_cast<float4*>(out + (size_t)b * K + k) = v;
  }
  const float f[4] = {v.x, v.y, v.z, v.w};
  __nv_bfloat16 hi[4], lo[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    hi[u] = __float2bfloat16_rn(f[u]);
    lo[u] = __float2bfloat16_rn(f[u] - __bfloat162float(hi[u]));
  }
  *reinterpret_cast<uint2*>(img + i) = *reinterpret_cast<const uint2*>(hi);
  *reinterpret_cast<uint2*>(img + lo_off + i) = *reinterpret_cast<const uint2*>(lo);
}

// column sums of d_s_tr [B, K] into d_b_s (+=)
__global__ void colsum_kernel(const float* x, int rows, int cols, float* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int r = 0; r < rows; ++r) s += x[(size_t)r * cols + c];
  out[c] += s;
}

}  // namespace

// workspace: s_tr [B, K] | d_s_tr [B, K] | e / d_a [B, Ts] | split-bf16 operands of the projection GEMMs
static size_t x3_bytes(int B, int K, int H) {
  return std::max({gemm_f32x3_workspace_bytes(false, false, B, K, H, false),   // s_tr = s W_s
                   gemm_f32x3_workspace_bytes(false, true, B, H, K, false),    // d s = d s_tr W_s^T
                   gemm_f32x3_workspace_bytes(true, false, H, K, B, true),     // [d W_s; d b_s]
                   gemm_f32x3_parts_workspace_bytes(false, false, B, K, H),    // (as partials)
                   gemm_f32x3_parts_workspace_bytes(false, true, B, H, K)});
}
static size_t ws_head(int B, int K, int Ts) {
  return (size_t)round_up((int64_t)2 * B * K * sizeof(float), 256) + (size_t)round_up((int64_t)B * Ts * 4, 256);
}
// after the GEMM scratch: the deferred backward's per-chunk d s_tr partials
static size_t ds_part_bytes(int B, int K, int Ts) { return (size_t)ceil_div(Ts, kJE) * B * K * sizeof(float); }
size_t attention_workspace_bytes(int B, int K, int H, int Ts) {
  return ws_head(B, K, Ts) + round_up(x3_bytes(B, K, H), 256) + ds_part_bytes(B, K, Ts) + 256;
}
static float* ds_part_buf(const AttnArgs& p, void* ws) {
  return reinterpret_cast<float*>(static_cast<char*>(ws) + ws_head(p.B, p.K, p.Ts) + round_up(x3_bytes(p.B, p.K, p.H), 256));
}
static float* row_buf(const AttnArgs& p, void* ws) {  // e (forward) / d_a (backward) [B, Ts]
  return reinterpret_cast<float*>(static_cast<char*>(ws) + round_up((int64_t)2 * p.B * p.K * sizeof(float), 256));
}
static void* x3_ws(const AttnArgs& p, void* ws) { return static_cast<char*>(ws) + ws_head(p.B, p.K, p.Ts); }

static bool al16(const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15) == 0; }
static bool al32(const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 31) == 0; }
// vector widths: 4 key / 8 encoder columns per thread when every row stays 16 B aligned
static int vec_k(const AttnArgs& p) {
  return (p.K % 4 == 0 && al16(p.enc_ctx) && al16(p.d_enc_ctx) && al16(p.s_tr) && al16(p.d_s_tr) && al16(p.b_fb) &&
          al16(p.W_fb) && al16(p.v) && al16(p.d_W_fb) && al16(p.d_b_fb) && al16(p.d_v))
             ? 4
             : 1;
}
static int vec_e(const AttnArgs& p) {
  bool copies = true;  // the copies' rows take the float4 stores
  for (int c = 0; c < 2; ++c) copies = copies && al16(p.att_copy[c]) && p.att_copy_ld[c] % 4 == 0;
  return (p.E % 8 == 0 && al32(p.enc) && al32(p.d_enc) && al32(p.d_att) && al32(p.att) && copies) ? 8 : 1;
}

void attention_fwd(AttnArgs p, const float* s, const float* W_s, const float* b_s, void* ws, cudaStream_t st) {
  p.s_tr = p.s_tr_out ? p.s_tr_out : static_cast<float*>(ws);
  if (p.W_s3_fwd)  // s_tr = s W_s + b_s (s from its image rows when given)
    gemm_f32x3_ex(false, false, p.B, p.K, p.H, s, p.H, p.s_img, nullptr, 0, p.W_s3_fwd, 0.f, p.s_tr, p.K, b_s,
                  nullptr, 0, x3_ws(p, ws), st, p.s_img ? p.s_img_ld : 0, p.s_img ? p.s_img_lo : 0);
  else
    gemm_f32x3(false, false, p.B, p.K, p.H, s, p.H, W_s, p.K, 0.f, p.s_tr, p.K, b_s, nullptr, 0, x3_ws(p, ws), st);
  float* e = row_buf(p, ws);
  Phase ph(st, "k8_attention_fwd", 0.0, 4.0 * p.B * p.Ts * (double)(p.K + p.E));
  const dim3 g1((unsigned)ceil_div(p.Ts, kJE), (unsigned)p.B);
  if (vec_k(p) == 4) attn_energy_kernel<4><<<g1, kThreads, 0, st>>>(p, e);
  else attn_energy_kernel<1><<<g1, kThreads, 0, st>>>(p, e);
  SL_CUDA_TRY(cudaGetLastError());
  const int ve = vec_e(p);
  const dim3 g2((unsigned)ceil_div(p.E, kCtxThreads * ve), (unsigned)p.B);
  const size_t smem = (size_t)(round_up(p.Ts, 8) + (kCtxGroups - 1) * kCtxThreads * ve) * sizeof(float);
  SL_REQUIRE(smem <= 48 * 1024, SL_ERR_UNSUPPORTED, "attention: src_time too large");
  if (ve == 8) attn_context_kernel<8><<<g2, kCtxThreads * kCtxGroups, smem, st>>>(p, e);
  else attn_context_kernel<1><<<g2, kCtxThreads * kCtxGroups, smem, st>>>(p, e);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch(2);
}

void attention_bwd(AttnArgs p, const float* s, const float* W_s, const float* b_s, float* d_s, float* d_W_s,
                   float* d_b_s, void* ws, cudaStream_t st) {
  p.d_s_tr = p.d_s_tr_out ? p.d_s_tr_out : static_cast<float*>(ws) + (size_t)p.B * p.K;
  if (p.s_tr_in) {  // the forward's s_tr
    p.s_tr = const_cast<float*>(p.s_tr_in);
  } else {  // recompute s_tr
    p.s_tr = static_cast<float*>(ws);
    gemm_f32x3(false, false, p.B, p.K, p.H, s, p.H, W_s, p.K, 0.f, p.s_tr, p.K, b_s, nullptr, 0, x3_ws(p, ws), st);
  }
  if (!p.accumulate && !p.defer) {
    SL_CUDA_TRY(cudaMemsetAsync(p.d_W_fb, 0, sizeof(float) * p.K, st));
    SL_CUDA_TRY(cudaMemsetAsync(p.d_b_fb, 0, sizeof(float) * p.K, st));
    SL_CUDA_TRY(cudaMemsetAsync(p.d_v, 0, sizeof(float) * p.K, st));
    SL_CUDA_TRY(cudaMemsetAsync(p.d_b_v, 0, sizeof(float), st));
    if (d_b_s && !d_W_s) SL_CUDA_TRY(cudaMemsetAsync(d_b_s, 0, sizeof(float) * p.K, st));
  }
  float* d_a = row_buf(p, ws);
  const bool ds_split = p.defer && vec_k(p) == 4;  // the paired tanh pass writes per-chunk partials
  p.ds_part = ds_split ? ds_part_buf(p, ws) : nullptr;
  if (!ds_split) SL_CUDA_TRY(cudaMemsetAsync(p.d_s_tr, 0, sizeof(float) * p.B * p.K, st));
  {
    Phase ph(st, "k8_attention_bwd", 0.0, 4.0 * p.B * p.Ts * (double)(2 * p.K + 2 * p.E));
    const dim3 g((unsigned)ceil_div(p.Ts, kJC), (unsigned)p.B), ge((unsigned)ceil_div(p.Ts, kJE), (unsigned)p.B);
    if (vec_e(p) == 8) attn_bwd_da_kernel<8><<<g, kThreads, 0, st>>>(p, d_a);
    else attn_bwd_da_kernel<1><<<g, kThreads, 0, st>>>(p, d_a);
    SL_CUDA_TRY(cudaGetLastError());
    if (vec_k(p) == 4 && p.defer) attn_bwd_de_kernel<4, true><<<ge, kThreads, 0, st>>>(p, d_a);
    else if (vec_k(p) == 4) attn_bwd_de_kernel<4, false><<<ge, kThreads, 0, st>>>(p, d_a);
    else attn_bwd_de_kernel<1, false><<<ge, kThreads, 0, st>>>(p, d_a);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch(2);
  }
  const float beta = p.accumulate ? 1.f : 0.f;
  const __nv_bfloat16* ds_img = nullptr;  // d s_tr's split image (deferred mode)
  const int64_t ds_ld = x3_img_ld(p.K);
  if (ds_split) {  // d s_tr = the chunks' partials summed in order, + its image for the d s GEMM
    auto* img = static_cast<__nv_bfloat16*>(x3_ws(p, ws));  // the GEMM scratch's A-image slot
    const int nchunk = (int)ceil_div(p.Ts, kJE);
    if (p.K % 4 == 0 && ds_ld % 4 == 0 && al16(p.d_s_tr) && al16(p.ds_part))
      attn_ds_sum_split4_kernel<<<(unsigned)ceil_div((int64_t)p.B * ds_ld / 4, 256), 256, 0, st>>>(
          p.ds_part, nchunk, p.B, p.K, p.d_s_tr, img, ds_ld, (int64_t)p.B * ds_ld);
    else
      attn_ds_sum_split_kernel<<<(unsigned)ceil_div((int64_t)p.B * ds_ld, 256), 256, 0, st>>>(
          p.ds_part, nchunk, p.B, p.K, p.d_s_tr, img, ds_ld, (int64_t)p.B * ds_ld);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
    ds_img = img;
  }
  if (d_s && p.W_s3_bwd && p.ds_parts_out)  // d s = d s_tr W_s^T, summed by the caller's consumer
    *p.ds_parts_out = gemm_f32x3_parts(false, true, p.B, p.H, p.K, p.d_s_tr, p.K, ds_img, nullptr, 0, p.W_s3_bwd,
                                       x3_ws(p, ws), st, ds_img ? ds_ld : 0, ds_img ? (int64_t)p.B * ds_ld : 0);
  else if (d_s && p.W_s3_bwd)  // d s = d s_tr W_s^T
    gemm_f32x3_pb(false, true, p.B, p.H, p.K, p.d_s_tr, p.K, p.W_s3_bwd, beta, d_s, p.H, nullptr, x3_ws(p, ws), st);
  else if (d_s)
    gemm_f32x3(false, true, p.B, p.H, p.K, p.d_s_tr, p.K, W_s, p.K, beta, d_s, p.H, nullptr, nullptr, 0,
               x3_ws(p, ws), st);
  if (d_W_s)  // [d W_s; d b_s] = [s | 1]^T d s_tr
    gemm_f32x3(true, false, p.H, p.K, p.B, s, p.H, p.d_s_tr, p.K, beta, d_W_s, p.K, nullptr, d_b_s, p.K,
               x3_ws(p, ws), st);
  else if (d_b_s) {
    colsum_kernel<<<(unsigned)ceil_div(p.K, 256), 256, 0, st>>>(p.d_s_tr, p.B, p.K, d_b_s);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
}

}  // namespace sl
