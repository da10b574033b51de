// The Listing-1 attention decoder over a teacher-forced target sequence
// (SURVEY §8 f1 + the decoder cell it feeds): the reference's `output`
// subnetwork (models.cpp:83-166, evaluated step by step by compiler.cpp's
// loop, 770-905) plus the base layer enc_ctx (models.cpp:60):
//
//   enc_ctx = enc W_ctx + b_ctx                                 (once)
//   for t:  s_t, c_t = lstm_step([trg_{t-1} ‖ att_{t-1}], s_{t-1}, c_{t-1})   (tape.cpp:1074-1141)
//           s_tr = s_t W_s + b_s
//           e    = tanh(enc_ctx + accum_{t-1} W_fb + b_fb + s_tr) v + b_v
//           a_t  = softmax over the valid source positions;  accum_t = accum_{t-1} + a_t
//           att_t = sum_j a_t[j] enc_j
//   readout = relu([s ‖ trg_prev ‖ att] W_ro + b_ro)           (all t at once)
//
// trg_{t-1} is the `trg` embedding of the previous target (zero at t = 0:
// initial_output 0, compiler.cpp:674-697), att_{-1} = s_{-1} = c_{-1} = 0.
//
// B200 design (bf16 operands, fp32 accumulation and cell state — the
// SL_PREC_BF16 contract):
//  * Everything that does not sit on the recurrence is hoisted into whole-
//    sequence tensor-core GEMMs: enc_ctx, the trg part of the cell input
//    (x W_trg + b for all t), the readout and, in the backward, every weight
//    gradient (one GEMM over all B*T rows each — the reference adds per-step
//    dW temporaries, tape.cpp:1174-1215) and d trg / d enc.
//  * Per step only the serial work remains: one split-K GEMM [att ‖ s] W_{att,R}
//    whose partial products are summed inside the gate kernel, the small s_tr
//    GEMM, and ONE attention kernel per batch row (energies + masked softmax +
//    context in one pass over that row's enc_ctx / enc, both bf16 and small
//    enough to stay L2-resident across the steps).
//  * Backward: the per-step attention kernel computes only what the
//    recurrence needs (d s_tr and d accum_{t-1}); the big accumulations over t
//    — d enc_ctx, d W_fb, d b_fb, d v, d enc = sum_t a_t (x) d att_t — run once
//    after the loop from small saved per-step vectors (a_t, d att_t, de_t),
//    recomputing tanh in registers, so the loop never read-modify-writes a
//    [B, Ts, K] accumulator.  All reductions are fixed-order (deterministic).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <memory>

#include "convert.h"
#include "decoder.h"
#include "embedding.h"
#include "gemm.h"
#include "profile.h"
#include "tc.cuh"

namespace sl {
namespace {

using bf16 = __nv_bfloat16;

constexpr int kAttThreads = 512;
constexpr int kAttWarps = kAttThreads / 32;
constexpr int kCtxPos = 8;  // source positions per CTA in the pass-2 d enc_ctx kernel

__constant__ int c_tanh_mode;  // 0: tanh.approx.f32 (one MUFU op), 1: 1 - 2 / (1 + e^{2x}) (two, ~1e-7 abs)
__device__ __forceinline__ float tanh_approx(float x) {
  if (c_tanh_mode) {
    x = fminf(fmaxf(x, -15.f), 15.f);
    return 1.f - __fdividef(2.f, 1.f + __expf(2.f * x));
  }
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// split cluster barrier: announce this CTA has started (its shared memory exists) early,
// wait for the peer just before the first remote shared-memory access
__device__ __forceinline__ void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
// bulk L2 prefetch of a contiguous 16 B-aligned range (multiple of 16 B): one instruction
// puts a whole row segment in flight, so a later phase's loads hit L2
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
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
__device__ __forceinline__ void unpack8(const uint4& q, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x, f[2 * i + 1] = v.y;
  }
}
__device__ __forceinline__ void ld8(const bf16* p, float (&f)[8]) { unpack8(*reinterpret_cast<const uint4*>(p), f); }
__device__ __forceinline__ void ld4(const bf16* p, float (&f)[4]) {
  const uint2 q = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.y));
  f[0] = a.x, f[1] = a.y, f[2] = b.x, f[3] = b.y;
}
__device__ __forceinline__ void st4(bf16* p, const float (&f)[4]) {
  const __nv_bfloat162 lo = __floats2bfloat162_rn(f[0], f[1]), hi = __floats2bfloat162_rn(f[2], f[3]);
  *reinterpret_cast<uint2*>(p) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
}
__device__ __forceinline__ float4 ldf4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void stf4(float* p, const float (&f)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
}
__device__ __forceinline__ void addf4(float (&a)[4], const float4& v) { a[0] += v.x, a[1] += v.y, a[2] += v.z, a[3] += v.w; }

// ---- decoder cell (reference tape.cpp:1095-1135 forward, 1157-1170 adjoint) --------------
struct CellFwd {
  int B, T, H, E, t, nsplit;
  const float* P;  // split-K partials of [att ‖ s]_{t-1} W_{att,R}: [z][B][p_ld]
  int64_t p_ld, p_stride;
  const float* xw;  // [B*T, 4H]: trg_{t-1} W_trg + b (hoisted)
  float* c_all;     // [B*T, H]
  float* gates;     // [B*T, 5H]: i f g o tanh(c)
  bf16* xa;         // [T*B, pxa] (time-major rows t*B + b): s_t -> row (t+1, b), column E
  int64_t pxa;
  bf16* ro;  // [T*B, pro]: s_t -> row (t, b), column 0
  int64_t pro;
};

__global__ void dec_cell_fwd_kernel(CellFwd a) {
  const int qn = a.H / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.B * qn) return;
  const int b = idx / qn, j = (idx - b * qn) * 4;
  const int64_t row = (int64_t)a.t * a.B + b;  // every per-step buffer is time-major: a step is contiguous
  const int H = a.H;
  float z[4][4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const float4 v = ldf4(a.xw + row * 4 * H + g * H + j);
    z[g][0] = v.x, z[g][1] = v.y, z[g][2] = v.z, z[g][3] = v.w;
  }
  for (int s = 0; s < a.nsplit; ++s) {
    const float* p = a.P + s * a.p_stride + (int64_t)b * a.p_ld + j;
#pragma unroll
    for (int g = 0; g < 4; ++g) addf4(z[g], ldf4(p + g * H));
  }
  float cp[4] = {0.f, 0.f, 0.f, 0.f};
  if (a.t > 0) {
    const float4 v = ldf4(a.c_all + (row - a.B) * H + j);
    cp[0] = v.x, cp[1] = v.y, cp[2] = v.z, cp[3] = v.w;
  }
  float gi[4], gf[4], gg[4], go[4], c[4], tc[4], h[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    gi[u] = sigmoidf_(z[0][u]);
    gf[u] = sigmoidf_(z[1][u]);
    gg[u] = tanhf(z[2][u]);
    go[u] = sigmoidf_(z[3][u]);
    c[u] = gf[u] * cp[u] + gi[u] * gg[u];
    tc[u] = tanhf(c[u]);
    h[u] = go[u] * tc[u];
  }
  stf4(a.c_all + row * H + j, c);
  float* gs = a.gates + row * 5 * H + j;
  stf4(gs, gi);
  stf4(gs + H, gf);
  stf4(gs + 2 * H, gg);
  stf4(gs + 3 * H, go);
  stf4(gs + 4 * H, tc);
  st4(a.ro + row * a.pro + j, h);
  if (a.t + 1 < a.T) st4(a.xa + (row + a.B) * a.pxa + a.E + j, h);
}

struct CellBwd {
  int B, T, H, E, t;
  int n1;  // G1 partials (DZ_{t+1} [W_att; R]^T): d h_t at columns E..E+H
  const float* P1;
  int64_t p1_ld, p1_stride;
  int n2;  // G2 partials (d s_tr_t W_s^T)
  const float* P2;
  int64_t p2_ld, p2_stride;
  const float* dro;  // readout-input gradient [B*T, prf], s at columns 0..H
  int64_t prf;
  const float* gates;
  const float* c_all;
  const float* dc_in;  // d c_t [B, H] (null at t = T-1)
  float* dc_out;       // d c_{t-1}
  bf16* dz;            // [B*T, pz]
  int64_t pz;
};

__global__ void dec_cell_bwd_kernel(CellBwd a) {
  const int qn = a.H / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.B * qn) return;
  const int b = idx / qn, j = (idx - b * qn) * 4;
  const int64_t row = (int64_t)a.t * a.B + b;
  const int H = a.H;
  float gh[4] = {0.f, 0.f, 0.f, 0.f}, gc[4] = {0.f, 0.f, 0.f, 0.f};
  addf4(gh, ldf4(a.dro + row * a.prf + j));
  for (int s = 0; s < a.n1; ++s) addf4(gh, ldf4(a.P1 + s * a.p1_stride + (int64_t)b * a.p1_ld + a.E + j));
  for (int s = 0; s < a.n2; ++s) addf4(gh, ldf4(a.P2 + s * a.p2_stride + (int64_t)b * a.p2_ld + j));
  if (a.dc_in) addf4(gc, ldf4(a.dc_in + (int64_t)b * H + j));
  const float* gs = a.gates + row * 5 * H + j;
  const float4 vi = ldf4(gs), vf = ldf4(gs + H), vg = ldf4(gs + 2 * H), vo = ldf4(gs + 3 * H), vt = ldf4(gs + 4 * H);
  const float gi[4] = {vi.x, vi.y, vi.z, vi.w}, gf[4] = {vf.x, vf.y, vf.z, vf.w}, gg[4] = {vg.x, vg.y, vg.z, vg.w},
              go[4] = {vo.x, vo.y, vo.z, vo.w}, tc[4] = {vt.x, vt.y, vt.z, vt.w};
  float cp[4] = {0.f, 0.f, 0.f, 0.f};
  if (a.t > 0) {
    const float4 v = ldf4(a.c_all + (row - a.B) * H + j);
    cp[0] = v.x, cp[1] = v.y, cp[2] = v.z, cp[3] = v.w;
  }
  float dzi[4], dzf[4], dzg[4], dzo[4], dcp[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float d_o = gh[u] * tc[u];
    const float dc = gc[u] + gh[u] * go[u] * (1.f - tc[u] * tc[u]);
    dcp[u] = dc * gf[u];
    dzi[u] = dc * gg[u] * gi[u] * (1.f - gi[u]);
    dzf[u] = dc * cp[u] * gf[u] * (1.f - gf[u]);
    dzg[u] = dc * gi[u] * (1.f - gg[u] * gg[u]);
    dzo[u] = d_o * go[u] * (1.f - go[u]);
  }
  bf16* d = a.dz + row * a.pz + j;
  st4(d, dzi);
  st4(d + H, dzf);
  st4(d + 2 * H, dzg);
  st4(d + 3 * H, dzo);
  stf4(a.dc_out + (int64_t)b * H + j, dcp);
}

// ---- attention step, one CTA per batch row ---------------------------------------------
struct AttFwd {
  int B, Ts, T, K, E, t, nsplit;
  const int32_t* lens;
  const float* P;  // split-K partials of s_t W_s: [z][B][p_ld]
  int64_t p_ld, p_stride;
  const float *b_s, *W_fb, *b_fb, *v, *b_v;
  const bf16* enc_ctx;  // [B*Ts, pk]
  int64_t pk;
  const bf16* enc;  // [B*Ts, ld_enc]
  int64_t ld_enc;
  float* str_all;  // [T][B][K]: s_tr (with b_s)
  float* a_all;    // [T][B][Ts]
  float* acc_all;  // [T+1][B][Ts]: acc_all[t] = accum_{t-1}
  bf16* ro;        // att_t -> row (t, b), column oa
  int64_t pro;
  int oa;
  bf16* xa;  // att_t -> row (t+1, b), column 0
  int64_t pxa;
};

// One CTA PAIR (a 2-CTA cluster) per batch row: CTA r takes the source positions
// s = r (mod 2) for the energies and half of the encoder columns for the context;
// the energies meet in both CTAs' shared memory over DSMEM.  Inside a CTA four
// groups of 128 threads split the positions and every thread owns 8 key columns
// (their s_tr, W_fb, v in registers); loads are issued four positions at a time
// so enough bytes are in flight to stream the row's enc_ctx / enc from L2.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kAttThreads) dec_attn_fwd_kernel(AttFwd a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ float sm[];
  const int Ts = a.Ts, K = a.K, tid = threadIdx.x, lane = tid % 32;
  const int r = (int)cl.block_rank(), b = blockIdx.x / 2;
  float* red = sm;            // [Ts][4] per-warp partial energies
  float* es = red + 4 * Ts;   // [Ts] energies, then a
  float* acc = es + Ts;       // [Ts] accum_{t-1}
  float* ctx = sm + (6 * Ts + 3) / 4 * 4;  // [256][4] context partials of the second position group (16 B aligned)
  cluster_arrive_relaxed();
  const int len = min(max(a.lens[b], 0), Ts);
  const size_t tb = (size_t)a.t * a.B + b;
  if (tid < 64) {  // this CTA's enc_ctx rows (energies) and enc column half (context) into L2 now
    for (int s = r + 2 * tid; s < len; s += 128)
      prefetch_l2(a.enc_ctx + ((int64_t)b * Ts + s) * a.pk, (uint32_t)K * 2);
  } else if (tid < 128) {
    for (int s = tid - 64; s < len; s += 64)
      prefetch_l2(a.enc + ((int64_t)b * Ts + s) * a.ld_enc + r * (a.E / 2), (uint32_t)a.E);
  }
  for (int s = tid; s < Ts; s += kAttThreads) acc[s] = a.acc_all[tb * Ts + s];
  const int g = tid / 128, q = tid % 128, wig = q / 32, k0 = q * 8;
  const bool act = k0 < K;
  float cv[8], wv[8], vk[8];
  if (act) {
    float st[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) st[i] = a.b_s[k0 + i];
    for (int z = 0; z < a.nsplit; ++z) {
      const float* pz = a.P + z * a.p_stride + (int64_t)b * a.p_ld + k0;
      const float4 u0 = ldf4(pz), u1 = ldf4(pz + 4);
      st[0] += u0.x, st[1] += u0.y, st[2] += u0.z, st[3] += u0.w;
      st[4] += u1.x, st[5] += u1.y, st[6] += u1.z, st[7] += u1.w;
    }
    if (r == 0 && g == 0) {
      const float s0[4] = {st[0], st[1], st[2], st[3]}, s1[4] = {st[4], st[5], st[6], st[7]};
      stf4(a.str_all + tb * K + k0, s0);
      stf4(a.str_all + tb * K + k0 + 4, s1);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      cv[i] = st[i] + a.b_fb[k0 + i];
      wv[i] = a.W_fb[k0 + i];
      vk[i] = a.v[k0 + i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = wv[i] = vk[i] = 0.f;
  }
  __syncthreads();
  // energies of this CTA's positions s = r + 2 (g + 4 m), four per batch
  for (int s0 = r + 2 * g; s0 < len; s0 += 32) {
    uint4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int s = s0 + 8 * u;
      x[u] = (act && s < len) ? *reinterpret_cast<const uint4*>(a.enc_ctx + ((int64_t)b * Ts + s) * a.pk + k0)
                              : make_uint4(0, 0, 0, 0);
    }
    float p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int s = s0 + 8 * u;
      float f[8];
      unpack8(x[u], f);
      const float as = s < len ? acc[s] : 0.f;
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += vk[i] * tanh_approx(f[i] + as * wv[i] + cv[i]);
      p[u] = warp_sum(act ? sum : 0.f);
    }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (s0 + 8 * u < len) red[(s0 + 8 * u) * 4 + wig] = p[u];
    }
  }
  __syncthreads();
  cluster_wait();
  float* peer_es = cl.map_shared_rank(es, r ^ 1);
  const float bv = *a.b_v;
  for (int s = r + 2 * tid; s < len; s += 2 * kAttThreads) {
    const float e = ((red[s * 4] + red[s * 4 + 1]) + red[s * 4 + 2]) + red[s * 4 + 3] + bv;
    es[s] = e;
    peer_es[s] = e;
  }
  cl.sync();
  if (tid < 32) {  // masked softmax over the valid positions (tape.cpp:952-960), in both CTAs
    float m = -INFINITY;
    for (int s = lane; s < len; s += 32) m = fmaxf(m, es[s]);
    m = warp_max(m);
    float sum = 0.f;
    for (int s = lane; s < len; s += 32) {
      const float ex = expf(es[s] - m);
      es[s] = ex;
      sum += ex;
    }
    sum = warp_sum(sum);
    const float inv = len > 0 ? 1.f / sum : 0.f;
    __syncwarp();
    for (int s = lane; s < Ts; s += 32) {
      const float av = s < len ? es[s] * inv : 0.f;
      es[s] = av;
      if (r == 0) {
        a.a_all[tb * Ts + s] = av;
        a.acc_all[((size_t)(a.t + 1) * a.B + b) * Ts + s] = acc[s] + av;
      }
    }
  }
  __syncthreads();
  {  // att = sum_s a_s enc_s (tape.cpp:1005-1014): this CTA's half of the columns, two position groups
    const int gc = tid / 256, qc = tid % 256, Eh = a.E / 2, e0 = r * Eh + qc * 4;
    const bool on = qc * 4 < Eh;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    const bf16* x = a.enc + (int64_t)b * Ts * a.ld_enc + e0;
    for (int s0 = gc; s0 < len; s0 += 8) {
      float f[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int s = s0 + 2 * u;
        if (on && s < len) ld4(x + (int64_t)s * a.ld_enc, f[u]);
        else f[u][0] = f[u][1] = f[u][2] = f[u][3] = 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float as = s0 + 2 * u < len ? es[s0 + 2 * u] : 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] += as * f[u][i];
      }
    }
    if (gc == 1 && on) stf4(ctx + qc * 4, o);
    __syncthreads();
    if (gc == 0 && on) {
      const float4 o2 = ldf4(ctx + qc * 4);
      o[0] += o2.x, o[1] += o2.y, o[2] += o2.z, o[3] += o2.w;
      const int64_t row = (int64_t)a.t * a.B + b;
      st4(a.ro + row * a.pro + a.oa + e0, o);
      if (a.t + 1 < a.T) st4(a.xa + (row + a.B) * a.pxa + e0, o);
    }
  }
}

struct AttBwd {
  int B, Ts, T, K, E, t, n1;
  const int32_t* lens;
  const float* P1;  // G1 partials: d att_t (from the cell at t+1) at columns 0..E
  int64_t p1_ld, p1_stride;
  const float* dro;  // readout-input gradient, att at column oa
  int64_t prf;
  int oa;
  const float *W_fb, *b_fb, *v;
  const bf16* enc_ctx;
  int64_t pk;
  const bf16* enc;
  int64_t ld_enc;
  const float *str_all, *a_all, *acc_all;
  const float* dacc_in;  // d accum_t [B][Ts] (null at t = T-1)
  float* dacc_out;       // d accum_{t-1}
  float* datt_all;       // [T][B][E]
  float* de_all;         // [T][B][Ts]
  bf16* ds;              // d s_tr -> row (t, b) of [T*B, pds]
  int64_t pds;
  float* ds32;  // [B*T, K]
};

// Adjoint of one attention step, restricted to what the recurrence needs:
// d_a = enc d_att + d accum_t (tape.cpp:1031-1041), de = a (d_a - <a, d_a>)
// (tape.cpp:966-978), d e_in = de v (1 - u^2) -> d s_tr = sum_s d e_in and
// d accum_{t-1} = d accum_t + d e_in W_fb.  One CTA pair per batch row (CTA r:
// positions s = r mod 2); d_a meets over DSMEM, the pair's d s_tr halves are
// summed in a fixed order by CTA 0.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kAttThreads) dec_attn_bwd_kernel(AttBwd a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ float sm[];
  const int K = a.K, Ts = a.Ts, E = a.E, tid = threadIdx.x, lane = tid % 32;
  const int r = (int)cl.block_rank(), b = blockIdx.x / 2;
  float* dsum = sm;             // [4][K]
  float* pdst = dsum + 4 * K;   // [K] this CTA's d s_tr
  float* av = pdst + K;         // [Ts]
  float* acc = av + Ts;         // [Ts]
  float* dacc = acc + Ts;       // [Ts] d accum_t
  float* da = dacc + Ts;        // [Ts]
  float* de = da + Ts;          // [Ts]
  float* red = de + Ts;         // [Ts][8]
  cluster_arrive_relaxed();
  const int len = min(max(a.lens[b], 0), Ts);
  const size_t tb = (size_t)a.t * a.B + b;
  const int64_t row = (int64_t)a.t * a.B + b;
  if (tid < 64) {  // this CTA's enc rows (d_a) and enc_ctx rows (tanh adjoint) into L2 now
    for (int s = r + 2 * tid; s < len; s += 128)
      prefetch_l2(a.enc + ((int64_t)b * Ts + s) * a.ld_enc, (uint32_t)E * 2);
  } else if (tid < 128) {
    for (int s = r + 2 * (tid - 64); s < len; s += 128)
      prefetch_l2(a.enc_ctx + ((int64_t)b * Ts + s) * a.pk, (uint32_t)K * 2);
  }
  for (int s = tid; s < Ts; s += kAttThreads) {
    av[s] = a.a_all[tb * Ts + s];
    acc[s] = a.acc_all[tb * Ts + s];
    dacc[s] = (a.dacc_in && s < len) ? a.dacc_in[(int64_t)b * Ts + s] : 0.f;
  }
  {  // d_a of this CTA's positions: two groups of 256 threads, 8 encoder columns each
    const int gc = tid / 256, qc = tid % 256, wig = qc / 32, e0 = qc * 8;
    const bool on = e0 < E;
    float dv[8];
    if (on) {
      const float* pd = a.dro + row * a.prf + a.oa + e0;
      const float4 u0 = ldf4(pd), u1 = ldf4(pd + 4);
      dv[0] = u0.x, dv[1] = u0.y, dv[2] = u0.z, dv[3] = u0.w, dv[4] = u1.x, dv[5] = u1.y, dv[6] = u1.z, dv[7] = u1.w;
      for (int z = 0; z < a.n1; ++z) {
        const float* pz = a.P1 + z * a.p1_stride + (int64_t)b * a.p1_ld + e0;
        const float4 w0 = ldf4(pz), w1 = ldf4(pz + 4);
        dv[0] += w0.x, dv[1] += w0.y, dv[2] += w0.z, dv[3] += w0.w;
        dv[4] += w1.x, dv[5] += w1.y, dv[6] += w1.z, dv[7] += w1.w;
      }
      if (r == 0 && gc == 0) {
        const float d0[4] = {dv[0], dv[1], dv[2], dv[3]}, d1[4] = {dv[4], dv[5], dv[6], dv[7]};
        stf4(a.datt_all + tb * E + e0, d0);
        stf4(a.datt_all + tb * E + e0 + 4, d1);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) dv[i] = 0.f;
    }
    for (int s0 = r + 2 * gc; s0 < len; s0 += 16) {  // positions s0, s0+4, s0+8, s0+12
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int s = s0 + 4 * u;
        x[u] = (on && s < len) ? *reinterpret_cast<const uint4*>(a.enc + ((int64_t)b * Ts + s) * a.ld_enc + e0)
                               : make_uint4(0, 0, 0, 0);
      }
      float p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float f[8];
        unpack8(x[u], f);
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) sum += dv[i] * f[i];
        p[u] = warp_sum(sum);
      }
      if (lane == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (s0 + 4 * u < len) red[(s0 + 4 * u) * 8 + wig] = p[u];
      }
    }
  }
  __syncthreads();
  cluster_wait();
  float* peer_da = cl.map_shared_rank(da, r ^ 1);
  for (int s = r + 2 * tid; s < len; s += 2 * kAttThreads) {
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += red[s * 8 + w];
    sum += dacc[s];
    da[s] = sum;
    peer_da[s] = sum;
  }
  cl.sync();
  if (tid < 32) {  // softmax adjoint, in both CTAs
    float dot = 0.f;
    for (int s = lane; s < len; s += 32) dot += av[s] * da[s];
    dot = warp_sum(dot);
    for (int s = lane; s < Ts; s += 32) {
      const float d = s < len ? av[s] * (da[s] - dot) : 0.f;
      de[s] = d;
      if (r == 0) a.de_all[tb * Ts + s] = d;
    }
  }
  __syncthreads();
  {  // tanh adjoint over this CTA's positions: four groups of 128 threads, 8 key columns each
    const int g = tid / 128, q = tid % 128, wig = q / 32, k0 = q * 8;
    const bool act = k0 < K;
    float wv[8], cv[8], vk[8], ds[8];
    if (act) {
      const float* st = a.str_all + tb * K + k0;
      const float4 s0v = ldf4(st), s1v = ldf4(st + 4);
      const float sv[8] = {s0v.x, s0v.y, s0v.z, s0v.w, s1v.x, s1v.y, s1v.z, s1v.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        wv[i] = a.W_fb[k0 + i];
        cv[i] = sv[i] + a.b_fb[k0 + i];
        vk[i] = a.v[k0 + i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) wv[i] = cv[i] = vk[i] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) ds[i] = 0.f;
    for (int s0 = r + 2 * g; s0 < len; s0 += 32) {  // positions s0 + 8u
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int s = s0 + 8 * u;
        x[u] = (act && s < len) ? *reinterpret_cast<const uint4*>(a.enc_ctx + ((int64_t)b * Ts + s) * a.pk + k0)
                                : make_uint4(0, 0, 0, 0);
      }
      float p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int s = s0 + 8 * u;
        const float as = s < len ? acc[s] : 0.f, des = s < len ? de[s] : 0.f;
        float f[8];
        unpack8(x[u], f);
        float pa = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float uu = tanh_approx(f[i] + as * wv[i] + cv[i]);
          const float dein = des * vk[i] * (1.f - uu * uu);
          ds[i] += dein;
          pa += wv[i] * dein;
        }
        p[u] = warp_sum(act ? pa : 0.f);
      }
      if (lane == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (s0 + 8 * u < len) red[(s0 + 8 * u) * 8 + wig] = p[u];  // (red reused: d_a is consumed)
      }
    }
    if (act) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dsum[g * K + k0 + i] = ds[i];
    }
  }
  __syncthreads();
  for (int k = tid; k < K; k += kAttThreads) pdst[k] = ((dsum[k] + dsum[K + k]) + dsum[2 * K + k]) + dsum[3 * K + k];
  for (int s = r + 2 * tid; s < Ts; s += 2 * kAttThreads)
    a.dacc_out[(int64_t)b * Ts + s] =
        s < len ? dacc[s] + (((red[s * 8] + red[s * 8 + 1]) + red[s * 8 + 2]) + red[s * 8 + 3]) : 0.f;
  cl.sync();
  if (r == 0) {
    const float* peer = cl.map_shared_rank(pdst, 1);
    for (int k = tid; k < K; k += kAttThreads) {
      const float d = pdst[k] + peer[k];
      a.ds32[row * K + k] = d;
      a.ds[row * a.pds + k] = __float2bfloat16_rn(d);
    }
  }
  cl.sync();  // CTA 1's shared memory stays alive until CTA 0 has read it
}

// ---- the same two attention kernels with the row's operands staged by TMA --------------
// C CTAs (one cluster) per batch row, 256 threads each.  CTA r owns the positions
// s = r (mod C) and, for the context, one 16 B-aligned column slice of enc; at
// kernel start one warp issues a 1-D bulk copy (cp.async.bulk) per row segment the
// CTA will read — its enc_ctx rows and enc slice in the forward, its enc and
// enc_ctx rows in the backward — completing on two mbarriers, so every byte is in
// flight at once and the phases then read shared memory.  ~95 KB per CTA: two
// CTAs per SM, one loading while the other computes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}
constexpr int kStThreads = 256;
__host__ __device__ inline int st_cols(int E, int C) { return ((E + C - 1) / C + 7) / 8 * 8; }
__host__ __device__ inline size_t st_align(size_t x) { return (x + 127) / 128 * 128; }
// shared-memory carve-ups (bytes), shared by host (launch size) and device
struct FwdSt {
  size_t red, es, acc, cpart, rctx, renc, total;
  __host__ __device__ FwdSt(int Ts, int K, int E, int C) {
    const int nrm = (Ts + C - 1) / C, Ec = st_cols(E, C);
    red = 16;
    es = red + (size_t)nrm * 4 * 4;
    acc = es + (size_t)Ts * 4;
    cpart = (acc + (size_t)Ts * 4 + 15) / 16 * 16;  // float4 accesses
    rctx = st_align(cpart + (size_t)Ec * 4);
    renc = st_align(rctx + (size_t)nrm * K * 2);
    total = renc + (size_t)Ts * Ec * 2;
  }
};
struct BwdSt {
  size_t av, acc, dacc, da, de, red, pdst, renc, rctx, total;
  __host__ __device__ BwdSt(int Ts, int K, int E, int C) {
    const int nrm = (Ts + C - 1) / C;
    av = 16;
    acc = av + (size_t)Ts * 4;
    dacc = acc + (size_t)Ts * 4;
    da = dacc + (size_t)Ts * 4;
    de = da + (size_t)Ts * 4;
    red = de + (size_t)Ts * 4;
    pdst = red + (size_t)nrm * 8 * 4;
    renc = st_align(pdst + (size_t)K * 4);
    const size_t renc_bytes = (size_t)nrm * E * 2, dsum_bytes = (size_t)2 * K * 4;
    rctx = st_align(renc + (renc_bytes > dsum_bytes ? renc_bytes : dsum_bytes));  // renc doubles as dsum [2][K]
    total = rctx + (size_t)nrm * K * 2;
  }
};

template <int C>
__global__ void __launch_bounds__(kStThreads) dec_attn_fwd_tma_kernel(AttFwd a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(128) uint8_t smraw[];
  const int Ts = a.Ts, K = a.K, E = a.E, tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int r = (int)cl.block_rank(), b = blockIdx.x / C;
  const FwdSt L(Ts, K, E, C);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw);
  float* red = reinterpret_cast<float*>(smraw + L.red);
  float* es = reinterpret_cast<float*>(smraw + L.es);
  float* acc = reinterpret_cast<float*>(smraw + L.acc);
  float* cpart = reinterpret_cast<float*>(smraw + L.cpart);
  bf16* rctx = reinterpret_cast<bf16*>(smraw + L.rctx);
  bf16* renc = reinterpret_cast<bf16*>(smraw + L.renc);
  const int Ec = st_cols(E, C), c0 = r * Ec, nc = max(0, min(E - c0, Ec));
  cluster_arrive_relaxed();
  const int len = min(max(a.lens[b], 0), Ts);
  const int nr = r < len ? (len - r + C - 1) / C : 0;  // this CTA's positions s = r + C j
  const size_t tb = (size_t)a.t * a.B + b;
  if (tid == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(&bars[0], (uint32_t)(nr * K * 2));
      tc::mbar_arrive_expect_tx(&bars[1], (uint32_t)(nc > 0 ? len * nc * 2 : 0));
    }
    __syncwarp();
    for (int j = lane; j < nr; j += 32)
      bulk_g2s(rctx + (size_t)j * K, a.enc_ctx + ((int64_t)b * Ts + r + C * j) * a.pk, (uint32_t)K * 2, &bars[0]);
    if (nc > 0)
      for (int s = lane; s < len; s += 32)
        bulk_g2s(renc + (size_t)s * Ec, a.enc + ((int64_t)b * Ts + s) * a.ld_enc + c0, (uint32_t)nc * 2, &bars[1]);
  }
  for (int s = tid; s < Ts; s += kStThreads) acc[s] = a.acc_all[tb * Ts + s];
  const int g = tid / 128, q = tid % 128, wig = q / 32, k0 = q * 8;
  const bool act = k0 < K;
  float cv[8], wv[8], vk[8];
  if (act) {
    float st[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) st[i] = a.b_s[k0 + i];
    for (int z = 0; z < a.nsplit; ++z) {
      const float* pz = a.P + z * a.p_stride + (int64_t)b * a.p_ld + k0;
      const float4 u0 = ldf4(pz), u1 = ldf4(pz + 4);
      st[0] += u0.x, st[1] += u0.y, st[2] += u0.z, st[3] += u0.w;
      st[4] += u1.x, st[5] += u1.y, st[6] += u1.z, st[7] += u1.w;
    }
    if (r == 0 && g == 0) {
      const float s0[4] = {st[0], st[1], st[2], st[3]}, s1[4] = {st[4], st[5], st[6], st[7]};
      stf4(a.str_all + tb * K + k0, s0);
      stf4(a.str_all + tb * K + k0 + 4, s1);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      cv[i] = st[i] + a.b_fb[k0 + i];
      wv[i] = a.W_fb[k0 + i];
      vk[i] = a.v[k0 + i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = wv[i] = vk[i] = 0.f;
  }
  __syncthreads();
  tc::mbar_wait(&bars[0], 0);
  for (int j = g; j < nr; j += 2) {  // e_s = <v, tanh(e_in_s)> over this CTA's positions
    const int s = r + C * j;
    float f[8];
    if (act) ld8(rctx + (size_t)j * K + k0, f);
    const float as = acc[s];
    float sum = 0.f;
    if (act) {
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += vk[i] * tanh_approx(f[i] + as * wv[i] + cv[i]);
    }
    sum = warp_sum(sum);
    if (lane == 0) red[j * 4 + wig] = sum;
  }
  __syncthreads();
  cluster_wait();
  const float bv = *a.b_v;
  for (int j = tid; j < nr; j += kStThreads) {
    const int s = r + C * j;
    const float e = ((red[j * 4] + red[j * 4 + 1]) + red[j * 4 + 2]) + red[j * 4 + 3] + bv;
#pragma unroll
    for (int p = 0; p < C; ++p) cl.map_shared_rank(es, p)[s] = e;
  }
  cl.sync();
  if (tid < 32) {  // masked softmax over the valid positions (tape.cpp:952-960), in every CTA
    float m = -INFINITY;
    for (int s = lane; s < len; s += 32) m = fmaxf(m, es[s]);
    m = warp_max(m);
    float sum = 0.f;
    for (int s = lane; s < len; s += 32) {
      const float ex = expf(es[s] - m);
      es[s] = ex;
      sum += ex;
    }
    sum = warp_sum(sum);
    const float inv = len > 0 ? 1.f / sum : 0.f;
    __syncwarp();
    for (int s = lane; s < Ts; s += 32) {
      const float av = s < len ? es[s] * inv : 0.f;
      es[s] = av;
      if (r == 0) {
        a.a_all[tb * Ts + s] = av;
        a.acc_all[((size_t)(a.t + 1) * a.B + b) * Ts + s] = acc[s] + av;
      }
    }
  }
  __syncthreads();
  {  // att (this CTA's column slice) = sum_s a_s enc_s (tape.cpp:1005-1014), two position groups
    const int gc = tid / 128, cq = tid % 128, cc = cq * 4;
    const bool on = cc < nc;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    if (nc > 0) tc::mbar_wait(&bars[1], 0);
    if (on) {
      for (int s = gc; s < len; s += 2) {
        float f[4];
        ld4(renc + (size_t)s * Ec + cc, f);
        const float as = es[s];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] += as * f[i];
      }
    }
    if (gc == 1 && on) stf4(cpart + cc, o);
    __syncthreads();
    if (gc == 0 && on) {
      const float4 o2 = ldf4(cpart + cc);
      o[0] += o2.x, o[1] += o2.y, o[2] += o2.z, o[3] += o2.w;
      const int64_t row = (int64_t)a.t * a.B + b;
      st4(a.ro + row * a.pro + a.oa + c0 + cc, o);
      if (a.t + 1 < a.T) st4(a.xa + (row + a.B) * a.pxa + c0 + cc, o);
    }
  }
}

template <int C>
__global__ void __launch_bounds__(kStThreads) dec_attn_bwd_tma_kernel(AttBwd a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(128) uint8_t smraw[];
  const int K = a.K, Ts = a.Ts, E = a.E, tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int r = (int)cl.block_rank(), b = blockIdx.x / C;
  const BwdSt L(Ts, K, E, C);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw);
  float* av = reinterpret_cast<float*>(smraw + L.av);
  float* acc = reinterpret_cast<float*>(smraw + L.acc);
  float* dacc = reinterpret_cast<float*>(smraw + L.dacc);
  float* da = reinterpret_cast<float*>(smraw + L.da);
  float* de = reinterpret_cast<float*>(smraw + L.de);
  float* red = reinterpret_cast<float*>(smraw + L.red);
  float* pdst = reinterpret_cast<float*>(smraw + L.pdst);
  bf16* renc = reinterpret_cast<bf16*>(smraw + L.renc);
  float* dsum = reinterpret_cast<float*>(smraw + L.renc);  // [2][K], after the d_a phase
  bf16* rctx = reinterpret_cast<bf16*>(smraw + L.rctx);
  cluster_arrive_relaxed();
  const int len = min(max(a.lens[b], 0), Ts);
  const int nr = r < len ? (len - r + C - 1) / C : 0;
  const size_t tb = (size_t)a.t * a.B + b;
  const int64_t row = (int64_t)a.t * a.B + b;
  if (tid == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(&bars[0], (uint32_t)(nr * E * 2));
      tc::mbar_arrive_expect_tx(&bars[1], (uint32_t)(nr * K * 2));
    }
    __syncwarp();
    for (int j = lane; j < nr; j += 32) {
      const int64_t src = (int64_t)b * Ts + r + C * j;
      bulk_g2s(renc + (size_t)j * E, a.enc + src * a.ld_enc, (uint32_t)E * 2, &bars[0]);
      bulk_g2s(rctx + (size_t)j * K, a.enc_ctx + src * a.pk, (uint32_t)K * 2, &bars[1]);
    }
  }
  for (int s = tid; s < Ts; s += kStThreads) {
    av[s] = a.a_all[tb * Ts + s];
    acc[s] = a.acc_all[tb * Ts + s];
    dacc[s] = (a.dacc_in && s < len) ? a.dacc_in[(int64_t)b * Ts + s] : 0.f;
  }
  {  // d att_t for this thread's 8 columns; d_a over this CTA's positions (all 8 warps per position)
    const int e0 = tid * 8;
    const bool on = e0 < E;
    float dv[8];
    if (on) {
      const float* pd = a.dro + row * a.prf + a.oa + e0;
      const float4 u0 = ldf4(pd), u1 = ldf4(pd + 4);
      dv[0] = u0.x, dv[1] = u0.y, dv[2] = u0.z, dv[3] = u0.w, dv[4] = u1.x, dv[5] = u1.y, dv[6] = u1.z, dv[7] = u1.w;
      for (int z = 0; z < a.n1; ++z) {
        const float* pz = a.P1 + z * a.p1_stride + (int64_t)b * a.p1_ld + e0;
        const float4 w0 = ldf4(pz), w1 = ldf4(pz + 4);
        dv[0] += w0.x, dv[1] += w0.y, dv[2] += w0.z, dv[3] += w0.w;
        dv[4] += w1.x, dv[5] += w1.y, dv[6] += w1.z, dv[7] += w1.w;
      }
      if (r == 0) {
        const float d0[4] = {dv[0], dv[1], dv[2], dv[3]}, d1[4] = {dv[4], dv[5], dv[6], dv[7]};
        stf4(a.datt_all + tb * E + e0, d0);
        stf4(a.datt_all + tb * E + e0 + 4, d1);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) dv[i] = 0.f;
    }
    tc::mbar_wait(&bars[0], 0);
    for (int j = 0; j < nr; ++j) {
      float sum = 0.f;
      if (on) {
        float f[8];
        ld8(renc + (size_t)j * E + e0, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) sum += dv[i] * f[i];
      }
      sum = warp_sum(sum);
      if (lane == 0) red[j * 8 + warp] = sum;
    }
  }
  __syncthreads();
  cluster_wait();
  for (int j = tid; j < nr; j += kStThreads) {
    const int s = r + C * j;
    float sum = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) sum += red[j * 8 + w];
    sum += dacc[s];
#pragma unroll
    for (int p = 0; p < C; ++p) cl.map_shared_rank(da, p)[s] = sum;
  }
  cl.sync();
  if (tid < 32) {  // softmax adjoint, in every CTA
    float dot = 0.f;
    for (int s = lane; s < len; s += 32) dot += av[s] * da[s];
    dot = warp_sum(dot);
    for (int s = lane; s < Ts; s += 32) {
      const float d = s < len ? av[s] * (da[s] - dot) : 0.f;
      de[s] = d;
      if (r == 0) a.de_all[tb * Ts + s] = d;
    }
  }
  __syncthreads();
  {  // tanh adjoint over this CTA's positions: two groups of 128 threads, 8 key columns each
    const int g = tid / 128, q = tid % 128, wig = q / 32, k0 = q * 8;
    const bool act = k0 < K;
    float wv[8], cv[8], vk[8], ds[8];
    if (act) {
      const float* st = a.str_all + tb * K + k0;
      const float4 s0v = ldf4(st), s1v = ldf4(st + 4);
      const float sv[8] = {s0v.x, s0v.y, s0v.z, s0v.w, s1v.x, s1v.y, s1v.z, s1v.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        wv[i] = a.W_fb[k0 + i];
        cv[i] = sv[i] + a.b_fb[k0 + i];
        vk[i] = a.v[k0 + i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) wv[i] = cv[i] = vk[i] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) ds[i] = 0.f;
    tc::mbar_wait(&bars[1], 0);
    for (int j = g; j < nr; j += 2) {
      const int s = r + C * j;
      const float as = acc[s], des = de[s];
      float pa = 0.f;
      if (act) {
        float f[8];
        ld8(rctx + (size_t)j * K + k0, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float uu = tanh_approx(f[i] + as * wv[i] + cv[i]);
          const float dein = des * vk[i] * (1.f - uu * uu);
          ds[i] += dein;
          pa += wv[i] * dein;
        }
      }
      pa = warp_sum(pa);
      if (lane == 0) red[j * 8 + wig] = pa;  // (red reused: the d_a partials are consumed)
    }
    if (act) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dsum[g * K + k0 + i] = ds[i];
    }
  }
  __syncthreads();
  for (int k = tid; k < K; k += kStThreads) pdst[k] = dsum[k] + dsum[K + k];
  for (int s = r + C * tid; s < Ts; s += C * kStThreads) {
    const int j = (s - r) / C;
    a.dacc_out[(int64_t)b * Ts + s] =
        s < len ? dacc[s] + (((red[j * 8] + red[j * 8 + 1]) + red[j * 8 + 2]) + red[j * 8 + 3]) : 0.f;
  }
  cl.sync();
  if (r == 0) {
    for (int k = tid; k < K; k += kStThreads) {
      float d = pdst[k];
#pragma unroll
      for (int p = 1; p < C; ++p) d += cl.map_shared_rank(pdst, p)[k];
      a.ds32[row * K + k] = d;
      a.ds[row * a.pds + k] = __float2bfloat16_rn(d);
    }
  }
  cl.sync();  // the peers' shared memory stays alive until CTA 0 has read it
}

// ---- after the loop: the accumulations over t ----------------------------------------------
struct CtxGrad {
  int B, Ts, T, K;
  const int32_t* lens;
  const bf16* enc_ctx;
  int64_t pk;
  const float *W_fb, *b_fb, *v;
  const float *str_all, *acc_all, *de_all;
  bf16* dctx;   // [B*Ts, pk]
  float* part;  // [blocks][4][K]: d W_fb, d b_fb, d v, d b_ctx partial sums of this CTA
};

// d enc_ctx[b, s, k] = sum_t de_t[b, s] v_k (1 - u_t^2), u recomputed; the CTA's
// (b, 8 positions) tile stays in registers across all T steps.
__global__ void __launch_bounds__(128) dec_ctx_grad_kernel(CtxGrad a) {
  extern __shared__ float sm[];  // [T][kCtxPos] de, then [T][kCtxPos] accum_{t-1}
  const int K = a.K, Ts = a.Ts, T = a.T, b = blockIdx.y, s0 = blockIdx.x * kCtxPos, tid = threadIdx.x;
  const int len = min(max(a.lens[b], 0), Ts);
  const int n = max(0, min(kCtxPos, len - s0));
  float* sde = sm;
  float* sacc = sm + T * kCtxPos;
  for (int i = tid; i < T * kCtxPos; i += 128) {
    const int t = i / kCtxPos, p = i % kCtxPos;
    const size_t o = ((size_t)t * a.B + b) * Ts + s0 + p;
    sde[i] = p < n ? a.de_all[o] : 0.f;
    sacc[i] = p < n ? a.acc_all[o] : 0.f;
  }
  __syncthreads();
  const int k0 = tid * 8;
  const bool act = k0 < K;
  float wv[8], bv[8], vk[8], dw[8], db[8], dv[8], dc[kCtxPos][8];
  uint4 x[kCtxPos];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    wv[i] = act ? a.W_fb[k0 + i] : 0.f;
    bv[i] = act ? a.b_fb[k0 + i] : 0.f;
    vk[i] = act ? a.v[k0 + i] : 0.f;
    dw[i] = db[i] = dv[i] = 0.f;
  }
#pragma unroll
  for (int p = 0; p < kCtxPos; ++p) {
    x[p] = (act && p < n) ? *reinterpret_cast<const uint4*>(a.enc_ctx + ((int64_t)b * Ts + s0 + p) * a.pk + k0)
                          : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) dc[p][i] = 0.f;
  }
  if (act && n > 0) {
    for (int t = 0; t < T; ++t) {
      const float* st = a.str_all + ((size_t)t * a.B + b) * K + k0;
      const float4 s0v = ldf4(st), s1v = ldf4(st + 4);
      const float sv[8] = {s0v.x + bv[0], s0v.y + bv[1], s0v.z + bv[2], s0v.w + bv[3],
                           s1v.x + bv[4], s1v.y + bv[5], s1v.z + bv[6], s1v.w + bv[7]};
#pragma unroll
      for (int p = 0; p < kCtxPos; ++p) {
        const float des = sde[t * kCtxPos + p];
        if (des == 0.f) continue;  // masked position (or an exactly-zero adjoint): contributes nothing
        const float as = sacc[t * kCtxPos + p];
        float f[8];
        unpack8(x[p], f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float u = tanh_approx(f[i] + as * wv[i] + sv[i]);
          const float dein = des * vk[i] * (1.f - u * u);
          dc[p][i] += dein;
          dw[i] += as * dein;
          db[i] += dein;
          dv[i] += des * u;
        }
      }
    }
  }
  if (act) {
#pragma unroll
    for (int p = 0; p < kCtxPos; ++p) {
      if (s0 + p >= Ts) break;
      bf16* d = a.dctx + ((int64_t)b * Ts + s0 + p) * a.pk + k0;
      const float lo[4] = {dc[p][0], dc[p][1], dc[p][2], dc[p][3]}, hi[4] = {dc[p][4], dc[p][5], dc[p][6], dc[p][7]};
      st4(d, lo);
      st4(d + 4, hi);
    }
    float* pp = a.part + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 4 * K + k0;
    float cs[8];  // d b_ctx = column sums of d enc_ctx in fp32 (its terms cancel: sum_s de = 0)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float q = 0.f;
#pragma unroll
      for (int p = 0; p < kCtxPos; ++p) q += dc[p][i];
      cs[i] = q;
    }
    const float c0[4] = {cs[0], cs[1], cs[2], cs[3]}, c1[4] = {cs[4], cs[5], cs[6], cs[7]};
    stf4(pp + 3 * K, c0), stf4(pp + 3 * K + 4, c1);
    const float w0[4] = {dw[0], dw[1], dw[2], dw[3]}, w1[4] = {dw[4], dw[5], dw[6], dw[7]};
    const float b0[4] = {db[0], db[1], db[2], db[3]}, b1[4] = {db[4], db[5], db[6], db[7]};
    const float v0[4] = {dv[0], dv[1], dv[2], dv[3]}, v1[4] = {dv[4], dv[5], dv[6], dv[7]};
    stf4(pp, w0), stf4(pp + 4, w1);
    stf4(pp + K, b0), stf4(pp + K + 4, b1);
    stf4(pp + 2 * K, v0), stf4(pp + 2 * K + 4, v1);
  }
}

// d enc[b, s, e] += sum_t a_t[b, s] d att_t[b, e]  (the generic_attention adjoint
// w.r.t. its base, tape.cpp:1047-1058, summed over the steps in t order).  A CTA
// covers (b, 16 positions, 512 columns): every thread keeps a 16 x 4 register tile,
// per step one float4 of d att and four float4 broadcasts of a from shared memory.
constexpr int kEncCols = 512, kEncPos = 16;
__global__ void __launch_bounds__(128) dec_enc_grad_kernel(int B, int Ts, int T, int E, const float* a_all,
                                                          const float* datt_all, float* d_enc, int64_t ld) {
  extern __shared__ float sa[];  // [T][kEncPos]
  const int b = blockIdx.z, s0 = blockIdx.y * kEncPos, e = blockIdx.x * kEncCols + threadIdx.x * 4;
  for (int i = threadIdx.x; i < T * kEncPos; i += 128) {
    const int t = i / kEncPos, s = s0 + i % kEncPos;
    sa[i] = s < Ts ? a_all[((size_t)t * B + b) * Ts + s] : 0.f;
  }
  __syncthreads();
  if (e >= E) return;
  float o[kEncPos][4];
#pragma unroll
  for (int s = 0; s < kEncPos; ++s) o[s][0] = o[s][1] = o[s][2] = o[s][3] = 0.f;
  for (int t = 0; t < T; ++t) {
    const float4 d = ldf4(datt_all + ((size_t)t * B + b) * E + e);
    const float4* at = reinterpret_cast<const float4*>(sa + t * kEncPos);
#pragma unroll
    for (int q = 0; q < kEncPos / 4; ++q) {
      const float4 a4 = at[q];
      const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        o[4 * q + u][0] += av[u] * d.x, o[4 * q + u][1] += av[u] * d.y;
        o[4 * q + u][2] += av[u] * d.z, o[4 * q + u][3] += av[u] * d.w;
      }
    }
  }
#pragma unroll
  for (int s = 0; s < kEncPos; ++s) {
    if (s0 + s >= Ts) break;
    float* p = d_enc + ((int64_t)b * Ts + s0 + s) * ld + e;
    float4 v = ldf4(p);
    v.x += o[s][0], v.y += o[s][1], v.z += o[s][2], v.w += o[s][3];
    *reinterpret_cast<float4*>(p) = v;
  }
}

// fixed-order column sums: out[c] = sum_r x[r * ld + c] (stage 1: row chunks, stage 2: chunks in order)
constexpr int kColChunks = 64;
__global__ void colsum1_kernel(const float* x, int64_t rows, int cols, int64_t ld, int64_t per, float* part) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= cols) return;
  const int64_t r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += x[r * ld + c];
  part[(int64_t)blockIdx.y * cols + c] = s;
}
__global__ void colsum2_kernel(const float* part, int chunks, int cols, float* out) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int i = 0; i < chunks; ++i) s += part[(int64_t)i * cols + c];
  out[c] = s;
}

// readout [b, t] = relu(pre [t*B + b]): the time-major GEMM rows to the caller's [B, T] layout
__global__ void relu_kernel(const float* pre, float* y, int B, int T, int cols) {
  const int q = cols / 4;
  const int64_t n = (int64_t)B * T * q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / q;  // output row b*T + t
    const int c = (int)(i - r * q) * 4, b = (int)(r / T), t = (int)(r - (int64_t)b * T);
    float4 v = ldf4(pre + ((int64_t)t * B + b) * cols + c);
    v.x = fmaxf(v.x, 0.f), v.y = fmaxf(v.y, 0.f), v.z = fmaxf(v.z, 0.f), v.w = fmaxf(v.w, 0.f);
    *reinterpret_cast<float4*>(y + r * cols + c) = v;
  }
}
// d (readout pre-activation) = d readout * [readout > 0] ([B, T] in), as the time-major bf16 GEMM operand
__global__ void relu_grad_kernel(const float* y, const float* dy, int B, int T, int cols, bf16* out, int64_t ld) {
  const int q = cols / 4;
  const int64_t n = (int64_t)B * T * q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / q;  // time-major row t*B + b
    const int c = (int)(i - r * q) * 4, t = (int)(r / B), b = (int)(r - (int64_t)t * B);
    const int64_t src = ((int64_t)b * T + t) * cols + c;
    const float4 v = ldf4(y + src), d = ldf4(dy + src);
    const float o[4] = {v.x > 0.f ? d.x : 0.f, v.y > 0.f ? d.y : 0.f, v.z > 0.f ? d.z : 0.f, v.w > 0.f ? d.w : 0.f};
    st4(out + r * ld + c, o);
  }
}
// the readout input's ones column (the [trg | 1] operand of d W_trg / d b) and the zero
// padding after it (read by the readout GEMM's K loop)
__global__ void ro_ones_kernel(bf16* ro, int64_t rows, int64_t pitch, int col, int n) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  bf16* p = ro + r * pitch + col;
  p[0] = __float2bfloat16_rn(1.f);
  for (int i = 1; i < n; ++i) p[i] = __float2bfloat16_rn(0.f);
}
// prev_ids [B, T] -> time-major [T, B]
__global__ void ids_to_time_major_kernel(const int32_t* ids, int B, int T, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * T) return;
  const int t = i / B, b = i - t * B;
  out[i] = ids[(int64_t)b * T + t];
}

// ---- host side -----------------------------------------------------------------------------
int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// split-K count for a batch-row GEMM (M <= 256 rows): fill the SM pairs, >= 4 K blocks per unit
// (the value gemm_bf16_tc2 re-derives: no empty units)
int ksplit_for(int M, int N, int K) {
  const int tiles = (int)(ceil_div(M, 256) * ceil_div(N, 256));
  const int nk = (int)ceil_div(K, 64);
  const int want = std::max(1, std::min(sm_count() / 2 / tiles, nk / 4));
  return (int)ceil_div(nk, ceil_div(nk, want));
}

struct Lay {
  int PZ, PXA, OA, PRO, PK, PR, PRF, PDR;  // PDR: pitch of the [DZ | d readout] rows
  int ks_f, ks_s, ks_1, ks_2;
  int ctx_blocks;
  bf16 *wd2, *wtrg, *wstr, *wctx, *wro, *wtrgcat;
  bf16 *enc_ctx, *xa, *ro, *dz, *ds, *drob, *dctx;
  int32_t* ids_tm;
  float *pre, *dtrg;
  float *xw, *pf, *pstr, *p1, *p2, *c_all, *gates, *str_all, *a_all, *acc_all, *de_all, *datt_all, *ds32, *dro,
      *dc, *dacc, *part, *colws, *tmp;
  void* emb_ws;
  size_t bytes;
};

Lay layout(const DecDims& d, void* base) {
  Lay L{};
  const int64_t BT = (int64_t)d.B * d.T, BTs = (int64_t)d.B * d.Ts;
  L.PZ = (int)round_up(4 * d.H, 64);
  L.PXA = (int)round_up(d.E + d.H, 64);
  L.OA = (int)round_up(d.H + d.Emb + 1, 8);
  L.PRO = (int)round_up(L.OA + d.E, 64);
  L.PK = (int)round_up(d.K, 64);
  L.PR = (int)round_up(d.Rd, 64);
  L.PRF = L.PRO;
  L.PDR = L.PZ + L.PR;
  L.ks_f = ksplit_for(d.B, 4 * d.H, d.E + d.H);
  L.ks_s = ksplit_for(d.B, d.K, d.H);
  L.ks_1 = ksplit_for(d.B, d.E + d.H, 4 * d.H);
  L.ks_2 = ksplit_for(d.B, d.H, d.K);
  L.ctx_blocks = (int)(d.B * ceil_div(d.Ts, kCtxPos));
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = round_up(off, 256);
    void* r = p ? p + off : nullptr;
    off += bytes;
    return r;
  };
  constexpr int64_t kSlack = 256;  // MN-major TMA boxes read whole 64-column blocks past the last row
  auto tb = [&](int64_t n) { return static_cast<bf16*>(take((size_t)(n + kSlack) * 2)); };
  auto tf = [&](int64_t n) { return static_cast<float*>(take((size_t)n * 4)); };
  L.wd2 = tb((int64_t)(d.E + d.H) * L.PZ);
  L.wtrg = tb((int64_t)d.Emb * L.PZ);
  L.wstr = tb((int64_t)d.H * L.PK);
  L.wctx = tb((int64_t)d.E * L.PK);
  L.wro = tb((int64_t)(L.OA + d.E) * L.PR);
  L.wtrgcat = tb((int64_t)d.Emb * L.PDR);
  L.enc_ctx = tb(BTs * L.PK);
  L.xa = tb(BT * L.PXA);
  L.ro = tb(BT * L.PRO);
  L.dz = tb(BT * L.PDR);  // [DZ (4H, pad to PZ) | d readout pre-activation (Rd, pad to PR)] per row
  L.ds = tb(BT * L.PK);
  L.drob = L.dz + L.PZ;
  L.dctx = tb(BTs * L.PK);
  L.ids_tm = static_cast<int32_t*>(take((size_t)BT * 4));
  L.pre = tf(BT * d.Rd);
  L.dtrg = tf(BT * d.Emb);
  L.xw = tf(BT * 4 * d.H);
  L.pf = tf((int64_t)L.ks_f * d.B * 4 * d.H);
  L.pstr = tf((int64_t)L.ks_s * d.B * L.PK);
  L.p1 = tf((int64_t)L.ks_1 * d.B * (d.E + d.H));
  L.p2 = tf((int64_t)L.ks_2 * d.B * L.PK);
  L.c_all = tf(BT * d.H);
  L.gates = tf(BT * 5 * d.H);
  L.str_all = tf((int64_t)d.T * d.B * d.K);
  L.a_all = tf((int64_t)d.T * d.B * d.Ts);
  L.acc_all = tf((int64_t)(d.T + 1) * d.B * d.Ts);
  L.de_all = tf((int64_t)d.T * d.B * d.Ts);
  L.datt_all = tf((int64_t)d.T * d.B * d.E);
  L.ds32 = tf(BT * d.K);
  L.dro = tf(BT * L.PRF);
  L.dc = tf((int64_t)2 * d.B * d.H);
  L.dacc = tf((int64_t)2 * d.B * d.Ts);
  L.part = tf((int64_t)L.ctx_blocks * 4 * d.K);
  L.colws = tf((int64_t)kColChunks * std::max(d.K, d.Ts));
  L.tmp = tf(std::max<int64_t>(d.Ts, 64));
  L.emb_ws = take(embedding_workspace_bytes(BT, d.Vt));
  L.bytes = off + 256;
  return L;
}

void colsum(const float* x, int64_t rows, int cols, int64_t ld, float* out, float* ws, cudaStream_t st) {
  const int64_t per = std::max<int64_t>(1, ceil_div(rows, kColChunks));
  const int chunks = (int)ceil_div(rows, per);
  colsum1_kernel<<<dim3((unsigned)ceil_div(cols, 256), (unsigned)chunks), 256, 0, st>>>(x, rows, cols, ld, per, ws);
  colsum2_kernel<<<(unsigned)ceil_div(cols, 256), 256, 0, st>>>(ws, chunks, cols, out);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch(2);
}

TcGemm mk(int M, int N, int K, const bf16* A, int64_t lda, bool a_mn, const bf16* B, int64_t ldb, bool b_mn, float* C,
          int64_t ldc) {
  TcGemm g{M, N, K, A, lda, a_mn, B, ldb, b_mn, C, ldc, 1.f, 0.f, nullptr};
  return g;
}
void gemm_split(TcGemm g, int ks, cudaStream_t st) {
  g.ksplit = ks;
  g.split_stride = (int64_t)g.M * g.ldc;
  gemm_bf16_tc(g, st);
}

size_t att_fwd_smem(const DecDims& d) { return (size_t)(6 * d.Ts + 4 + 1024) * 4; }
size_t att_bwd_smem(const DecDims& d) { return (size_t)(5 * d.K + 13 * d.Ts) * 4; }

template <int C, typename Args>
void launch_cluster(void (*kern)(Args), int B, size_t smem, const Args& args, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(C * B));
  cfg.blockDim = dim3(kStThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args));
}

// cluster size of the TMA-staged attention kernels: the smallest C whose per-CTA
// staging fits two CTAs per SM; 0 = the register-streaming kernels (or SL_DEC_ATT_REGS)
int att_cluster(const DecDims& d) {
  if (getenv("SL_DEC_ATT_REGS")) return 0;
  if (d.E > 2 * 1024) return 0;
  for (int C : {4, 8}) {
    if (st_cols(d.E, C) > 512) continue;
    const size_t need = std::max(FwdSt(d.Ts, d.K, d.E, C).total, BwdSt(d.Ts, d.K, d.E, C).total);
    if (need <= 110 * 1024) return C;
  }
  return 0;
}

void configure() {  // opt in to > 48 KB dynamic shared memory once
  static bool done = false;
  if (done) return;
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_ctx_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_enc_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_attn_fwd_tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_attn_fwd_tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_attn_bwd_tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_attn_bwd_tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
  const char* m = getenv("SL_DEC_TANH");
  const int mode = m ? atoi(m) : 0;
  SL_CUDA_TRY(cudaMemcpyToSymbol(c_tanh_mode, &mode, sizeof(int)));
  done = true;
}

}  // namespace

void decoder_check(const DecDims& d) {
  SL_REQUIRE(d.B > 0 && d.B <= 256 && d.Ts > 0 && d.T > 0 && d.Emb > 0 && d.E > 0 && d.H > 0 && d.K > 0 &&
                 d.Rd > 0 && d.Vt > 0,
             SL_ERR_SHAPE, "attn_decoder: dimensions must be positive, batch <= 256 per call");
  SL_REQUIRE(d.H % 8 == 0 && d.E % 8 == 0 && d.K % 8 == 0 && d.Rd % 8 == 0, SL_ERR_UNSUPPORTED,
             "attn_decoder: hidden, enc, key and readout dims must be multiples of 8");
  SL_REQUIRE(d.K <= 1024 && d.E <= 2048 && d.Ts <= 1024 && d.T <= 1024 && (int64_t)d.T * d.Ts <= 48 * 1024,
             SL_ERR_UNSUPPORTED,
             "attn_decoder: key_dim <= 1024, enc_dim <= 2048, src/trg time <= 1024, src*trg time <= 48K supported");
}

size_t decoder_workspace_bytes(const DecDims& d) { return layout(d, nullptr).bytes; }

void decoder_fwd(const DecDims& d, const DecParams& p, const bf16* enc, int64_t ld_enc, const int32_t* src_lens,
                 const int32_t* prev_ids, float* readout, int32_t* bad_row, void* ws, cudaStream_t st) {
  decoder_check(d);
  configure();
  SL_REQUIRE(ld_enc >= round_up(d.E + 1, 64) && ((uintptr_t)enc & 15) == 0, SL_ERR_INVALID_ARGUMENT,
             "attn_decoder: enc must be the padded bf16 layout (ld >= sl_lstm_bf16_pitch(enc_dim))");
  const Lay L = layout(d, ws);
  const int B = d.B, T = d.T, H = d.H, E = d.E, K = d.K;
  const int64_t BT = (int64_t)B * T, BTs = (int64_t)B * d.Ts;
  const double flops = 2.0 * BTs * E * K + 2.0 * BT * d.Emb * 4 * H + 2.0 * BT * (E + H) * 4 * H +
                       2.0 * BT * H * K + 2.0 * BT * (L.OA + E) * d.Rd;
  (void)flops;
  std::unique_ptr<Phase> ph(new Phase(st, "k10_dec_fwd_hoisted", 2.0 * BTs * E * K + 2.0 * BT * d.Emb * 4 * H));
  SL_CUDA_TRY(cudaMemsetAsync(L.xa, 0, (size_t)B * L.PXA * 2, st));  // step 0's [att ‖ s]_{-1} = 0
  SL_CUDA_TRY(cudaMemsetAsync(L.acc_all, 0, (size_t)BTs * 4, st));
  // packed bf16 weights (rows of the reference layouts; see the GEMMs for the majorness)
  f32_to_bf16(E, 4 * H, p.s_W + (int64_t)d.Emb * 4 * H, 4 * H, L.wd2, L.PZ, st);
  f32_to_bf16(H, 4 * H, p.s_R, 4 * H, L.wd2 + (int64_t)E * L.PZ, L.PZ, st);
  f32_to_bf16(d.Emb, 4 * H, p.s_W, 4 * H, L.wtrg, L.PZ, st);
  f32_to_bf16(H, K, p.str_W, K, L.wstr, L.PK, st);
  f32_to_bf16(E, K, p.ctx_W, K, L.wctx, L.PK, st);
  f32_to_bf16(H + d.Emb, d.Rd, p.ro_W, d.Rd, L.wro, L.PR, st);
  SL_CUDA_TRY(cudaMemsetAsync(L.wro + (int64_t)(H + d.Emb) * L.PR, 0, (size_t)(L.OA - H - d.Emb) * L.PR * 2, st));
  f32_to_bf16(E, d.Rd, p.ro_W + (int64_t)(H + d.Emb) * d.Rd, d.Rd, L.wro + (int64_t)L.OA * L.PR, L.PR, st);
  // [W_trg | W_ro(trg rows)] along K: d trg_{t-1} = [DZ | d ro] [W_trg | W_ro,trg]^T in one GEMM
  SL_CUDA_TRY(cudaMemsetAsync(L.wtrgcat, 0, (size_t)d.Emb * L.PDR * 2, st));
  f32_to_bf16(d.Emb, 4 * H, p.s_W, 4 * H, L.wtrgcat, L.PDR, st);
  f32_to_bf16(d.Emb, d.Rd, p.ro_W + (int64_t)H * d.Rd, d.Rd, L.wtrgcat + L.PZ, L.PDR, st);
  // trg_{t-1} into the readout-input rows (columns H..H+Emb) + the ones column
  ids_to_time_major_kernel<<<(unsigned)ceil_div(BT, 256), 256, 0, st>>>(prev_ids, B, T, L.ids_tm);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
  embedding_fwd_bf16(BT, L.ids_tm, d.Vt, d.Emb, p.trg_W, L.ro + H, L.PRO, SL_EMB_NEGATIVE_ZERO, bad_row, st);
  ro_ones_kernel<<<(unsigned)ceil_div(BT, 256), 256, 0, st>>>(L.ro, BT, L.PRO, H + d.Emb, L.OA - H - d.Emb);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
  {  // enc_ctx = enc W_ctx + b_ctx (bf16 out); x W_trg + b for all t
    TcGemm g = mk((int)BTs, K, E, enc, ld_enc, false, L.wctx, L.PK, true, nullptr, L.PK);
    g.bias = p.ctx_b;
    g.Cb = L.enc_ctx;
    gemm_bf16_tc(g, st);
    TcGemm x = mk((int)BT, 4 * H, d.Emb, L.ro + H, L.PRO, false, L.wtrg, L.PZ, true, L.xw, 4 * H);
    x.bias = p.s_b;
    gemm_bf16_tc(x, st);
  }
  ph.reset();
  const int cell_threads = B * (H / 4);
  const double att_bytes = 2.0 * B * d.Ts * (K + E);
  const int ac = att_cluster(d);
  for (int t = 0; t < T; ++t) {
    if (t > 0) {
      Phase p1(st, "k10_cell_gemm", 2.0 * B * (E + H) * 4 * H);
      gemm_split(mk(B, 4 * H, E + H, L.xa + (int64_t)t * B * L.PXA, L.PXA, false, L.wd2, L.PZ, true, L.pf, 4 * H),
                 L.ks_f, st);
    }
    ph.reset(new Phase(st, "k10_cell_fwd", 0.0, 4.0 * B * H * 16));
    CellFwd cf{B, T, H, E, t, t > 0 ? L.ks_f : 0, L.pf, 4 * H, (int64_t)B * 4 * H, L.xw, L.c_all, L.gates,
               L.xa, L.PXA, L.ro, L.PRO};
    dec_cell_fwd_kernel<<<(unsigned)ceil_div(cell_threads, 256), 256, 0, st>>>(cf);
    ph.reset(new Phase(st, "k10_str_gemm", 2.0 * B * H * K));
    gemm_split(mk(B, K, H, L.ro + (int64_t)t * B * L.PRO, L.PRO, false, L.wstr, L.PK, true, L.pstr, L.PK),
               L.ks_s, st);
    AttFwd af{B, d.Ts, T, K, E, t, L.ks_s, src_lens, L.pstr, L.PK, (int64_t)B * L.PK, p.str_b, p.fb_W, p.fb_b,
              p.e_W, p.e_b, L.enc_ctx, L.PK, enc, ld_enc, L.str_all, L.a_all, L.acc_all, L.ro, L.PRO, L.OA,
              L.xa, L.PXA};
    ph.reset(new Phase(st, "k10_attn_fwd", 0.0, att_bytes));
    if (ac == 4) launch_cluster<4>(dec_attn_fwd_tma_kernel<4>, B, FwdSt(d.Ts, K, E, 4).total, af, st);
    else if (ac == 8) launch_cluster<8>(dec_attn_fwd_tma_kernel<8>, B, FwdSt(d.Ts, K, E, 8).total, af, st);
    else dec_attn_fwd_kernel<<<2 * B, kAttThreads, att_fwd_smem(d), st>>>(af);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch(2);
    ph.reset();
  }
  ph.reset(new Phase(st, "k10_dec_fwd_hoisted", 2.0 * BT * (L.OA + E) * d.Rd));
  TcGemm r = mk((int)BT, d.Rd, L.OA + E, L.ro, L.PRO, false, L.wro, L.PR, true, L.pre, d.Rd);
  r.bias = p.ro_b;
  gemm_bf16_tc(r, st);
  relu_kernel<<<sm_count() * 4, 256, 0, st>>>(L.pre, readout, B, T, d.Rd);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void decoder_bwd(const DecDims& d, const DecParams& p, const DecGrads& g, const bf16* enc, int64_t ld_enc,
                 const int32_t* src_lens, const int32_t* prev_ids, const float* readout, const float* d_readout,
                 float* d_enc, void* ws, cudaStream_t st) {
  decoder_check(d);
  configure();
  const Lay L = layout(d, ws);
  const int B = d.B, T = d.T, H = d.H, E = d.E, K = d.K, Emb = d.Emb, Rd = d.Rd;
  const int64_t BT = (int64_t)B * T, BTs = (int64_t)B * d.Ts;
  const double flops = 2.0 * (2.0 * BTs * E * K + 2.0 * BT * Emb * 4 * H + 2.0 * BT * (E + H) * 4 * H +
                              2.0 * BT * H * K + 2.0 * BT * (L.OA + E) * Rd);
  (void)flops;
  std::unique_ptr<Phase> ph(new Phase(st, "k10_dec_bwd_hoisted", 4.0 * BT * (L.OA + E) * Rd));
  // readout: relu adjoint, d [s ‖ trg ‖ att], d W_ro (three row blocks) and d b_ro (ones column)
  // zero pads of the [DZ | d ro] rows (inside the K range of the d trg GEMM)
  SL_CUDA_TRY(cudaMemset2DAsync(L.dz + 4 * H, (size_t)L.PDR * 2, 0, (size_t)(L.PZ - 4 * H) * 2, BT, st));
  SL_CUDA_TRY(cudaMemset2DAsync(L.drob + Rd, (size_t)L.PDR * 2, 0, (size_t)(L.PR - Rd) * 2, BT, st));
  relu_grad_kernel<<<sm_count() * 4, 256, 0, st>>>(readout, d_readout, B, T, Rd, L.drob, L.PDR);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
  gemm_bf16_tc(mk((int)BT, L.OA + E, Rd, L.drob, L.PDR, false, L.wro, L.PR, false, L.dro, L.PRF), st);
  gemm_bf16_tc(mk(H, Rd, (int)BT, L.ro, L.PRO, true, L.drob, L.PDR, true, g.ro_W, Rd), st);
  {
    TcGemm w = mk(Emb + 1, Rd, (int)BT, L.ro + H, L.PRO, true, L.drob, L.PDR, true, g.ro_W + (int64_t)H * Rd, Rd);
    w.m_split = Emb;
    w.C2 = g.ro_b;
    w.ldc2 = Rd;
    gemm_bf16_tc(w, st);
  }
  gemm_bf16_tc(mk(E, Rd, (int)BT, L.ro + L.OA, L.PRO, true, L.drob, L.PDR, true, g.ro_W + (int64_t)(H + Emb) * Rd, Rd),
               st);
  ph.reset();
  const int cell_threads = B * (H / 4);
  const double att_bytes = 2.0 * B * d.Ts * (K + E);
  const int ac = att_cluster(d);
  for (int t = T - 1; t >= 0; --t) {
    const bool last = t == T - 1;
    if (!last) {
      Phase p1(st, "k10_g1_gemm", 2.0 * B * (E + H) * 4 * H);
      gemm_split(mk(B, E + H, 4 * H, L.dz + (int64_t)(t + 1) * B * L.PDR, L.PDR, false, L.wd2, L.PZ, false, L.p1,
                    E + H),
                 L.ks_1, st);
    }
    ph.reset(new Phase(st, "k10_attn_bwd", 0.0, att_bytes));
    AttBwd ab{B, d.Ts, T, K, E, t, last ? 0 : L.ks_1, src_lens, L.p1, E + H, (int64_t)B * (E + H), L.dro, L.PRF,
              L.OA, p.fb_W, p.fb_b, p.e_W, L.enc_ctx, L.PK, enc, ld_enc, L.str_all, L.a_all, L.acc_all,
              last ? nullptr : L.dacc + (int64_t)((t + 1) % 2) * B * d.Ts, L.dacc + (int64_t)(t % 2) * B * d.Ts,
              L.datt_all, L.de_all, L.ds, L.PK, L.ds32};
    if (ac == 4) launch_cluster<4>(dec_attn_bwd_tma_kernel<4>, B, BwdSt(d.Ts, K, E, 4).total, ab, st);
    else if (ac == 8) launch_cluster<8>(dec_attn_bwd_tma_kernel<8>, B, BwdSt(d.Ts, K, E, 8).total, ab, st);
    else dec_attn_bwd_kernel<<<2 * B, kAttThreads, att_bwd_smem(d), st>>>(ab);
    ph.reset(new Phase(st, "k10_g2_gemm", 2.0 * B * H * K));
    gemm_split(mk(B, H, K, L.ds + (int64_t)t * B * L.PK, L.PK, false, L.wstr, L.PK, false, L.p2, L.PK),
               L.ks_2, st);
    CellBwd cb{B, T, H, E, t, last ? 0 : L.ks_1, L.p1, E + H, (int64_t)B * (E + H), L.ks_2, L.p2, L.PK,
               (int64_t)B * L.PK, L.dro, L.PRF, L.gates, L.c_all,
               last ? nullptr : L.dc + (int64_t)((t + 1) % 2) * B * H, L.dc + (int64_t)(t % 2) * B * H, L.dz, L.PDR};
    ph.reset(new Phase(st, "k10_cell_bwd", 0.0, 4.0 * B * H * 20));
    dec_cell_bwd_kernel<<<(unsigned)ceil_div(cell_threads, 256), 256, 0, st>>>(cb);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch(2);
    ph.reset();
  }
  ph.reset(new Phase(st, "k10_dec_bwd_hoisted",
                     2.0 * BT * 4 * H * (E + H + Emb + 1) + 2.0 * BT * Emb * 4 * H + 2.0 * BT * H * K));
  // the decoder cell's weight gradients over all B*T rows: [W_att; R] from [att ‖ s]_{t-1},
  // [W_trg; b] from [trg_{t-1} | 1]; d trg_{t-1} -> the trg table
  gemm_bf16_tc(mk(E, 4 * H, (int)BT, L.xa, L.PXA, true, L.dz, L.PDR, true, g.s_W + (int64_t)Emb * 4 * H, 4 * H), st);
  gemm_bf16_tc(mk(H, 4 * H, (int)BT, L.xa + E, L.PXA, true, L.dz, L.PDR, true, g.s_R, 4 * H), st);
  {
    TcGemm w = mk(Emb + 1, 4 * H, (int)BT, L.ro + H, L.PRO, true, L.dz, L.PDR, true, g.s_W, 4 * H);
    w.m_split = Emb;
    w.C2 = g.s_b;
    w.ldc2 = 4 * H;
    gemm_bf16_tc(w, st);
    // d trg_{t-1} = [DZ | d ro] [W_trg | W_ro,trg]^T (the cell input and the readout input, one GEMM)
    gemm_bf16_tc(mk((int)BT, Emb, L.PZ + Rd, L.dz, L.PDR, false, L.wtrgcat, L.PDR, false, L.dtrg, Emb), st);
  }
  embedding_bwd(BT, L.ids_tm, d.Vt, Emb, L.dtrg, Emb, g.trg_W, false, L.emb_ws, st);
  // s_tr: d W_s over all rows, d b_s as a fixed-order column sum
  gemm_bf16_tc(mk(H, K, (int)BT, L.ro, L.PRO, true, L.ds, L.PK, true, g.str_W, K), st);
  colsum(L.ds32, BT, K, K, g.str_b, L.colws, st);
  // the attention's accumulations over t
  ph.reset(new Phase(st, "k10_attn_accum", 0.0, 2.0 * BTs * K + 4.0 * T * B * (K + E)));
  {
    CtxGrad cg{B, d.Ts, T, K, src_lens, L.enc_ctx, L.PK, p.fb_W, p.fb_b, p.e_W, L.str_all, L.acc_all, L.de_all,
               L.dctx, L.part};
    dec_ctx_grad_kernel<<<dim3((unsigned)ceil_div(d.Ts, kCtxPos), (unsigned)B), 128,
                          (size_t)2 * T * kCtxPos * 4, st>>>(cg);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
    colsum(L.part, L.ctx_blocks, K, 4 * K, g.fb_W, L.colws, st);
    colsum(L.part + K, L.ctx_blocks, K, 4 * K, g.fb_b, L.colws, st);
    colsum(L.part + 2 * K, L.ctx_blocks, K, 4 * K, g.e_W, L.colws, st);
    colsum(L.part + 3 * K, L.ctx_blocks, K, 4 * K, g.ctx_b, L.colws, st);
    colsum(L.de_all, (int64_t)T * B, d.Ts, d.Ts, L.tmp, L.colws, st);
    colsum(L.tmp, d.Ts, 1, 1, g.e_b, L.colws, st);
  }
  ph.reset(new Phase(st, "k10_dec_bwd_hoisted", 4.0 * BTs * E * K));
  {
    gemm_bf16_tc(mk((int)BTs, E, K, L.dctx, L.PK, false, L.wctx, L.PK, false, d_enc, E), st);
    gemm_bf16_tc(mk(E, K, (int)BTs, enc, ld_enc, true, L.dctx, L.PK, true, g.ctx_W, K), st);
  }
  ph.reset(new Phase(st, "k10_attn_accum", 0.0, 4.0 * T * B * E + 8.0 * BTs * E));
  dec_enc_grad_kernel<<<dim3((unsigned)ceil_div(E, kEncCols), (unsigned)ceil_div(d.Ts, kEncPos), (unsigned)B), 128,
                        (size_t)T * kEncPos * 4, st>>>(
      B, d.Ts, T, E, L.a_all, L.datt_all, d_enc, E);  // += sum_t a_t (x) d att_t
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();

}

}  // namespace sl
