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
//    GEMM, and two attention kernels (energies per (row, 8 positions); softmax +
//    context per (row, 512 columns)) reading enc_ctx / enc in bf16; the backward
//    mirrors it (G1 GEMM, d_a per (row, 512 columns), softmax + tanh adjoint per
//    (row, 8 positions), a fixed-order d s_tr reduction, G2 GEMM, gate adjoint).
//    Time-major per-step buffers (a step's rows are contiguous), loads issued
//    unconditionally before their first use, programmatic dependent launch
//    between the per-step kernels.
//  * Backward: the per-step attention kernels compute only what the recurrence
//    needs (d s_tr and d accum_{t-1}); the big accumulations over t — d enc_ctx,
//    d W_fb, d b_fb, d v, d enc = sum_t a_t (x) d att_t — run once after the loop
//    from small saved per-step vectors (a_t, d att_t, de_t), recomputing tanh in
//    registers, so the loop never read-modify-writes a [B, Ts, K] accumulator.
//    All reductions are fixed-order (deterministic).
#include <algorithm>
#include <cmath>
#include <memory>
#include <utility>

#include "convert.h"
#include "decoder.h"
#include "embedding.h"
#include "gemm.h"
#include "profile.h"

namespace sl {
namespace {

using bf16 = __nv_bfloat16;

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
// Programmatic dependent launch (PDL): the per-step kernels are launched with
// programmatic stream serialization, trigger their dependents at entry and, after
// a prologue that only touches data that is static during the loop (enc, enc_ctx,
// weights, the hoisted GEMM outputs), wait for the preceding grid.  The next
// kernel's launch, its CTAs' ramp-up and its big static loads overlap the tail of
// the previous one.  (Kernels launched without the attribute: both are no-ops.)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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
  int b0, nb;  // this launch's batch rows [b0, b0 + nb) (concurrent batch slices)
};

__global__ void dec_cell_fwd_kernel(CellFwd a) {
  pdl_trigger();
  pdl_wait();
  const int qn = a.H / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.nb * qn) return;
  const int b = a.b0 + idx / qn, j = (idx % qn) * 4;
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
  int b0, nb;
};

__global__ void dec_cell_bwd_kernel(CellBwd a) {
  pdl_trigger();
  pdl_wait();
  const int qn = a.H / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.nb * qn) return;
  const int b = a.b0 + idx / qn, j = (idx % qn) * 4;
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

// ---- attention step: small independent CTAs ------------------------------------------------
// Every step's attention is split into kernels whose CTAs need no cross-CTA
// synchronisation — (row, 8 positions) for the energies and the tanh adjoint,
// (row, 512 encoder columns) for the context and d_a — ~1000-2000 CTAs per launch, so
// the loads of many resident CTAs overlap each other's arithmetic (a CTA per row, with
// its phases separated by barriers, left the step latency-bound at ~30 % of HBM).
// Inside a CTA every load a thread needs is issued before the first use (no
// dependent chains of memory latencies), and the per-row softmax (and its adjoint)
// over the Ts energies is recomputed by every CTA that needs it.  All cross-CTA sums
// are written as partials and reduced in a fixed order (deterministic).
constexpr int kPos = 8;        // positions per CTA (energies, tanh adjoint)
constexpr int kCols = 512;     // encoder columns per CTA (context, d_a): 128 threads x 4
constexpr int kAtt = 128;      // threads per (row, 8 positions) CTA
constexpr int kGrp = 4;        // position groups of the (row, 512 columns) CTAs: 4 x 128 threads
constexpr int kPerGrp = 16;    // positions per thread and batch in those CTAs (context)
constexpr int kPerGrpDa = 8;   // (d_a: one warp reduction per position, fewer registers)
constexpr int kMaxSplit = 8;   // split-K partials summed in-kernel

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
  float* es;       // [B][Ts] energies of this step
  float* str_all;  // [T][B][K]: s_tr (with b_s)
  float* a_all;    // [T][B][Ts]
  float* acc_all;  // [T+1][B][Ts]: acc_all[t] = accum_{t-1}
  bf16* ro;        // att_t -> row (t, b), column oa
  int64_t pro;
  int oa;
  bf16* xa;  // att_t -> row (t+1, b), column 0
  int64_t pxa;
  int b0;  // grid.y covers rows [b0, b0 + gridDim.y)
};

// s_tr (+ b_s) for 8 key columns: the split-K partials, all loads issued together
__device__ __forceinline__ void str_cols(const float* P, int nsplit, int64_t p_stride, const float* bias, int k0,
                                         float (&st)[8]) {
  constexpr int kMaxStr = 4;  // the s_tr GEMM's split count (ksplit_for(..., 4))
  float4 u[kMaxStr][2];
#pragma unroll
  for (int z = 0; z < kMaxStr; ++z) {  // unconditional (clamped) loads: all in flight together
    const int zc = max(min(z, nsplit - 1), 0);
    u[z][0] = ldf4(P + zc * p_stride + k0);
    u[z][1] = ldf4(P + zc * p_stride + k0 + 4);
  }
  const float4 b0 = ldf4(bias + k0), b1 = ldf4(bias + k0 + 4);
  st[0] = b0.x, st[1] = b0.y, st[2] = b0.z, st[3] = b0.w, st[4] = b1.x, st[5] = b1.y, st[6] = b1.z, st[7] = b1.w;
#pragma unroll
  for (int z = 0; z < kMaxStr; ++z)
    if (z < nsplit) {
      st[0] += u[z][0].x, st[1] += u[z][0].y, st[2] += u[z][0].z, st[3] += u[z][0].w;
      st[4] += u[z][1].x, st[5] += u[z][1].y, st[6] += u[z][1].z, st[7] += u[z][1].w;
    }
}

// e[b, s] = <v, tanh(enc_ctx[b, s] + accum_{t-1}[b, s] W_fb + b_fb + s_tr[b])> + b_v
// for 8 positions; a thread owns 8 key columns (K <= 1024)
__global__ void __launch_bounds__(kAtt, 6) dec_att_energy_kernel(AttFwd a) {
  __shared__ float red[kPos][4];
  pdl_trigger();
  const int b = a.b0 + blockIdx.y, j0 = blockIdx.x * kPos, Ts = a.Ts, K = a.K, tid = threadIdx.x;
  const int lane = tid % 32, warp = tid / 32, k0 = tid * 8;
  const bool act = k0 < K;
  const size_t tb = (size_t)a.t * a.B + b;
  // Unconditional loads from clamped (always valid) addresses, masked when consumed: a
  // `cond ? load : 0` select makes the compiler retire each load before issuing the next.
  uint4 x[kPos];
  const int kc = act ? k0 : 0;
#pragma unroll
  for (int p = 0; p < kPos; ++p)
    x[p] = *reinterpret_cast<const uint4*>(a.enc_ctx + ((int64_t)b * Ts + min(j0 + p, Ts - 1)) * a.pk + kc);
  const int len = min(max(a.lens[b], 0), Ts);
  float4 f0, f1, w0, w1, v0, v1;
  if (act) f0 = ldf4(a.b_fb + k0), f1 = ldf4(a.b_fb + k0 + 4), w0 = ldf4(a.W_fb + k0), w1 = ldf4(a.W_fb + k0 + 4),
           v0 = ldf4(a.v + k0), v1 = ldf4(a.v + k0 + 4);
  pdl_wait();  // s_tr partials (s_tr GEMM) and accum_{t-1} (previous step) from here on
  float acp[kPos];
#pragma unroll
  for (int p = 0; p < kPos; ++p) acp[p] = a.acc_all[tb * Ts + min(j0 + p, Ts - 1)];
  float st[8], cv[8], wv[8], vk[8];
  if (act) {
    str_cols(a.P + (int64_t)b * a.p_ld, a.nsplit, a.p_stride, a.b_s, k0, st);
    const float bf[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
    const float wf[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const float vf[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = st[i] + bf[i], wv[i] = wf[i], vk[i] = vf[i];
    if (blockIdx.x == 0) {
      const float s0[4] = {st[0], st[1], st[2], st[3]}, s1[4] = {st[4], st[5], st[6], st[7]};
      stf4(a.str_all + tb * K + k0, s0);
      stf4(a.str_all + tb * K + k0 + 4, s1);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = wv[i] = vk[i] = 0.f;
  }
  const int n = min(kPos, len - j0);
#pragma unroll
  for (int p = 0; p < kPos; ++p) {
    float sum = 0.f;
    if (p < n) {
      float f[8];
      unpack8(x[p], f);
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += vk[i] * tanh_approx(f[i] + acp[p] * wv[i] + cv[i]);
    }
    sum = warp_sum(sum);
    if (lane == 0) red[p][warp] = sum;
  }
  __syncthreads();
  if (tid < n) a.es[(int64_t)b * Ts + j0 + tid] = ((red[tid][0] + red[tid][1]) + red[tid][2]) + red[tid][3] + *a.b_v;
}

// masked softmax of a row's energies into shared memory (tape.cpp:952-960); warp 0.
// The first 128 energies come in with one round of loads (registers), the rest (Ts > 128) in a loop.
__device__ __forceinline__ void row_softmax(const float* e, int len, int Ts, float* a_sm) {
  const int lane = threadIdx.x % 32;
  float r[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) r[i] = lane + 32 * i < Ts ? e[lane + 32 * i] : 0.f;  // (no wait on len)
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (lane + 32 * i >= len) r[i] = -INFINITY;
  float m = fmaxf(fmaxf(r[0], r[1]), fmaxf(r[2], r[3]));
  for (int s = lane + 128; s < len; s += 32) m = fmaxf(m, e[s]);
  m = warp_max(m);
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float ex = lane + 32 * i < len ? expf(r[i] - m) : 0.f;
    r[i] = ex;
    sum += ex;
  }
  for (int s = lane + 128; s < len; s += 32) {
    const float ex = expf(e[s] - m);
    a_sm[s] = ex;
    sum += ex;
  }
  sum = warp_sum(sum);
  const float inv = len > 0 ? 1.f / sum : 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (lane + 32 * i < Ts) a_sm[lane + 32 * i] = r[i] * inv;
  __syncwarp();
  for (int s = lane + 128; s < Ts; s += 32) a_sm[s] = s < len ? a_sm[s] * inv : 0.f;
}

// a = softmax(e) (recomputed per CTA), accum_t = accum_{t-1} + a, att = sum_s a_s enc_s
// (tape.cpp:1005-1014) for 512 encoder columns: 4 groups of 128 threads split the
// positions, each thread loads its (up to) 16 positions' 4 columns at once
__global__ void __launch_bounds__(kAtt * kGrp, 2) dec_att_context_kernel(AttFwd a) {
  extern __shared__ float asm_[];  // [Ts] a, then [kGrp - 1][kCols] partial contexts
  pdl_trigger();
  float* part = asm_ + (a.Ts + 3) / 4 * 4;
  const int b = a.b0 + blockIdx.y, Ts = a.Ts, tid = threadIdx.x, g = tid / kAtt, q = tid % kAtt;
  const int c = blockIdx.x * kCols + q * 4;
  const bool on = c < a.E;
  const size_t tb = (size_t)a.t * a.B + b;
  const int len = min(max(a.lens[b], 0), Ts);
  const bf16* x = a.enc + (int64_t)b * Ts * a.ld_enc + c;
  float o[4] = {0.f, 0.f, 0.f, 0.f};
  uint2 raw[kPerGrp];
  const bf16* xc = on ? x : x - c;  // unconditional loads from clamped rows / columns, masked when consumed
  auto load = [&](int s0) {
#pragma unroll
    for (int u = 0; u < kPerGrp; ++u)
      raw[u] = *reinterpret_cast<const uint2*>(xc + (int64_t)min(s0 + kGrp * u, Ts - 1) * a.ld_enc);
  };
  load(g);    // the first batch of encoder rows is in flight before the wait ...
  pdl_wait();  // ... for the energies of this step
  if (tid < 32) row_softmax(a.es + (int64_t)b * Ts, len, Ts, asm_);
  __syncthreads();  // a is ready
  for (int s0 = g; s0 < len; s0 += kGrp * kPerGrp) {
    if (s0 != g) load(s0);
#pragma unroll
    for (int u = 0; u < kPerGrp; ++u) {
      const int s = s0 + kGrp * u;
      const float as = s < len ? asm_[s] : 0.f;
      const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[u].x));
      const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[u].y));
      o[0] += as * lo.x, o[1] += as * lo.y, o[2] += as * hi.x, o[3] += as * hi.y;
    }
  }
  if (blockIdx.x == 0)
    for (int s = tid; s < Ts; s += kAtt * kGrp) {
      a.a_all[tb * Ts + s] = asm_[s];
      a.acc_all[((size_t)(a.t + 1) * a.B + b) * Ts + s] = a.acc_all[tb * Ts + s] + asm_[s];
    }
  if (g > 0) stf4(part + (g - 1) * kCols + q * 4, o);
  __syncthreads();
  if (g == 0 && on) {
#pragma unroll
    for (int h = 0; h < kGrp - 1; ++h) addf4(o, ldf4(part + h * kCols + q * 4));
    const int64_t row = (int64_t)a.t * a.B + b;
    st4(a.ro + row * a.pro + a.oa + c, o);
    if (a.t + 1 < a.T) st4(a.xa + (row + a.B) * a.pxa + c, o);
  }
}

struct AttBwd {
  int B, Ts, T, K, E, t, n1, nch, nsc;
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
  float* dap;            // [B][nch][Ts] d_a partials per column chunk
  float* dsp;            // [B][nsc][K] d s_tr partials per position chunk
  float* datt_all;       // [T][B][E]
  float* de_all;         // [T][B][Ts]
  bf16* ds;              // d s_tr -> row (t, b) of [T*B, pds]
  int64_t pds;
  float* ds32;  // [T*B, K]
  int b0;
};

// d att_t (readout part + the cell at t+1's dx) for 512 columns, and this chunk's part of
// d_a[s] = <d att_t, enc_s> for every position (tape.cpp:1031-1041); the position split
// and batched loads as in the context kernel
__global__ void __launch_bounds__(kAtt * kGrp, 2) dec_att_da_kernel(AttBwd a) {
  extern __shared__ float red[];  // [Ts][4]: per-warp partials (the 4 warps of the position's group)
  pdl_trigger();
  const int b = a.b0 + blockIdx.y, Ts = a.Ts, tid = threadIdx.x, lane = tid % 32, g = tid / kAtt, q = tid % kAtt;
  const int wig = q / 32, c = blockIdx.x * kCols + q * 4;
  const bool on = c < a.E;
  const size_t tb = (size_t)a.t * a.B + b;
  const int64_t row = (int64_t)a.t * a.B + b;
  const int len = min(max(a.lens[b], 0), Ts);
  const bf16* x = a.enc + (int64_t)b * Ts * a.ld_enc + c;
  uint2 raw[kPerGrpDa];
  const bf16* xc = on ? x : x - c;  // unconditional clamped loads (see the context kernel)
  auto load = [&](int s0) {
#pragma unroll
    for (int u = 0; u < kPerGrpDa; ++u)
      raw[u] = *reinterpret_cast<const uint2*>(xc + (int64_t)min(s0 + kGrp * u, Ts - 1) * a.ld_enc);
  };
  load(g);     // the first batch of encoder rows is in flight before the wait ...
  pdl_wait();  // ... for d att_t (G1 partials)
  float dv[4] = {0.f, 0.f, 0.f, 0.f};
  if (on) {
    addf4(dv, ldf4(a.dro + row * a.prf + a.oa + c));
    if (a.n1 > 0) {
      float4 u[kMaxSplit];  // unconditional (clamped) loads: all in flight together
#pragma unroll
      for (int z = 0; z < kMaxSplit; ++z) u[z] = ldf4(a.P1 + min(z, a.n1 - 1) * a.p1_stride + (int64_t)b * a.p1_ld + c);
#pragma unroll
      for (int z = 0; z < kMaxSplit; ++z)
        if (z < a.n1) addf4(dv, u[z]);
    }
    if (g == 0) stf4(a.datt_all + tb * a.E + c, dv);
  }
  for (int s0 = g; s0 < len; s0 += kGrp * kPerGrpDa) {
    if (s0 != g) load(s0);
#pragma unroll
    for (int u = 0; u < kPerGrpDa; ++u) {
      const int s = s0 + kGrp * u;
      const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[u].x));
      const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[u].y));
      float sum = ((dv[0] * lo.x + dv[1] * lo.y) + dv[2] * hi.x) + dv[3] * hi.y;
      sum = warp_sum(sum);
      if (lane == 0 && s < len) red[s * 4 + wig] = sum;
    }
  }
  __syncthreads();
  for (int s = tid; s < len; s += kAtt * kGrp)
    a.dap[((int64_t)b * a.nch + blockIdx.x) * Ts + s] = ((red[s * 4] + red[s * 4 + 1]) + red[s * 4 + 2]) + red[s * 4 + 3];
}

// softmax adjoint de = a (d_a - <a, d_a>) (tape.cpp:966-978; recomputed per CTA from the
// d_a partials), then for 8 positions d e_in = de v (1 - u^2): this chunk's d s_tr
// partial and d accum_{t-1} = d accum_t + d e_in W_fb
__global__ void __launch_bounds__(kAtt, 6) dec_att_tanh_kernel(AttBwd a) {
  extern __shared__ float sm[];  // de[Ts], a[Ts], then red[kPos][4]
  pdl_trigger();
  float* de = sm;
  float* as_ = sm + a.Ts;
  float* red = sm + 2 * a.Ts;
  const int b = a.b0 + blockIdx.y, j0 = blockIdx.x * kPos, Ts = a.Ts, K = a.K, tid = threadIdx.x;
  const int lane = tid % 32, warp = tid / 32, k0 = tid * 8;
  const size_t tb = (size_t)a.t * a.B + b;
  const bool act = k0 < K;
  uint4 x[kPos];  // unconditional clamped loads (see the energy kernel)
  const int kc = act ? k0 : 0;
#pragma unroll
  for (int p = 0; p < kPos; ++p)
    x[p] = *reinterpret_cast<const uint4*>(a.enc_ctx + ((int64_t)b * Ts + min(j0 + p, Ts - 1)) * a.pk + kc);
  const int len = min(max(a.lens[b], 0), Ts);
  pdl_wait();  // d_a partials (previous kernel) and the step's saves from here on
  float acp[kPos];
#pragma unroll
  for (int p = 0; p < kPos; ++p) acp[p] = a.acc_all[tb * Ts + min(j0 + p, Ts - 1)];
  for (int s = tid; s < Ts; s += kAtt) {  // d_a = sum of the column-chunk partials + d accum_t
    float u[kMaxSplit];  // unconditional (clamped) loads, masked below
#pragma unroll
    for (int h = 0; h < kMaxSplit; ++h) u[h] = a.dap[((int64_t)b * a.nch + min(h, a.nch - 1)) * Ts + s];
    const float dacc = a.dacc_in ? a.dacc_in[(int64_t)b * Ts + s] : 0.f;
    as_[s] = a.a_all[tb * Ts + s];
    float d = 0.f;
#pragma unroll
    for (int h = 0; h < kMaxSplit; ++h)
      if (h < a.nch) d += u[h];
    de[s] = s < len ? d + dacc : 0.f;
  }
  float st[8], wv[8], cv[8], vk[8], ds[8];
  if (act) {
    const float4 s0v = ldf4(a.str_all + tb * K + k0), s1v = ldf4(a.str_all + tb * K + k0 + 4);
    const float4 f0 = ldf4(a.b_fb + k0), f1 = ldf4(a.b_fb + k0 + 4), w0 = ldf4(a.W_fb + k0), w1 = ldf4(a.W_fb + k0 + 4);
    const float4 v0 = ldf4(a.v + k0), v1 = ldf4(a.v + k0 + 4);
    st[0] = s0v.x, st[1] = s0v.y, st[2] = s0v.z, st[3] = s0v.w, st[4] = s1v.x, st[5] = s1v.y, st[6] = s1v.z, st[7] = s1v.w;
    const float bf[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
    const float wf[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const float vf[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = st[i] + bf[i], wv[i] = wf[i], vk[i] = vf[i];
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) cv[i] = wv[i] = vk[i] = 0.f;
  }
  const int n = min(kPos, len - j0);
  __syncthreads();
  if (tid < 32) {
    float dot = 0.f;
    for (int s = lane; s < len; s += 32) dot += as_[s] * de[s];
    dot = warp_sum(dot);
    __syncwarp();
    for (int s = lane; s < Ts; s += 32) {
      const float d = s < len ? as_[s] * (de[s] - dot) : 0.f;
      de[s] = d;
      if (blockIdx.x == 0) a.de_all[tb * Ts + s] = d;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) ds[i] = 0.f;
#pragma unroll
  for (int p = 0; p < kPos; ++p) {
    float pa = 0.f;
    if (p < n && act) {
      const float des = de[j0 + p];
      float f[8];
      unpack8(x[p], f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float uu = tanh_approx(f[i] + acp[p] * wv[i] + cv[i]);
        const float dein = des * vk[i] * (1.f - uu * uu);
        ds[i] += dein;
        pa += wv[i] * dein;
      }
    }
    pa = warp_sum(pa);
    if (lane == 0) red[p * 4 + warp] = pa;
  }
  if (act && n > 0) {
    float* d = a.dsp + ((int64_t)b * a.nsc + blockIdx.x) * K + k0;
    const float d0[4] = {ds[0], ds[1], ds[2], ds[3]}, d1[4] = {ds[4], ds[5], ds[6], ds[7]};
    stf4(d, d0);
    stf4(d + 4, d1);
  }
  __syncthreads();
  if (tid < n) {
    const int s = j0 + tid;
    a.dacc_out[(int64_t)b * Ts + s] = (a.dacc_in ? a.dacc_in[(int64_t)b * Ts + s] : 0.f) +
                                      (((red[tid * 4] + red[tid * 4 + 1]) + red[tid * 4 + 2]) + red[tid * 4 + 3]);
  }
  if (blockIdx.x == 0)
    for (int s = len + tid; s < Ts; s += kAtt) a.dacc_out[(int64_t)b * Ts + s] = 0.f;
}

// d s_tr[b] = sum of the position-chunk partials in chunk order -> fp32 and the bf16 GEMM operand
__global__ void dec_att_dstr_kernel(AttBwd a) {
  pdl_trigger();
  pdl_wait();
  const int b = a.b0 + blockIdx.y, k = blockIdx.x * 256 + threadIdx.x;
  if (k >= a.K) return;
  const int len = min(max(a.lens[b], 0), a.Ts);
  const int nsc = (len + kPos - 1) / kPos;  // chunks that ran
  float d = 0.f;
  for (int q = 0; q < nsc; ++q) d += a.dsp[((int64_t)b * a.nsc + q) * a.K + k];
  const int64_t row = (int64_t)a.t * a.B + b;
  a.ds32[row * a.K + k] = d;
  a.ds[row * a.pds + k] = __float2bfloat16_rn(d);
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
  const int kc = act ? k0 : 0;
#pragma unroll
  for (int p = 0; p < kCtxPos; ++p) {  // unconditional clamped loads (masked by des = 0 below)
    x[p] = *reinterpret_cast<const uint4*>(a.enc_ctx + ((int64_t)b * Ts + min(s0 + p, Ts - 1)) * a.pk + kc);
#pragma unroll
    for (int i = 0; i < 8; ++i) dc[p][i] = 0.f;
  }
  if (act && n > 0) {
    const float* str = a.str_all + (size_t)b * K + k0;
    const size_t tstride = (size_t)a.B * K;
    float4 n0 = ldf4(str), n1 = ldf4(str + 4);  // s_tr of step t + 1 in flight while step t computes
    for (int t = 0; t < T; ++t) {
      const float4 s0v = n0, s1v = n1;
      if (t + 1 < T) n0 = ldf4(str + (t + 1) * tstride), n1 = ldf4(str + (t + 1) * tstride + 4);
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
  const float* dp = datt_all + (size_t)b * E + e;
  const size_t tstride = (size_t)B * E;
  float4 nd = ldf4(dp);  // d att of step t + 1 in flight while step t accumulates
  for (int t = 0; t < T; ++t) {
    const float4 d = nd;
    if (t + 1 < T) nd = ldf4(dp + (t + 1) * tstride);
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

// sum of split-K partials in split order -> rows < m_split to C, the rest to C2
__global__ void splitk_sum_kernel(const float* __restrict__ part, int ks, int64_t stride, int M, int N, int64_t ldp,
                                  float* C, int64_t ldc, int m_split, float* C2, int64_t ldc2) {
  const int r = blockIdx.y;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (c >= N) return;
  const float* p = part + (int64_t)r * ldp + c;
  float* dst = r < m_split ? C + (int64_t)r * ldc : C2 + (int64_t)(r - m_split) * ldc2;
  if (c + 4 <= N && (ldp % 4) == 0 && (((uintptr_t)(dst + c)) & 15) == 0) {
    float4 acc = ldf4(p);
    for (int z = 1; z < ks; ++z) {
      const float4 v = ldf4(p + z * stride);
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
    *reinterpret_cast<float4*>(dst + c) = acc;
  } else {
    for (int i = 0; i < 4 && c + i < N; ++i) {
      float acc = p[i];
      for (int z = 1; z < ks; ++z) acc += p[z * stride + i];
      dst[c + i] = acc;
    }
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

// Weight-gradient GEMMs (K = all B*T rows) with few output tiles leave most SMs idle:
// split K so the tiles x splits fill the CTA pairs, then sum the fp32 partials in a
// fixed order (deterministic).  Returns the split count (1: run as is).
int wgrad_ks(int M, int N, int K) {
  const int pairs = sm_count() / 2, tiles = (int)(ceil_div(M, 256) * ceil_div(N, 256));
  if (tiles * 2 >= pairs) return 1;
  const int nk = (int)ceil_div(K, 64);
  const int want = std::max(1, std::min(std::min(pairs / tiles, nk / 8), 8));
  return (int)ceil_div(nk, ceil_div(nk, want));
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
#ifdef SL_EXPERIMENTS
  static const bool off = getenv("SL_DEC_NO_PDL") != nullptr;
#else
  constexpr bool off = false;
#endif
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// split-K count for a batch-row GEMM (M <= 256 rows): fill the SM pairs, >= 4 K blocks per unit
// (the value gemm_bf16_tc2 re-derives: no empty units)
int ksplit_for(int M, int N, int K, int max_split = kMaxSplit) {
  const int tiles = (int)(ceil_div(M, 256) * ceil_div(N, 256));
  const int nk = (int)ceil_div(K, 64);
  const int want = std::max(1, std::min(std::min(sm_count() / 2 / tiles, nk / 4), max_split));
  return (int)ceil_div(nk, ceil_div(nk, want));
}

struct Lay {
  int PZ, PXA, OA, PRO, PK, PR, PRF, PDR;  // PDR: pitch of the [DZ | d readout] rows
  int PH;  // pitch of the d s = d s_tr W_s^T partials (H columns)
  int ks_f, ks_s, ks_1, ks_2;
  bool small;
  int ctx_blocks;
  bf16 *wd2, *wtrg, *wstr, *wctx, *wro, *wtrgcat;
  bf16 *enc_ctx, *xa, *ro, *dz, *ds, *drob, *dctx;
  int32_t* ids_tm;
  float *pre, *dtrg, *es, *dap, *dsp;
  float* wpart;  // split-K partials of the weight-gradient GEMMs
  size_t wpart_floats;
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
  L.PH = (int)round_up(d.H, 64);
  L.PR = (int)round_up(d.Rd, 64);
  L.PRF = L.PRO;
  L.PDR = L.PZ + L.PR;
  L.ks_f = ksplit_for(d.B, 4 * d.H, d.E + d.H);
  // the s_tr / d s projections (K = H or K columns, ~0.5 GFLOP) run on the mma.sync small-M
  // GEMM (SL_DEC_TC_SMALL=1: the tcgen05 pair GEMM with split-K instead)
#ifdef SL_EXPERIMENTS
  L.small = getenv("SL_DEC_TC_SMALL") == nullptr;
#else
  L.small = true;
#endif
  L.ks_s = L.small ? 1 : ksplit_for(d.B, d.K, d.H, 4);  // summed in the energy kernel (str_cols: at most 4)
  L.ks_1 = ksplit_for(d.B, d.E + d.H, 4 * d.H);
  L.ks_2 = L.small ? 1 : ksplit_for(d.B, d.H, d.K);
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
  L.es = tf((int64_t)d.B * d.Ts);
  L.dap = tf((int64_t)d.B * ceil_div(d.E, kCols) * d.Ts);
  L.dsp = tf((int64_t)d.B * ceil_div(d.Ts, kPos) * d.K);
  {
    const int64_t BT = (int64_t)d.B * d.T, BTs = (int64_t)d.B * d.Ts;
    const int64_t shapes[][3] = {{d.H, d.Rd, BT}, {d.Emb + 1, d.Rd, BT}, {d.E, d.Rd, BT}, {d.H, d.K, BT},
                                 {d.E, d.K, BTs}, {d.Emb + 1, 4 * d.H, BT}, {d.H, 4 * d.H, BT}};
    size_t need = 0;
    for (const auto& sh : shapes) {
      const int ks = wgrad_ks((int)sh[0], (int)sh[1], (int)sh[2]);
      if (ks > 1) need = std::max(need, (size_t)ks * sh[0] * round_up(sh[1], 4));
    }
    L.wpart_floats = need;
    L.wpart = need ? tf((int64_t)need) : nullptr;
  }
  L.xw = tf(BT * 4 * d.H);
  L.pf = tf((int64_t)L.ks_f * d.B * 4 * d.H);
  L.pstr = tf((int64_t)L.ks_s * d.B * L.PK);
  L.p1 = tf((int64_t)L.ks_1 * d.B * (d.E + d.H));
  L.p2 = tf((int64_t)L.ks_2 * d.B * L.PH);
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

void gemm_wgrad(const TcGemm& g, float* part, size_t part_floats, cudaStream_t st) {
  const int ks = wgrad_ks(g.M, g.N, g.K);
  const int64_t ldp = round_up(g.N, 4);
  if (ks <= 1 || !part || (size_t)ks * g.M * ldp > part_floats || g.beta != 0.f || g.bias || g.Cb) {
    gemm_bf16_tc(g, st);
    return;
  }
  TcGemm p = g;
  p.C = part;
  p.ldc = ldp;
  p.m_split = 1 << 30;
  p.C2 = nullptr;
  p.ldc2 = 0;
  p.ksplit = ks;
  p.split_stride = (int64_t)g.M * ldp;
  gemm_bf16_tc(p, st);
  splitk_sum_kernel<<<dim3((unsigned)ceil_div(ceil_div(g.N, 4), 256), (unsigned)g.M), 256, 0, st>>>(
      part, ks, (int64_t)g.M * ldp, g.M, g.N, ldp, g.C, g.ldc, g.m_split, g.C2, g.ldc2);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}
// split-K partials of a batch slice: partial z at C + z * stride (stride = full batch x ldc)
void gemm_split(TcGemm g, int ks, int64_t stride, cudaStream_t st) {
  g.ksplit = ks;
  g.split_stride = stride;
  gemm_bf16_tc(g, st);
}


void configure() {  // opt in to > 48 KB dynamic shared memory once
  static bool done = false;
  if (done) return;
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_ctx_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SL_CUDA_TRY(cudaFuncSetAttribute(dec_enc_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#ifdef SL_EXPERIMENTS
  const char* m = getenv("SL_DEC_TANH");
  const int mode = m ? atoi(m) : 0;
#else
  constexpr int mode = 0;
#endif
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
  SL_REQUIRE(d.K <= 1024 && d.E <= 4096 && d.Ts <= 1024 && d.T <= 1024 && (int64_t)d.T * d.Ts <= 48 * 1024,
             SL_ERR_UNSUPPORTED,
             "attn_decoder: key_dim <= 1024, enc_dim <= 4096, src/trg time <= 1024, src*trg time <= 48K supported");
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
  ph.reset();
  const double ctx_bytes = 2.0 * B * d.Ts * K, enc_bytes = 2.0 * B * d.Ts * E;  // per step, bf16 enc_ctx / enc
  for (int t = 0; t < T; ++t) {
    {  // (the launches take a batch-row range [b0, b0 + nb): one range = the whole batch)
      const int b0 = 0, nb = B;
      cudaStream_t ss = st;
      const int64_t r0 = (int64_t)t * B + b0;  // first time-major row of the slice at step t
      if (t > 0) {
        Phase q(ss, "k10_cell_gemm", 2.0 * nb * (E + H) * 4 * H);
        gemm_split(mk(nb, 4 * H, E + H, L.xa + r0 * L.PXA, L.PXA, false, L.wd2, L.PZ, true, L.pf + (int64_t)b0 * 4 * H,
                      4 * H),
                   L.ks_f, (int64_t)B * 4 * H, ss);
      }
      std::unique_ptr<Phase> q(new Phase(ss, "k10_cell_fwd", 0.0, 4.0 * nb * H * (4 * L.ks_f + 12)));
      CellFwd cf{B, T, H, E, t, t > 0 ? L.ks_f : 0, L.pf, 4 * H, (int64_t)B * 4 * H, L.xw, L.c_all, L.gates,
                 L.xa, L.PXA, L.ro, L.PRO, b0, nb};
      launch_pdl(dec_cell_fwd_kernel, dim3((unsigned)ceil_div(nb * (H / 4), 256)), dim3(256), 0, ss, cf);
      q.reset(new Phase(ss, "k10_str_gemm", 2.0 * nb * H * K));
      if (L.small)  // s_tr = s_t W_s on the mma.sync small-M GEMM: one fp32 result, no split
        small_gemm_bf16(nb, K, H, L.ro + r0 * L.PRO, L.PRO, L.wstr, L.PK, true, L.pstr + (int64_t)b0 * L.PK, L.PK,
                        nullptr, ss);
      else
        gemm_split(mk(nb, K, H, L.ro + r0 * L.PRO, L.PRO, false, L.wstr, L.PK, true, L.pstr + (int64_t)b0 * L.PK,
                      L.PK),
                   L.ks_s, (int64_t)B * L.PK, ss);
      AttFwd af{B, d.Ts, T, K, E, t, L.ks_s, src_lens, L.pstr, L.PK, (int64_t)B * L.PK, p.str_b, p.fb_W, p.fb_b,
                p.e_W, p.e_b, L.enc_ctx, L.PK, enc, ld_enc, L.es, L.str_all, L.a_all, L.acc_all, L.ro, L.PRO,
                L.OA, L.xa, L.PXA, b0};
      q.reset(new Phase(ss, "k10_att_energy", 0.0, ctx_bytes));
      launch_pdl(dec_att_energy_kernel, dim3((unsigned)ceil_div(d.Ts, kPos), (unsigned)nb), dim3(kAtt), 0, ss, af);
      q.reset(new Phase(ss, "k10_att_context", 0.0, enc_bytes));
      launch_pdl(dec_att_context_kernel, dim3((unsigned)ceil_div(E, kCols), (unsigned)nb), dim3(kAtt * kGrp),
                 (size_t)((d.Ts + 3) / 4 * 4 + (kGrp - 1) * kCols) * 4, ss, af);
      SL_CUDA_TRY(cudaGetLastError());
      count_launch(3);
    }
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
  gemm_wgrad(mk(H, Rd, (int)BT, L.ro, L.PRO, true, L.drob, L.PDR, true, g.ro_W, Rd), L.wpart, L.wpart_floats, st);
  {
    TcGemm w = mk(Emb + 1, Rd, (int)BT, L.ro + H, L.PRO, true, L.drob, L.PDR, true, g.ro_W + (int64_t)H * Rd, Rd);
    w.m_split = Emb;
    w.C2 = g.ro_b;
    w.ldc2 = Rd;
    gemm_wgrad(w, L.wpart, L.wpart_floats, st);
  }
  gemm_wgrad(mk(E, Rd, (int)BT, L.ro + L.OA, L.PRO, true, L.drob, L.PDR, true, g.ro_W + (int64_t)(H + Emb) * Rd, Rd),
             L.wpart, L.wpart_floats, st);
  ph.reset();
  ph.reset();
  const double ctx_bytes = 2.0 * B * d.Ts * K, enc_bytes = 2.0 * B * d.Ts * E;
  const int nch = (int)ceil_div(E, kCols), nsc = (int)ceil_div(d.Ts, kPos);
  for (int t = T - 1; t >= 0; --t) {
    const bool last = t == T - 1;
    {
      const int b0 = 0, nb = B;
      cudaStream_t ss = st;
      std::unique_ptr<Phase> q;
      if (!last) {
        q.reset(new Phase(ss, "k10_g1_gemm", 2.0 * nb * (E + H) * 4 * H));
        gemm_split(mk(nb, E + H, 4 * H, L.dz + ((int64_t)(t + 1) * B + b0) * L.PDR, L.PDR, false, L.wd2, L.PZ, false,
                      L.p1 + (int64_t)b0 * (E + H), E + H),
                   L.ks_1, (int64_t)B * (E + H), ss);
      }
      AttBwd ab{B, d.Ts, T, K, E, t, last ? 0 : L.ks_1, nch, nsc, src_lens, L.p1, E + H, (int64_t)B * (E + H), L.dro,
                L.PRF, L.OA, p.fb_W, p.fb_b, p.e_W, L.enc_ctx, L.PK, enc, ld_enc, L.str_all, L.a_all, L.acc_all,
                last ? nullptr : L.dacc + (int64_t)((t + 1) % 2) * B * d.Ts, L.dacc + (int64_t)(t % 2) * B * d.Ts,
                L.dap, L.dsp, L.datt_all, L.de_all, L.ds, L.PK, L.ds32, b0};
      q.reset(new Phase(ss, "k10_att_da", 0.0, enc_bytes));
      launch_pdl(dec_att_da_kernel, dim3((unsigned)nch, (unsigned)nb), dim3(kAtt * kGrp), (size_t)d.Ts * 16, ss, ab);
      q.reset(new Phase(ss, "k10_att_tanh", 0.0, ctx_bytes));
      launch_pdl(dec_att_tanh_kernel, dim3((unsigned)nsc, (unsigned)nb), dim3(kAtt), (size_t)(2 * d.Ts + 4 * kPos) * 4,
                 ss, ab);
      q.reset(new Phase(ss, "k10_att_dstr", 0.0, 4.0 * nb * K * (nsc + 2)));
      launch_pdl(dec_att_dstr_kernel, dim3((unsigned)ceil_div(K, 256), (unsigned)nb), dim3(256), 0, ss, ab);
      q.reset(new Phase(ss, "k10_g2_gemm", 2.0 * nb * H * K));
      if (L.small)  // d s += d s_tr W_s^T on the small-M GEMM
        small_gemm_bf16(nb, H, K, L.ds + ((int64_t)t * B + b0) * L.PK, L.PK, L.wstr, L.PK, false,
                        L.p2 + (int64_t)b0 * L.PH, L.PH, nullptr, ss);
      else
        gemm_split(mk(nb, H, K, L.ds + ((int64_t)t * B + b0) * L.PK, L.PK, false, L.wstr, L.PK, false,
                      L.p2 + (int64_t)b0 * L.PH, L.PH),
                   L.ks_2, (int64_t)B * L.PH, ss);
      CellBwd cb{B, T, H, E, t, last ? 0 : L.ks_1, L.p1, E + H, (int64_t)B * (E + H), L.ks_2, L.p2, L.PH,
                 (int64_t)B * L.PH, L.dro, L.PRF, L.gates, L.c_all,
                 last ? nullptr : L.dc + (int64_t)((t + 1) % 2) * B * H, L.dc + (int64_t)(t % 2) * B * H, L.dz, L.PDR,
                 b0, nb};
      q.reset(new Phase(ss, "k10_cell_bwd", 0.0, 4.0 * nb * H * (4 * L.ks_1 + 4 * L.ks_2 + 16)));
      launch_pdl(dec_cell_bwd_kernel, dim3((unsigned)ceil_div(nb * (H / 4), 256)), dim3(256), 0, ss, cb);
      SL_CUDA_TRY(cudaGetLastError());
      count_launch(4);
    }
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
  gemm_wgrad(mk(H, K, (int)BT, L.ro, L.PRO, true, L.ds, L.PK, true, g.str_W, K), L.wpart, L.wpart_floats, st);
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
    gemm_wgrad(mk(E, K, (int)BTs, enc, ld_enc, true, L.dctx, L.PK, true, g.ctx_W, K), L.wpart, L.wpart_floats, st);
  }
  ph.reset(new Phase(st, "k10_attn_accum", 0.0, 4.0 * T * B * E + 8.0 * BTs * E));
  dec_enc_grad_kernel<<<dim3((unsigned)ceil_div(E, kEncCols), (unsigned)ceil_div(d.Ts, kEncPos), (unsigned)B), 128,
                        (size_t)T * kEncPos * 4, st>>>(
      B, d.Ts, T, E, L.a_all, L.datt_all, d_enc, E);  // += sum_t a_t (x) d att_t
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();

}

}  // namespace sl
