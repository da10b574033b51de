// The Listing-1 attention decoder at the reference's precision (SL_PREC_FP32):
// the same computation as decoder.cu — the `output` subnetwork of models.cpp:
// 83-166 run step by step with teacher forcing as compiler.cpp:770-905 does,
// plus the base layer enc_ctx (models.cpp:60) —
//
//   enc_ctx = enc W_ctx + b_ctx                                   (once)
//   for t:  s_t, c_t = lstm_step([trg_{t-1} ‖ att_{t-1}], s_{t-1}, c_{t-1})   (tape.cpp:1074-1141)
//           s_tr = s_t W_s + b_s;  e = tanh(enc_ctx + accum_{t-1} W_fb + b_fb + s_tr) v + b_v
//           a_t = softmax over the valid source positions;  accum_t = accum_{t-1} + a_t
//           att_t = sum_j a_t[j] enc_j
//   readout = relu([s ‖ trg_prev ‖ att] W_ro + b_ro)             (all t at once)
//
// with every product fp32-class: the split-bf16 tcgen05 GEMM (gemm_f32x3.cu,
// A B = A_hi B_hi + A_lo B_hi + A_hi B_lo in fp32 TMEM, relative error ~1e-5),
// fp32 activations, cell state and attention (attention.cu, the 1e-4-tested
// single-step kernels), expf / tanhf.
//   * hoisted whole-sequence GEMMs: enc_ctx, trg_{t-1} W_trg + b for all t, the
//     readout, and in the backward every weight gradient over all T*B rows, d trg
//     and d enc through W_ctx;
//   * per step only the recurrence: [att ‖ s]_{t-1} [W_att; R] (weights split
//     once per call, only the [B, E+H] activations per step), the fused gate
//     kernel, the attention step; the backward mirrors it (attention adjoint,
//     gate adjoint, DZ_t [W_att; R]^T).
// Time-major per-step buffers (row t*B + b), fixed-order reductions.
#include <algorithm>

#include "attention.h"
#include "decoder.h"
#include "fastmath.cuh"
#include "embedding.h"
#include "gemm.h"
#include "profile.h"

namespace sl {
namespace {

constexpr int kEncPos = 30;   // positions per thread in the d enc accumulation (Ts = 60: d att read twice)
constexpr int kCtxPos = 8;    // positions per thread in the d enc_ctx accumulation
constexpr int kRedSlices = 64;  // f32_ctx_reduce1/2: row slices of the deferred attention partials

struct FLay {
  int64_t XA, RO;  // row pitches: [att ‖ s] (E + H), readout input [s ‖ trg ‖ att] (H + Emb + E)
  float *xw, *ro, *s_all, *att_all, *c_all, *gates, *enc_ctx, *a_all, *acc_all;
  __nv_bfloat16* xai;  // [att ‖ s]_{t-1} per step t as its split image [(T+1)*B, XA] (GEMM operand only)
  int64_t xai_ld, xai_lo;
  float *dro, *dpre, *dc, *ds, *dacc, *dctx;
  __nv_bfloat16* dzi;  // the cell's DZ [B*T, 4H] as its split image (every consumer is a GEMM)
  int64_t dzi_ld;
  float *datt_all, *de_all, *ds_all, *apart, *apart2;  // deferred attention accumulations (per step saves)
  int32_t* ids_tm;
  __nv_bfloat16 *wd2_f, *wd2_b;  // [W_att; R] split for z = xa W (fwd) and d xa = DZ W^T (bwd)
  __nv_bfloat16 *ws_f, *ws_b;    // W_s split for s_tr = s W_s and d s = d s_tr W_s^T
  float* str_all;                // [T, B, K] s_tr of every step (the backward reuses it)
  // split images of operands two GEMMs each read (one split serves both): the readout
  // input and enc with their ones columns (the bias-gradient rows), d pre and d enc_ctx
  __nv_bfloat16 *roi, *enci, *dprei, *dctxi;
  int64_t roi_ld, enci_ld, dprei_ld, dctxi_ld;
  void *att_ws, *gws, *emb_ws;
  size_t bytes;
};

size_t gemm_ws_bytes(const DecDims& d) {
  const int B = d.B, H = d.H, E = d.E, K = d.K, Emb = d.Emb, Rd = d.Rd;
  const int BT = B * d.T, BTs = B * d.Ts, XA = E + H, RO = H + Emb + E;
  return std::max({gemm_f32x3_workspace_bytes(false, false, BTs, K, E, false),      // enc_ctx
                   gemm_f32x3_workspace_bytes(false, false, BT, 4 * H, Emb, false),  // trg W_trg + b
                   gemm_f32x3_parts_workspace_bytes(false, false, B, 4 * H, XA),     // z (partials)
                   gemm_f32x3_parts_workspace_bytes(false, true, B, XA, 4 * H),      // d xa (partials)
                   gemm_f32x3_workspace_bytes(false, false, BT, Rd, RO, false),      // readout
                   gemm_f32x3_workspace_bytes(false, true, BT, RO, Rd, false),       // d readout input
                   gemm_f32x3_workspace_bytes(true, false, RO, Rd, BT, true),        // [d W_ro; d b_ro]
                   gemm_f32x3_workspace_bytes(true, false, E, 4 * H, BT, false),     // d W_att
                   gemm_f32x3_workspace_bytes(true, false, H, 4 * H, BT, false),     // d R
                   gemm_f32x3_workspace_bytes(true, false, Emb, 4 * H, BT, true),    // [d W_trg; d b]
                   gemm_f32x3_workspace_bytes(false, true, BT, Emb, 4 * H, false),   // d trg
                   gemm_f32x3_workspace_bytes(true, false, E, K, BTs, true),         // [d W_ctx; d b_ctx]
                   gemm_f32x3_workspace_bytes(false, true, BTs, E, K, false),        // d enc += d enc_ctx W_ctx^T
                   gemm_f32x3_workspace_bytes(true, false, H, K, BT, true)});        // [d W_s; d b_s]
}

FLay flayout(const DecDims& d, void* base) {
  FLay L{};
  const int64_t B = d.B, T = d.T, H = d.H, E = d.E, K = d.K;
  const int64_t BT = B * T, BTs = B * d.Ts;
  L.XA = E + H;
  L.RO = H + d.Emb + E;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = round_up(off, 256);
    void* r = p ? p + off : nullptr;
    off += bytes;
    return r;
  };
  auto tf = [&](int64_t n) { return static_cast<float*>(take((size_t)n * 4)); };
  L.xw = tf(BT * 4 * H);
  L.xai = static_cast<__nv_bfloat16*>(take(x3_img_elems((int)((T + 1) * B), (int)L.XA) * 2));
  L.xai_ld = x3_img_ld((int)L.XA);
  L.xai_lo = (T + 1) * B * L.xai_ld;
  L.ro = tf(BT * L.RO);
  L.s_all = tf(BT * H);
  L.att_all = tf(BT * E);
  L.c_all = tf(BT * H);
  L.gates = tf(BT * 5 * H);
  L.enc_ctx = tf(BTs * K);
  L.a_all = tf(T * B * d.Ts);
  L.acc_all = tf((T + 1) * B * d.Ts);
  L.dro = tf(BT * L.RO);
  L.dpre = tf(BT * d.Rd);
  L.dzi = static_cast<__nv_bfloat16*>(take(x3_img_elems((int)BT, (int)(4 * H)) * 2));
  L.dzi_ld = x3_img_ld((int)(4 * H));
  L.dc = tf(2 * B * H);
  L.ds = tf(B * H);
  L.dacc = tf(2 * B * d.Ts);
  L.dctx = tf(BTs * K);
  L.datt_all = tf(T * B * E);
  L.de_all = tf(T * B * d.Ts);
  L.ds_all = tf(T * B * K);
  L.apart = tf(B * ceil_div(d.Ts, kCtxPos) * 3 * K + 64);
  L.apart2 = tf(kRedSlices * (3 * K + 1));
  L.ids_tm = static_cast<int32_t*>(take((size_t)BT * 4));
  // the split images of [W_att; R] and W_s serve both the forward (B) and the backward (B^T) products
  L.wd2_f = static_cast<__nv_bfloat16*>(take(x3_img_elems((int)L.XA, (int)(4 * H)) * 2));
  L.wd2_b = L.wd2_f;
  L.ws_f = static_cast<__nv_bfloat16*>(take(x3_img_elems((int)H, (int)K) * 2));
  L.ws_b = L.ws_f;
  L.str_all = tf(T * B * K);
  auto timg = [&](int64_t rows, int64_t cols, __nv_bfloat16*& img, int64_t& ld) {
    img = static_cast<__nv_bfloat16*>(take(x3_img_elems((int)rows, (int)cols) * 2));
    ld = x3_img_ld((int)cols);
  };
  timg(BT, L.RO + 1, L.roi, L.roi_ld);
  timg(BTs, E + 1, L.enci, L.enci_ld);
  timg(BT, d.Rd, L.dprei, L.dprei_ld);
  timg(BTs, K, L.dctxi, L.dctxi_ld);
  L.att_ws = take(attention_workspace_bytes(d.B, d.K, d.H, d.Ts));
  L.gws = take(gemm_ws_bytes(d));
  L.emb_ws = take(embedding_workspace_bytes(BT, d.Vt));
  L.bytes = off + 256;
  return L;
}

__global__ void f32_ids_tm_kernel(const int32_t* __restrict__ ids, int B, int T, int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * T) return;
  const int t = (int)(i / B), b = (int)(i % B);
  out[i] = ids[(int64_t)b * T + t];
}

// the cell at step t (tape.cpp:1095-1135): z = [att ‖ s]_{t-1} [W_att; R] (null at t = 0) +
// trg_{t-1} W_trg + b; s_t into s_all, the next step's [att ‖ s] row and the readout input
struct GateF {
  int B, T, H, E, t;
  X3Parts z;         // [B, 4H] = h_{t-1} part of the gates as split-K partials (n = 0: none)
  const float* xw;   // [T*B, 4H]
  float *gates, *c_all, *s_all;
  __nv_bfloat16* xai;  // [att ‖ s] image rows (s written at column E of block t + 1)
  int64_t xai_ld, xai_lo;
  float* ro;         // [T*B, RO]
  int64_t RO;
};
__global__ void f32_cell_fwd_kernel(GateF a) {
  const int64_t n = (int64_t)a.B * a.H;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int b = (int)(e / a.H), j = (int)(e % a.H), H = a.H;
  const int64_t row = (int64_t)a.t * a.B + b;
  const float* x = a.xw + row * 4 * H;
  float z[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) z[g] = x[g * H + j] + x3_parts_sum(a.z, b, g * H + j);
  const float cp = a.t > 0 ? a.c_all[(row - a.B) * H + j] : 0.f;
  const float gi = sigmoidf_(z[0]), gf = sigmoidf_(z[1]), gg = tanhf(z[2]), go = sigmoidf_(z[3]);
  const float c = gf * cp + gi * gg;
  const float tc = tanhf(c);
  const float h = go * tc;
  a.c_all[row * H + j] = c;
  float* gs = a.gates + row * 5 * H + j;
  gs[0] = gi, gs[H] = gf, gs[2 * H] = gg, gs[3 * H] = go, gs[4 * H] = tc;
  a.s_all[row * H + j] = h;
  a.ro[row * a.RO + j] = h;
  {
    __nv_bfloat16* q = a.xai + (row + a.B) * a.xai_ld + a.E + j;
    const __nv_bfloat16 hh = __float2bfloat16_rn(h);
    q[0] = hh;
    q[a.xai_lo] = __float2bfloat16_rn(h - __bfloat162float(hh));
  }
}

// the same for 4 consecutive units per thread (H % 4 == 0, 16 B aligned rows): 16 B
// loads of x W and of the split-K partials, 16 B stores, identical arithmetic
__global__ void f32_cell_fwd4_kernel(GateF a) {
  const int H = a.H, H4 = H / 4;
  const int64_t n = (int64_t)a.B * H4;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int b = (int)(e / H4), j = (int)(e % H4) * 4;
  const int64_t row = (int64_t)a.t * a.B + b;
  const float* x = a.xw + row * 4 * H;
  float z[4][4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const float4 xv = *reinterpret_cast<const float4*>(x + g * H + j);
    float4 pv[8];
    const float* pp = a.z.p + (int64_t)b * a.z.ld + g * H + j;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      pv[q] = q < a.z.n ? __ldg(reinterpret_cast<const float4*>(pp + q * a.z.stride)) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 sv = make_float4(0.f, 0.f, 0.f, 0.f);  // the partials in order, as x3_parts_sum
#pragma unroll
    for (int q = 0; q < 8; ++q) sv.x += pv[q].x, sv.y += pv[q].y, sv.z += pv[q].z, sv.w += pv[q].w;
    for (int q = 8; q < a.z.n; ++q) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(pp + q * a.z.stride));
      sv.x += t.x, sv.y += t.y, sv.z += t.z, sv.w += t.w;
    }
    z[g][0] = xv.x + sv.x, z[g][1] = xv.y + sv.y, z[g][2] = xv.z + sv.z, z[g][3] = xv.w + sv.w;
  }
  const float4 cp4 = a.t > 0 ? *reinterpret_cast<const float4*>(a.c_all + (row - a.B) * H + j)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  const float cpv[4] = {cp4.x, cp4.y, cp4.z, cp4.w};
  float gi[4], gf[4], gg[4], go[4], c[4], tc[4], h[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    gi[u] = sigmoidf_(z[0][u]), gf[u] = sigmoidf_(z[1][u]), gg[u] = tanhf(z[2][u]), go[u] = sigmoidf_(z[3][u]);
    c[u] = gf[u] * cpv[u] + gi[u] * gg[u];
    tc[u] = tanhf(c[u]);
    h[u] = go[u] * tc[u];
  }
  auto st4 = [](float* p, const float (&v)[4]) { *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]); };
  st4(a.c_all + row * H + j, c);
  float* gs = a.gates + row * 5 * H + j;
  st4(gs, gi), st4(gs + H, gf), st4(gs + 2 * H, gg), st4(gs + 3 * H, go), st4(gs + 4 * H, tc);
  st4(a.s_all + row * H + j, h);
  st4(a.ro + row * a.RO + j, h);
  __nv_bfloat16 hh[4], hl[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    hh[u] = __float2bfloat16_rn(h[u]);
    hl[u] = __float2bfloat16_rn(h[u] - __bfloat162float(hh[u]));
  }
  __nv_bfloat16* q = a.xai + (row + a.B) * a.xai_ld + a.E + j;
  *reinterpret_cast<uint2*>(q) = *reinterpret_cast<const uint2*>(hh);
  *reinterpret_cast<uint2*>(q + a.xai_lo) = *reinterpret_cast<const uint2*>(hl);
}

// readout [b, t] = relu(pre [t*B + b])
__global__ void f32_relu_kernel(const float* __restrict__ pre, float* __restrict__ out, int B, int T, int Rd) {
  const int64_t n = (int64_t)B * T * Rd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % Rd);
    const int64_t bt = i / Rd;
    const int b = (int)(bt / T), t = (int)(bt % T);
    out[i] = fmaxf(pre[((int64_t)t * B + b) * Rd + c], 0.f);
  }
}

// the same two maps with one CTA per row (b, t) and 4 columns per thread (Rd % 4 == 0):
// no per-element index division, 16 B accesses
__global__ void f32_relu4_kernel(const float* __restrict__ pre, float* __restrict__ out, int B, int T, int Rd) {
  for (int64_t r = blockIdx.x; r < (int64_t)B * T; r += gridDim.x) {  // r = b * T + t (the readout row)
    const int b = (int)(r / T), t = (int)(r - (int64_t)b * T);
    const float* src = pre + ((int64_t)t * B + b) * Rd;
    float* dst = out + r * Rd;
    for (int c = threadIdx.x * 4; c < Rd; c += blockDim.x * 4) {
      const float4 v = *reinterpret_cast<const float4*>(src + c);
      *reinterpret_cast<float4*>(dst + c) = make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
    }
  }
}
__global__ void f32_relu_bwd4_kernel(const float* __restrict__ ro, const float* __restrict__ dro,
                                     float* __restrict__ dpre, int B, int T, int Rd) {
  for (int64_t r = blockIdx.x; r < (int64_t)B * T; r += gridDim.x) {
    const int b = (int)(r / T), t = (int)(r - (int64_t)b * T);
    float* dst = dpre + ((int64_t)t * B + b) * Rd;
    for (int c = threadIdx.x * 4; c < Rd; c += blockDim.x * 4) {
      const float4 y = *reinterpret_cast<const float4*>(ro + r * Rd + c);
      const float4 g = *reinterpret_cast<const float4*>(dro + r * Rd + c);
      *reinterpret_cast<float4*>(dst + c) =
          make_float4(y.x > 0.f ? g.x : 0.f, y.y > 0.f ? g.y : 0.f, y.z > 0.f ? g.z : 0.f, y.w > 0.f ? g.w : 0.f);
    }
  }
}

// d pre [t*B + b] = d readout [b, t] * [readout > 0]
__global__ void f32_relu_bwd_kernel(const float* __restrict__ ro, const float* __restrict__ dro,
                                    float* __restrict__ dpre, int B, int T, int Rd) {
  const int64_t n = (int64_t)B * T * Rd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % Rd);
    const int64_t bt = i / Rd;
    const int b = (int)(bt / T), t = (int)(bt % T);
    dpre[((int64_t)t * B + b) * Rd + c] = ro[i] > 0.f ? dro[i] : 0.f;
  }
}

// the upstream gradients of step t: d att_t (readout + the cell at t + 1), d s_t (readout +
// the cell at t + 1; the attention adds its d s_tr W_s^T)
struct GradIn {
  int B, H, E, t, has_next;
  const float* dro;  // [T*B, RO]
  int64_t RO;
  int Emb;
  X3Parts dxa;       // [B, XA]: d [att ‖ s]_t from the cell at t + 1, as split-K partials
  float *datt, *ds;
};
__global__ void f32_grad_in_kernel(GradIn a) {
  const int W = a.E + a.H;
  const int64_t n = (int64_t)a.B * W;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int b = (int)(e / W), c = (int)(e % W);
  const float* r = a.dro + ((int64_t)a.t * a.B + b) * a.RO;
  if (c < a.E) {
    float v = r[a.H + a.Emb + c];
    if (a.has_next) v += x3_parts_sum(a.dxa, b, c);
    a.datt[(int64_t)b * a.E + c] = v;
  } else {
    const int j = c - a.E;
    float v = r[j];
    if (a.has_next) v += x3_parts_sum(a.dxa, b, a.E + j);
    a.ds[(int64_t)b * a.H + j] = v;
  }
}

// the same for 4 consecutive columns per thread (E % 4 == H % 4 == 0, 16 B aligned rows)
__global__ void f32_grad_in4_kernel(GradIn a) {
  const int W4 = (a.E + a.H) / 4;
  const int64_t n = (int64_t)a.B * W4;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int b = (int)(e / W4), c = (int)(e % W4) * 4;
  const float* r = a.dro + ((int64_t)a.t * a.B + b) * a.RO;
  const bool att = c < a.E;
  float4 v = *reinterpret_cast<const float4*>(att ? r + a.H + a.Emb + c : r + (c - a.E));
  if (a.has_next) {  // the partials in order, as x3_parts_sum
    const float* pp = a.dxa.p + (int64_t)b * a.dxa.ld + c;
    float4 pv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      pv[q] = q < a.dxa.n ? __ldg(reinterpret_cast<const float4*>(pp + q * a.dxa.stride)) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 sv = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 8; ++q) sv.x += pv[q].x, sv.y += pv[q].y, sv.z += pv[q].z, sv.w += pv[q].w;
    for (int q = 8; q < a.dxa.n; ++q) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(pp + q * a.dxa.stride));
      sv.x += t.x, sv.y += t.y, sv.z += t.z, sv.w += t.w;
    }
    v.x += sv.x, v.y += sv.y, v.z += sv.z, v.w += sv.w;
  }
  float* dst = att ? a.datt + (int64_t)b * a.E + c : a.ds + (int64_t)b * a.H + (c - a.E);
  *reinterpret_cast<float4*>(dst) = v;
}

// the cell adjoint at step t (tape.cpp:1157-1170): gh = d s_t, gc = d c_t -> DZ_t, d c_{t-1}
struct CellBF {
  int B, H, t;
  const float *ds, *gates, *c_all, *dc_in;
  X3Parts ds_att;      // the attention's d s = d s_tr W_s^T as split-K partials (added to ds)
  __nv_bfloat16* dzi;  // DZ image: hi rows at dzi (stride ld), lo rows lo elements further on
  int64_t ld, lo;
  float* dc_out;
};
__device__ __forceinline__ void put_split(__nv_bfloat16* hi, int64_t lo, float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  hi[0] = h;
  hi[lo] = __float2bfloat16_rn(v - __bfloat162float(h));
}
__global__ void f32_cell_bwd_kernel(CellBF a) {
  const int64_t n = (int64_t)a.B * a.H;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int b = (int)(e / a.H), j = (int)(e % a.H), H = a.H;
  const int64_t row = (int64_t)a.t * a.B + b;
  const float gh = a.ds[e] + x3_parts_sum(a.ds_att, b, j), gc = a.dc_in ? a.dc_in[e] : 0.f;
  const float* gs = a.gates + row * 5 * H + j;
  const float gi = gs[0], gf = gs[H], gg = gs[2 * H], go = gs[3 * H], tc = gs[4 * H];
  const float cp = a.t > 0 ? a.c_all[(row - a.B) * H + j] : 0.f;
  const float d_o = gh * tc;
  const float dc = gc + gh * go * (1.f - tc * tc);
  a.dc_out[e] = dc * gf;
  __nv_bfloat16* dz = a.dzi + row * a.ld + j;
  put_split(dz, a.lo, dc * gg * gi * (1.f - gi));
  put_split(dz + H, a.lo, dc * cp * gf * (1.f - gf));
  put_split(dz + 2 * H, a.lo, dc * gi * (1.f - gg * gg));
  put_split(dz + 3 * H, a.lo, d_o * go * (1.f - go));
}

// the same for 4 consecutive units per thread (16 B loads and stores, 8 B image stores)
__global__ void f32_cell_bwd4_kernel(CellBF a) {
  const int H = a.H, H4 = H / 4;
  const int64_t n = (int64_t)a.B * H4;
  const int64_t e4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e4 >= n) return;
  const int b = (int)(e4 / H4), j = (int)(e4 % H4) * 4;
  const int64_t e = (int64_t)b * H + j, row = (int64_t)a.t * a.B + b;
  auto ld4 = [](const float* p, float (&v)[4]) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
  };
  float ds[4], gc[4] = {0.f, 0.f, 0.f, 0.f}, gi[4], gf[4], gg[4], go[4], tc[4], cp[4] = {0.f, 0.f, 0.f, 0.f};
  ld4(a.ds + e, ds);
  {  // + the attention's d s partials, in order (as x3_parts_sum)
    float4 pv[8];
    const float* pp = a.ds_att.p + (int64_t)b * a.ds_att.ld + j;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      pv[q] = q < a.ds_att.n ? __ldg(reinterpret_cast<const float4*>(pp + q * a.ds_att.stride))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 sv = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < 8; ++q) sv.x += pv[q].x, sv.y += pv[q].y, sv.z += pv[q].z, sv.w += pv[q].w;
    for (int q = 8; q < a.ds_att.n; ++q) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(pp + q * a.ds_att.stride));
      sv.x += t.x, sv.y += t.y, sv.z += t.z, sv.w += t.w;
    }
    ds[0] += sv.x, ds[1] += sv.y, ds[2] += sv.z, ds[3] += sv.w;
  }
  if (a.dc_in) ld4(a.dc_in + e, gc);
  const float* gs = a.gates + row * 5 * H + j;
  ld4(gs, gi), ld4(gs + H, gf), ld4(gs + 2 * H, gg), ld4(gs + 3 * H, go), ld4(gs + 4 * H, tc);
  if (a.t > 0) ld4(a.c_all + (row - a.B) * H + j, cp);
  float dco[4], z[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float gh = ds[u];
    const float d_o = gh * tc[u];
    const float dc = gc[u] + gh * go[u] * (1.f - tc[u] * tc[u]);
    dco[u] = dc * gf[u];
    z[0][u] = dc * gg[u] * gi[u] * (1.f - gi[u]);
    z[1][u] = dc * cp[u] * gf[u] * (1.f - gf[u]);
    z[2][u] = dc * gi[u] * (1.f - gg[u] * gg[u]);
    z[3][u] = d_o * go[u] * (1.f - go[u]);
  }
  *reinterpret_cast<float4*>(a.dc_out + e) = make_float4(dco[0], dco[1], dco[2], dco[3]);
  __nv_bfloat16* dz = a.dzi + row * a.ld + j;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    __nv_bfloat16 hi[4], lo[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      hi[u] = __float2bfloat16_rn(z[g][u]);
      lo[u] = __float2bfloat16_rn(z[g][u] - __bfloat162float(hi[u]));
    }
    *reinterpret_cast<uint2*>(dz + g * H) = *reinterpret_cast<const uint2*>(hi);
    *reinterpret_cast<uint2*>(dz + g * H + a.lo) = *reinterpret_cast<const uint2*>(lo);
  }
}

// d enc[b, s, :] = sum_t a_t[b, s] d att_t[b, :]  (the generic_attention adjoint w.r.t.
// its base, tape.cpp:1047-1058, accumulated over the steps in t order).  A thread owns 4
// columns x kEncPos positions; the block stages a_t[b, s0 .. s0 + kEncPos) of every t.
__global__ void __launch_bounds__(128) f32_enc_grad_kernel(int B, int Ts, int T, int E, const float* __restrict__ a_all,
                                                         const float* __restrict__ datt_all, float* __restrict__ d_enc) {
  extern __shared__ float a_sh[];  // [T][kEncPos]
  const int b = blockIdx.z, s0 = blockIdx.y * kEncPos, e = (blockIdx.x * 128 + threadIdx.x) * 4;
  for (int i = threadIdx.x; i < T * kEncPos; i += 128) {
    const int t = i / kEncPos, j = i % kEncPos;
    a_sh[i] = s0 + j < Ts ? a_all[((int64_t)t * B + b) * Ts + s0 + j] : 0.f;
  }
  __syncthreads();
  if (e >= E) return;
  float4 acc[kEncPos];
#pragma unroll
  for (int j = 0; j < kEncPos; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  int t = 0;
  for (; t + 4 <= T; t += 4) {  // four steps' d att rows in flight, then the updates in t order
    float4 g[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) g[i] = *reinterpret_cast<const float4*>(datt_all + ((int64_t)(t + i) * B + b) * E + e);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < kEncPos; ++j) {
        const float w = a_sh[(t + i) * kEncPos + j];
        acc[j].x += w * g[i].x, acc[j].y += w * g[i].y, acc[j].z += w * g[i].z, acc[j].w += w * g[i].w;
      }
  }
  for (; t < T; ++t) {
    const float4 g = *reinterpret_cast<const float4*>(datt_all + ((int64_t)t * B + b) * E + e);
#pragma unroll
    for (int j = 0; j < kEncPos; ++j) {
      const float w = a_sh[t * kEncPos + j];
      acc[j].x += w * g.x, acc[j].y += w * g.y, acc[j].z += w * g.z, acc[j].w += w * g.w;
    }
  }
#pragma unroll
  for (int j = 0; j < kEncPos; ++j)
    if (s0 + j < Ts) *reinterpret_cast<float4*>(d_enc + ((int64_t)b * Ts + s0 + j) * E + e) = acc[j];
}

__device__ __forceinline__ float tanh_fast_f(float x) {  // as attention.cu's energies
  x = fminf(fmaxf(x, -15.f), 15.f);
  return 1.f - __fdividef(2.f, 1.f + __expf(2.f * x));
}

// the energy adjoints summed over the steps (tape.cpp:966-978 then the tanh / weight
// feedback adjoints): d enc_ctx[b, s, k] = sum_t de_t[b, s] v_k (1 - u_t^2) with
// u_t = tanh(enc_ctx + accum_{t-1} W_fb + b_fb + s_tr_t) recomputed, and this block's
// partial sums over its positions of d W_fb (accum gk), d b_fb (gk), d v (u de) per k
// (reduced in a fixed order afterwards).  A thread owns one k x kCtxPos positions.
__global__ void __launch_bounds__(128) f32_ctx_grad_kernel(int B, int Ts, int T, int K, const float* __restrict__ enc_ctx,
                                                         const float* __restrict__ acc_all,
                                                         const float* __restrict__ de_all,
                                                         const float* __restrict__ str_all, const float* __restrict__ W_fb,
                                                         const float* __restrict__ b_fb, const float* __restrict__ v,
                                                         float* __restrict__ d_ctx, float* __restrict__ part) {
  extern __shared__ float sh[];  // acc [T][kCtxPos], de [T][kCtxPos]
  float* acc_sh = sh;
  float* de_sh = sh + T * kCtxPos;
  const int b = blockIdx.z, sc = blockIdx.y, s0 = sc * kCtxPos, k = blockIdx.x * 128 + threadIdx.x;
  for (int i = threadIdx.x; i < T * kCtxPos; i += 128) {
    const int t = i / kCtxPos, j = i % kCtxPos;
    const bool ok = s0 + j < Ts;
    acc_sh[i] = ok ? acc_all[((int64_t)t * B + b) * Ts + s0 + j] : 0.f;  // accum_{t-1} (block t)
    de_sh[i] = ok ? de_all[((int64_t)t * B + b) * Ts + s0 + j] : 0.f;
  }
  __syncthreads();
  if (k >= K) return;
  float x[kCtxPos], g[kCtxPos];
#pragma unroll
  for (int j = 0; j < kCtxPos; ++j) {
    x[j] = s0 + j < Ts ? enc_ctx[((int64_t)b * Ts + s0 + j) * K + k] : 0.f;
    g[j] = 0.f;
  }
  const float w = W_fb[k], c = b_fb[k], vk = v[k];
  // paired-fp32 math over pairs of positions (two per instruction; MUFU-bound after)
  using namespace fm;
  float2 g2[kCtxPos / 2], dwf2 = s2(0.f), dbf2 = s2(0.f), dv2 = s2(0.f);
#pragma unroll
  for (int j = 0; j < kCtxPos / 2; ++j) g2[j] = s2(0.f);
  for (int t = 0; t < T; ++t) {
    const float cs = c + str_all[((int64_t)t * B + b) * K + k];
#pragma unroll
    for (int j = 0; j < kCtxPos / 2; ++j) {
      const float2 a = *reinterpret_cast<const float2*>(acc_sh + t * kCtxPos + 2 * j);
      const float2 de = *reinterpret_cast<const float2*>(de_sh + t * kCtxPos + 2 * j);
      const float2 u = tanh2(fma2(a, s2(w), add2(make_float2(x[2 * j], x[2 * j + 1]), s2(cs))));
      const float2 gk = mul2(mul2(de, s2(vk)), fma2(make_float2(-u.x, -u.y), u, s2(1.f)));
      g2[j] = add2(g2[j], gk);
      dwf2 = fma2(a, gk, dwf2);
      dbf2 = add2(dbf2, gk);
      dv2 = fma2(u, de, dv2);
    }
  }
  const float dwf = dwf2.x + dwf2.y, dbf = dbf2.x + dbf2.y, dv = dv2.x + dv2.y;
#pragma unroll
  for (int j = 0; j < kCtxPos; ++j)
    g[j] = (j & 1) ? g2[j / 2].y : g2[j / 2].x;
#pragma unroll
  for (int j = 0; j < kCtxPos; ++j)
    if (s0 + j < Ts) d_ctx[((int64_t)b * Ts + s0 + j) * K + k] = g[j];
  const int64_t row = (int64_t)b * gridDim.y + sc;
  part[(row * 3 + 0) * K + k] = dwf;
  part[(row * 3 + 1) * K + k] = dbf;
  part[(row * 3 + 2) * K + k] = dv;
}

// out_q[k] = sum over rows r (ascending) of part[(r * 3 + q) * K + k], q = 0, 1, 2;
// and (thread 0 of block 0) *dbv = sum of de_all in a fixed order
// Deterministic two-stage reduction of f32_ctx_grad's per-(b, source chunk) partials
// and of d b_v = sum of every energy adjoint: stage 1 sums fixed row slices (and a
// fixed segment of de_all per slice), stage 2 sums the slices in order.
__global__ void __launch_bounds__(128) f32_ctx_reduce1_kernel(int rows, int K, const float* __restrict__ part,
                                                              const float* __restrict__ de_all, int64_t n_de,
                                                              float* __restrict__ part2) {
  const int slice = blockIdx.y, k = blockIdx.x * 128 + threadIdx.x;
  const int rps = (rows + kRedSlices - 1) / kRedSlices;
  const int r0 = slice * rps, r1 = min(rows, r0 + rps);
  if (k < K) {
    float a = 0.f, c = 0.f, e = 0.f;
    for (int r = r0; r < r1; ++r) {
      a += part[((int64_t)r * 3 + 0) * K + k];
      c += part[((int64_t)r * 3 + 1) * K + k];
      e += part[((int64_t)r * 3 + 2) * K + k];
    }
    part2[((int64_t)slice * 3 + 0) * K + k] = a;
    part2[((int64_t)slice * 3 + 1) * K + k] = c;
    part2[((int64_t)slice * 3 + 2) * K + k] = e;
  }
  if (blockIdx.x == 0) {  // this slice's segment of the energy adjoints
    __shared__ float red[4];
    const int64_t seg = (n_de + kRedSlices - 1) / kRedSlices;
    const int64_t i0 = slice * seg, i1 = min(n_de, i0 + seg);
    float sum = 0.f;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += 128) sum += de_all[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) part2[(int64_t)kRedSlices * 3 * K + slice] = (red[0] + red[1]) + (red[2] + red[3]);
  }
}

__global__ void __launch_bounds__(128) f32_ctx_reduce2_kernel(int K, const float* __restrict__ part2, float* dwf,
                                                              float* dbf, float* dv, float* dbv) {
  const int k = blockIdx.x * 128 + threadIdx.x;
  if (k < K) {
    float a = 0.f, c = 0.f, e = 0.f;
    for (int r = 0; r < kRedSlices; ++r) {
      a += part2[((int64_t)r * 3 + 0) * K + k];
      c += part2[((int64_t)r * 3 + 1) * K + k];
      e += part2[((int64_t)r * 3 + 2) * K + k];
    }
    dwf[k] = a, dbf[k] = c, dv[k] = e;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    float sum = 0.f;
    for (int r = 0; r < kRedSlices; ++r) sum += part2[(int64_t)kRedSlices * 3 * K + r];
    *dbv = sum;
  }
}

unsigned grid_of(int64_t n) { return (unsigned)ceil_div(n, 256); }

AttnArgs att_args(const DecDims& d, const FLay& L, const DecParams& p, const float* enc, const int32_t* lens,
                  int t) {
  AttnArgs a{};
  a.B = d.B;
  a.Ts = d.Ts;
  a.K = d.K;
  a.E = d.E;
  a.H = d.H;
  a.lens = lens;
  a.enc_ctx = L.enc_ctx;
  a.enc = enc;
  a.accum = L.acc_all + (int64_t)t * d.B * d.Ts;  // accum_{t-1}
  a.W_fb = p.fb_W;
  a.b_fb = p.fb_b;
  a.v = p.e_W;
  a.b_v = p.e_b;
  a.W_s3_fwd = L.ws_f;
  a.W_s3_bwd = L.ws_b;
  return a;
}

}  // namespace

size_t decoder_f32_workspace_bytes(const DecDims& d) { return flayout(d, nullptr).bytes; }

void decoder_f32_check(const DecDims& d) {
  SL_REQUIRE(d.B > 0 && d.Ts > 0 && d.T > 0 && d.Emb > 0 && d.E > 0 && d.H > 0 && d.K > 0 && d.Rd > 0 && d.Vt > 0,
             SL_ERR_SHAPE, "attn_decoder: dimensions must be positive");
  SL_REQUIRE(d.Ts <= 4096 && d.T <= 1024, SL_ERR_UNSUPPORTED, "attn_decoder (fp32): src_time <= 4096, trg_time <= 1024");
  SL_REQUIRE(d.E % 4 == 0, SL_ERR_UNSUPPORTED, "attn_decoder (fp32): enc_dim must be a multiple of 4");
}

void decoder_f32_fwd(const DecDims& d, const DecParams& p, const float* enc, const int32_t* src_lens,
                     const int32_t* prev_ids, float* readout, int32_t* bad_row, void* ws, cudaStream_t st) {
  decoder_f32_check(d);
  const FLay L = flayout(d, ws);
  const int B = d.B, T = d.T, H = d.H, E = d.E, K = d.K, Emb = d.Emb;
  const int64_t BT = (int64_t)B * T, BTs = (int64_t)B * d.Ts;
  {
    Phase ph(st, "k10_dec_fwd_hoisted", 2.0 * BTs * E * K + 2.0 * BT * Emb * 4 * H);
    // [att ‖ s]_{-1} = 0 (hi and lo rows of block 0)
    SL_CUDA_TRY(cudaMemsetAsync(L.xai, 0, sizeof(__nv_bfloat16) * B * L.xai_ld, st));
    SL_CUDA_TRY(cudaMemsetAsync(L.xai + L.xai_lo, 0, sizeof(__nv_bfloat16) * B * L.xai_ld, st));
    SL_CUDA_TRY(cudaMemsetAsync(L.acc_all, 0, sizeof(float) * BTs, st));  // accum_{-1} = 0
    // [W_att; R] (rows Emb.. of s/W stacked on s/R) split once into the image the per-step
    // GEMMs read in both roles: each block straight into its rows of the image
    {
      const int64_t wl = x3_img_ld((int)(4 * H)), wlo = (int64_t)L.XA * wl;
      x3_split_into(p.s_W + (int64_t)Emb * 4 * H, 4 * H, E, 4 * H, -1, L.wd2_f, wl, wl, wlo, st);
      x3_split_into(p.s_R, 4 * H, H, 4 * H, -1, L.wd2_f + (int64_t)E * wl, wl, wl, wlo, st);
    }
    x3_split_img(p.str_W, K, H, K, L.ws_f, st);  // W_s [H, K], both roles
    f32_ids_tm_kernel<<<grid_of(BT), 256, 0, st>>>(prev_ids, B, T, L.ids_tm);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
    // trg_{t-1} straight into the readout-input rows (columns H..H+Emb)
    embedding_fwd(BT, L.ids_tm, d.Vt, Emb, p.trg_W, L.ro + H, L.RO, SL_EMB_NEGATIVE_ZERO, bad_row, st);
    // enc's image (ones column at E for the backward's d b_ctx row), kept for that GEMM
    x3_split_into(enc, E, (int)BTs, E, E, L.enci, L.enci_ld, L.enci_ld, BTs * L.enci_ld, st);
    gemm_f32x3_ex(false, false, (int)BTs, K, E, nullptr, 0, L.enci, p.ctx_W, K, nullptr, 0.f, L.enc_ctx, K, p.ctx_b,
                  nullptr, 0, L.gws, st, L.enci_ld, BTs * L.enci_ld);
    gemm_f32x3(false, false, (int)BT, 4 * H, Emb, L.ro + H, L.RO, p.s_W, 4 * H, 0.f, L.xw, 4 * H, p.s_b, nullptr, 0,
               L.gws, st);
  }
  for (int t = 0; t < T; ++t) {
    X3Parts zp{nullptr, 0, 0, 0};
    if (t > 0) {  // [att ‖ s]_{t-1} [W_att; R] as split-K partials, summed by the gate kernel
      Phase q(st, "k10_cell_gemm", 2.0 * B * (E + H) * 4.0 * H);
      zp = gemm_f32x3_parts(false, false, B, 4 * H, E + H, nullptr, 0, L.xai + (int64_t)t * B * L.xai_ld, nullptr,
                            0, L.wd2_f, L.gws, st, L.xai_ld, L.xai_lo);
    }
    {
      Phase q(st, "k10_cell_fwd", 0.0, 4.0 * B * H * 12);
      GateF g{B, T, H, E, t, zp, L.xw, L.gates, L.c_all, L.s_all, L.xai, L.xai_ld, L.xai_lo, L.ro, L.RO};
      // 4 units per thread where every row and partial is 16 B aligned
      const bool v4 = H % 4 == 0 && L.RO % 4 == 0 && (zp.n == 0 || (zp.ld % 4 == 0 && zp.stride % 4 == 0 &&
                                                                   (reinterpret_cast<uintptr_t>(zp.p) & 15) == 0)) &&
                      (E + L.xai_ld) % 4 == 0 && L.xai_lo % 4 == 0;
      if (v4) f32_cell_fwd4_kernel<<<grid_of((int64_t)B * H / 4), 256, 0, st>>>(g);
      else f32_cell_fwd_kernel<<<grid_of((int64_t)B * H), 256, 0, st>>>(g);
      SL_CUDA_TRY(cudaGetLastError());
      count_launch();
    }
    AttnArgs a = att_args(d, L, p, enc, src_lens, t);
    a.att = L.att_all + (int64_t)t * B * E;
    a.a = L.a_all + (int64_t)t * B * d.Ts;
    a.accum_out = L.acc_all + (int64_t)(t + 1) * B * d.Ts;
    a.s_tr_out = L.str_all + (int64_t)t * B * K;
    // att_t also -> the readout input (columns H + Emb..) and the next step's [att ‖ s] row
    a.att_copy[0] = L.ro + (int64_t)t * B * L.RO + H + Emb;
    a.att_copy_ld[0] = L.RO;
    a.att_copy[1] = nullptr;
    a.att_img = t + 1 < T ? L.xai + (int64_t)(t + 1) * B * L.xai_ld : nullptr;
    a.att_img_ld = L.xai_ld;
    a.att_img_lo = L.xai_lo;
    a.s_img = L.xai + (int64_t)(t + 1) * B * L.xai_ld + E;  // s_t: block t + 1, columns E..
    a.s_img_ld = L.xai_ld;
    a.s_img_lo = L.xai_lo;
    attention_fwd(a, L.s_all + (int64_t)t * B * H, p.str_W, p.str_b, L.att_ws, st);
  }
  {
    Phase ph(st, "k10_dec_fwd_hoisted", 2.0 * BT * L.RO * d.Rd);
    // the readout input's image (ones column at RO for d b_ro), kept for the backward's d W_ro
    x3_split_into(L.ro, L.RO, (int)BT, (int)L.RO, (int)L.RO, L.roi, L.roi_ld, L.roi_ld, BT * L.roi_ld, st);
    gemm_f32x3_ex(false, false, (int)BT, d.Rd, (int)L.RO, nullptr, 0, L.roi, p.ro_W, d.Rd, nullptr, 0.f, L.dpre,
                  d.Rd, p.ro_b, nullptr, 0, L.gws, st, L.roi_ld, BT * L.roi_ld);  // pre-activation (dpre is free until the backward)
    const bool v4 = d.Rd % 4 == 0 && ((reinterpret_cast<uintptr_t>(readout) | reinterpret_cast<uintptr_t>(L.dpre)) & 15) == 0;
    if (v4) f32_relu4_kernel<<<(unsigned)std::min<int64_t>(BT, 148 * 16), 256, 0, st>>>(L.dpre, readout, B, T, d.Rd);
    else f32_relu_kernel<<<std::min<unsigned>(grid_of(BT * d.Rd), 148 * 8), 256, 0, st>>>(L.dpre, readout, B, T, d.Rd);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
}

void decoder_f32_bwd(const DecDims& d, const DecParams& p, const DecGrads& g, const float* enc,
                     const int32_t* src_lens, const int32_t* prev_ids, const float* readout, const float* d_readout,
                     float* d_enc, void* ws, cudaStream_t st) {
  decoder_f32_check(d);
  (void)prev_ids;  // the forward's time-major ids are in the workspace
  const FLay L = flayout(d, ws);
  const int B = d.B, T = d.T, H = d.H, E = d.E, K = d.K, Emb = d.Emb, Rd = d.Rd;
  const int64_t BT = (int64_t)B * T, BTs = (int64_t)B * d.Ts;
  {
    Phase ph(st, "k10_dec_bwd_hoisted", 4.0 * BT * L.RO * Rd);
    const bool v4 = Rd % 4 == 0 &&
                    ((reinterpret_cast<uintptr_t>(readout) | reinterpret_cast<uintptr_t>(d_readout) |
                      reinterpret_cast<uintptr_t>(L.dpre)) & 15) == 0;
    if (v4)
      f32_relu_bwd4_kernel<<<(unsigned)std::min<int64_t>(BT, 148 * 16), 256, 0, st>>>(readout, d_readout, L.dpre, B, T,
                                                                                      Rd);
    else
      f32_relu_bwd_kernel<<<std::min<unsigned>(grid_of(BT * Rd), 148 * 8), 256, 0, st>>>(readout, d_readout, L.dpre,
                                                                                           B, T, Rd);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
    // d readout input = d pre W_ro^T; [d W_ro; d b_ro] = [X | 1]^T d pre
    x3_split_into(L.dpre, Rd, (int)BT, Rd, -1, L.dprei, L.dprei_ld, L.dprei_ld, BT * L.dprei_ld, st);
    gemm_f32x3_ex(false, true, (int)BT, (int)L.RO, Rd, nullptr, 0, L.dprei, p.ro_W, Rd, nullptr, 0.f, L.dro, L.RO,
                  nullptr, nullptr, 0, L.gws, st, L.dprei_ld, BT * L.dprei_ld);
    gemm_f32x3_ex(true, false, (int)L.RO, Rd, (int)BT, nullptr, 0, L.roi, nullptr, 0, L.dprei, 0.f, g.ro_W, Rd,
                  nullptr, g.ro_b, Rd, L.gws, st, L.roi_ld, BT * L.roi_ld, L.dprei_ld, BT * L.dprei_ld);
  }
  X3Parts dxp{nullptr, 0, 0, 0};  // d [att ‖ s]_t from step t + 1 (partials)
  for (int t = T - 1; t >= 0; --t) {
    const int cur = t & 1, nxt = cur ^ 1;  // ping-pong: d c / d accum of step t in [cur], of t - 1 -> [nxt]
    {
      Phase q(st, "k10_cell_bwd", 0.0, 4.0 * B * (E + H) * 3);
      GradIn gi{B, H, E, t, t + 1 < T, L.dro, L.RO, Emb, dxp, L.datt_all + (int64_t)t * B * E, L.ds};
      const bool v4 = E % 4 == 0 && H % 4 == 0 && L.RO % 4 == 0 && (H + Emb) % 4 == 0 &&
                      (dxp.n == 0 || (dxp.ld % 4 == 0 && dxp.stride % 4 == 0 &&
                                      (reinterpret_cast<uintptr_t>(dxp.p) & 15) == 0));
      if (v4) f32_grad_in4_kernel<<<grid_of((int64_t)B * (E + H) / 4), 256, 0, st>>>(gi);
      else f32_grad_in_kernel<<<grid_of((int64_t)B * (E + H)), 256, 0, st>>>(gi);
      SL_CUDA_TRY(cudaGetLastError());
      count_launch();
    }
    AttnArgs a = att_args(d, L, p, enc, src_lens, t);
    a.a_saved = L.a_all + (int64_t)t * B * d.Ts;
    a.d_att = L.datt_all + (int64_t)t * B * E;
    a.d_accum_out = t + 1 < T ? L.dacc + (int64_t)cur * B * d.Ts : nullptr;
    a.d_accum = L.dacc + (int64_t)nxt * B * d.Ts;
    a.d_enc_ctx = L.dctx;
    a.d_enc = d_enc;
    a.d_W_fb = g.fb_W;
    a.d_b_fb = g.fb_b;
    a.d_v = g.e_W;
    a.d_b_v = g.e_b;
    a.accumulate = 1;  // d s accumulates onto the readout / next-step part; d accum_{t-1} zeroed per step
    a.s_tr_in = L.str_all + (int64_t)t * B * K;
    a.defer = 1;  // d enc, d enc_ctx, d W_fb, d b_fb, d v, d b_v, d W_s, d b_s: after the loop
    a.d_s_tr_out = L.ds_all + (int64_t)t * B * K;
    a.de_out = L.de_all + (int64_t)t * B * d.Ts;
    a.d_accum_fresh = 1;  // the tanh pass writes every position of d accum_{t-1} (no memset)
    X3Parts dsp{nullptr, 0, 0, 0};
    a.ds_parts_out = &dsp;
    attention_bwd(a, L.s_all + (int64_t)t * B * H, p.str_W, p.str_b, L.ds, nullptr, nullptr, L.att_ws, st);
    {
      Phase q(st, "k10_cell_bwd", 0.0, 4.0 * B * H * 12);
      CellBF cb{B, H, t, L.ds, L.gates, L.c_all, t + 1 < T ? L.dc + (int64_t)cur * B * H : nullptr, dsp, L.dzi,
                L.dzi_ld, BT * L.dzi_ld, L.dc + (int64_t)nxt * B * H};
      const bool v4 = H % 4 == 0 && L.dzi_ld % 4 == 0 && (BT * L.dzi_ld) % 4 == 0 &&
                      (dsp.n == 0 || (dsp.ld % 4 == 0 && dsp.stride % 4 == 0 &&
                                      (reinterpret_cast<uintptr_t>(dsp.p) & 15) == 0));
      if (v4) f32_cell_bwd4_kernel<<<grid_of((int64_t)B * H / 4), 256, 0, st>>>(cb);
      else f32_cell_bwd_kernel<<<grid_of((int64_t)B * H), 256, 0, st>>>(cb);
      SL_CUDA_TRY(cudaGetLastError());
      count_launch();
    }
    if (t > 0) {  // d [att ‖ s]_{t-1} = DZ_t [W_att; R]^T
      Phase q(st, "k10_g1_gemm", 2.0 * B * 4.0 * H * (E + H));
      dxp = gemm_f32x3_parts(false, true, B, (int)L.XA, 4 * H, nullptr, 0, L.dzi + (int64_t)t * B * L.dzi_ld,
                             nullptr, 0, L.wd2_b, L.gws, st, L.dzi_ld, BT * L.dzi_ld);
    }
  }
  {
    Phase ph(st, "k10_dec_bwd_hoisted",
             2.0 * BT * 4 * H * (E + H + 2.0 * Emb) + 4.0 * BTs * E * K);
    // the cell's weight gradients over all B*T rows: [W_att; R] from [att ‖ s]_{t-1} (block t of xa)
    // (A = the [att ‖ s] image; the 64-wide blocks of d R's column window run 16 columns
    // into the next row, which block T of the image keeps in bounds)
    gemm_f32x3_ex(true, false, E, 4 * H, (int)BT, nullptr, 0, L.xai, nullptr, 0, L.dzi, 0.f,
                  g.s_W + (int64_t)Emb * 4 * H, 4 * H, nullptr, nullptr, 0, L.gws, st, L.xai_ld, L.xai_lo);
    gemm_f32x3_ex(true, false, H, 4 * H, (int)BT, nullptr, 0, L.xai + E, nullptr, 0, L.dzi, 0.f, g.s_R, 4 * H,
                  nullptr, nullptr, 0, L.gws, st, L.xai_ld, L.xai_lo);
    // [W_trg; b] from [trg_{t-1} | 1]
    gemm_f32x3_ex(true, false, Emb, 4 * H, (int)BT, L.ro + H, L.RO, nullptr, nullptr, 0, L.dzi, 0.f, g.s_W, 4 * H,
                  nullptr, g.s_b, 4 * H, L.gws, st);
    // d trg_{t-1} = DZ W_trg^T + the readout's trg columns -> the trg table
    // (in place: the readout's trg columns of d ro accumulate DZ W_trg^T; d ro has no later reader)
    gemm_f32x3_ex(false, true, (int)BT, Emb, 4 * H, nullptr, 0, L.dzi, p.s_W, 4 * H, nullptr, 1.f, L.dro + H, L.RO,
                  nullptr, nullptr, 0, L.gws, st, L.dzi_ld, BT * L.dzi_ld);
    embedding_bwd(BT, L.ids_tm, d.Vt, Emb, L.dro + H, L.RO, g.trg_W, false, L.emb_ws, st);
    // the attention's accumulations over t (deferred out of the loop)
    {
      Phase q(st, "k10_dec_bwd_deferred", 2.0 * T * BTs * (E + 6.0 * K));
      const dim3 ge((unsigned)ceil_div(E, 512), (unsigned)ceil_div(d.Ts, kEncPos), (unsigned)B);
      f32_enc_grad_kernel<<<ge, 128, (size_t)T * kEncPos * 4, st>>>(B, d.Ts, T, E, L.a_all, L.datt_all, d_enc);
      SL_CUDA_TRY(cudaGetLastError());
      const int nsc = (int)ceil_div(d.Ts, kCtxPos);
      const dim3 gc((unsigned)ceil_div(K, 128), (unsigned)nsc, (unsigned)B);
      f32_ctx_grad_kernel<<<gc, 128, (size_t)2 * T * kCtxPos * 4, st>>>(B, d.Ts, T, K, L.enc_ctx, L.acc_all, L.de_all,
                                                                          L.str_all, p.fb_W, p.fb_b, p.e_W, L.dctx,
                                                                          L.apart);
      SL_CUDA_TRY(cudaGetLastError());
      f32_ctx_reduce1_kernel<<<dim3((unsigned)ceil_div(K, 128), kRedSlices), 128, 0, st>>>(
          B * nsc, K, L.apart, L.de_all, (int64_t)T * B * d.Ts, L.apart2);
      SL_CUDA_TRY(cudaGetLastError());
      f32_ctx_reduce2_kernel<<<(unsigned)ceil_div(K, 128), 128, 0, st>>>(K, L.apart2, g.fb_W, g.fb_b, g.e_W, g.e_b);
      SL_CUDA_TRY(cudaGetLastError());
      count_launch(4);
      // s_tr = s W_s + b_s: [d W_s; d b_s] = [S | 1]^T d S_tr over all T*B rows
      gemm_f32x3(true, false, H, K, (int)BT, L.s_all, H, L.ds_all, K, 0.f, g.str_W, K, nullptr, g.str_b, K, L.gws,
                 st);
    }
    // enc_ctx = enc W_ctx + b_ctx: [d W_ctx; d b_ctx] = [enc | 1]^T d enc_ctx; d enc += d enc_ctx W_ctx^T
    x3_split_into(L.dctx, K, (int)BTs, K, -1, L.dctxi, L.dctxi_ld, L.dctxi_ld, BTs * L.dctxi_ld, st);
    gemm_f32x3_ex(true, false, E, K, (int)BTs, nullptr, 0, L.enci, nullptr, 0, L.dctxi, 0.f, g.ctx_W, K, nullptr,
                  g.ctx_b, K, L.gws, st, L.enci_ld, BTs * L.enci_ld, L.dctxi_ld, BTs * L.dctxi_ld);
    gemm_f32x3_ex(false, true, (int)BTs, E, K, nullptr, 0, L.dctxi, p.ctx_W, K, nullptr, 1.f, d_enc, E, nullptr,
                  nullptr, 0, L.gws, st, L.dctxi_ld, BTs * L.dctxi_ld);
  }
}

}  // namespace sl
