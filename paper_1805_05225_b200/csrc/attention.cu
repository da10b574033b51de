// The decoder's MLP attention step, forward and backward, as
// the reference's Listing-1 subnet wires it (models.cpp:107-154, evaluated by
// compiler.cpp:616-639):
//   s_tr  = s W_s + b_s                                  [B, K]
//   e     = tanh(enc_ctx + accum W_fb + b_fb + s_tr) v + b_v   [B, Ts]
//   a     = softmax over the valid source positions       (tape.cpp:926-985)
//   accum'= accum + a
//   att   = sum_j a_j enc_j                               (tape.cpp:987-1072)
// One CTA per batch row streams its [Ts, K] energy inputs and [Ts, E] encoder
// states once per step (both L2-resident across the decoder's steps at the
// config-4 shape), with the tanh / softmax / weighted sum fused; the small
// projections (s_tr and its gradients) are fp32 GEMMs.  fp32 throughout: the
// step is bandwidth-bound, not tensor-bound.
#include "attention.h"
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

// dynamic smem: c[K] (= b_fb + s_tr[b]), wfb[K], v[K], e[Ts] (+ bwd: 4 [K] accumulators)
__global__ void __launch_bounds__(kThreads) attn_fwd_kernel(AttnArgs p) {
  extern __shared__ float sm[];
  const int b = blockIdx.x, K = p.K, Ts = p.Ts, E = p.E;
  float* c = sm;
  float* wfb = c + K;
  float* v = wfb + K;
  float* e = v + K;
  for (int k = threadIdx.x; k < K; k += kThreads) {
    c[k] = p.b_fb[k] + p.s_tr[(size_t)b * K + k];
    wfb[k] = p.W_fb[k];
    v[k] = p.v[k];
  }
  __syncthreads();
  const int len = min(max(p.lens[b], 0), Ts);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float bv = *p.b_v;
  for (int j = warp; j < len; j += kWarps) {  // energies e_j (tape.cpp ops: add, tanh, matmul v)
    const float* ctx = p.enc_ctx + ((size_t)b * Ts + j) * K;
    const float acc_j = p.accum[(size_t)b * Ts + j];
    float s = 0.f;
    for (int k = lane; k < K; k += 32) s += v[k] * tanhf(ctx[k] + acc_j * wfb[k] + c[k]);
    s = warp_sum(s);
    if (lane == 0) e[j] = s + bv;
  }
  __syncthreads();
  if (warp == 0) {  // masked softmax over the source positions (tape.cpp:952-960)
    float m = -INFINITY;
    for (int j = lane; j < len; j += 32) m = fmaxf(m, e[j]);
    m = warp_max(m);
    float z = 0.f;
    for (int j = lane; j < len; j += 32) z += expf(e[j] - m);
    z = warp_sum(z);
    for (int j = lane; j < Ts; j += 32) {
      const float a = j < len ? expf(e[j] - m) / z : 0.f;
      e[j] = a;
      p.a[(size_t)b * Ts + j] = a;
      p.accum_out[(size_t)b * Ts + j] = p.accum[(size_t)b * Ts + j] + a;
    }
  }
  __syncthreads();
  // context att[b] = sum_j a_j enc[b, j] (tape.cpp:1005-1014)
  for (int x = threadIdx.x; x < E; x += kThreads) {
    float s = 0.f;
    for (int j = 0; j < len; ++j) s += e[j] * p.enc[((size_t)b * Ts + j) * E + x];
    p.att[(size_t)b * E + x] = s;
  }
}

__global__ void __launch_bounds__(kThreads) attn_bwd_kernel(AttnArgs p) {
  extern __shared__ float sm[];
  const int b = blockIdx.x, K = p.K, Ts = p.Ts, E = p.E;
  float* c = sm;
  float* wfb = c + K;
  float* v = wfb + K;
  float* ds = v + K;    // d s_tr[b]
  float* dwf = ds + K;  // d W_fb partial
  float* dbf = dwf + K; // d b_fb partial
  float* dv = dbf + K;  // d v partial
  float* de = dv + K;   // d_a -> d_e [Ts]
  float* aa = de + Ts;  // a [Ts]
  for (int k = threadIdx.x; k < K; k += kThreads) {
    c[k] = p.b_fb[k] + p.s_tr[(size_t)b * K + k];
    wfb[k] = p.W_fb[k];
    v[k] = p.v[k];
    ds[k] = dwf[k] = dbf[k] = dv[k] = 0.f;
  }
  const int len = min(max(p.lens[b], 0), Ts);
  for (int j = threadIdx.x; j < Ts; j += kThreads) aa[j] = p.a_saved[(size_t)b * Ts + j];
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float* dattb = p.d_att + (size_t)b * E;
  // d_a_j = <d_att, enc_j> + d_accum'_j (masked, tape.cpp:1031-1041); d enc_j = a_j d_att
  for (int j = warp; j < Ts; j += kWarps) {
    const float* encj = p.enc + ((size_t)b * Ts + j) * E;
    float* genc = p.d_enc + ((size_t)b * Ts + j) * E;
    const float aj = aa[j];
    float s = 0.f;
    for (int x = lane; x < E; x += 32) {
      const float g = dattb[x];
      s += g * encj[x];
      genc[x] = (p.accumulate ? genc[x] : 0.f) + aj * g;
    }
    s = warp_sum(s);
    if (lane == 0) de[j] = j < len ? s + (p.d_accum_out ? p.d_accum_out[(size_t)b * Ts + j] : 0.f) : 0.f;
  }
  __syncthreads();
  if (warp == 0) {  // softmax adjoint (tape.cpp:966-978)
    float dot = 0.f;
    for (int j = lane; j < len; j += 32) dot += de[j] * aa[j];
    dot = warp_sum(dot);
    for (int j = lane; j < Ts; j += 32) de[j] = j < len ? aa[j] * (de[j] - dot) : 0.f;
  }
  __syncthreads();
  // through tanh and the adds: d e_in[j, k] = d_e_j v_k (1 - u^2)
  float dbv = 0.f;
  for (int j = warp; j < Ts; j += kWarps) {
    const float dej = de[j];
    const float* ctx = p.enc_ctx + ((size_t)b * Ts + j) * K;
    float* gctx = p.d_enc_ctx + ((size_t)b * Ts + j) * K;
    const float acc_j = p.accum[(size_t)b * Ts + j];
    float dacc = 0.f;
    for (int k = lane; k < K; k += 32) {
      float g = 0.f;
      if (j < len) {
        const float u = tanhf(ctx[k] + acc_j * wfb[k] + c[k]);
        g = dej * v[k] * (1.f - u * u);
        atomicAdd(&dv[k], u * dej);
        atomicAdd(&ds[k], g);
        atomicAdd(&dwf[k], acc_j * g);
        atomicAdd(&dbf[k], g);
        dacc += g * wfb[k];
      }
      gctx[k] = (p.accumulate ? gctx[k] : 0.f) + g;
    }
    dacc = warp_sum(dacc);
    if (lane == 0) {
      const float up = (j < len && p.d_accum_out) ? p.d_accum_out[(size_t)b * Ts + j] : 0.f;
      float* ga = p.d_accum + (size_t)b * Ts + j;
      *ga = (p.accumulate ? *ga : 0.f) + up + dacc;
      dbv += dej;
    }
  }
  if (lane == 0 && dbv != 0.f) atomicAdd(p.d_b_v, dbv);
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += kThreads) {
    p.d_s_tr[(size_t)b * K + k] = ds[k];
    atomicAdd(&p.d_W_fb[k], dwf[k]);
    atomicAdd(&p.d_b_fb[k], dbf[k]);
    atomicAdd(&p.d_v[k], dv[k]);
  }
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

size_t attention_workspace_bytes(int B, int K) { return (size_t)2 * B * K * sizeof(float) + 256; }

static size_t fwd_smem(const AttnArgs& p) { return (size_t)(3 * p.K + p.Ts) * sizeof(float); }
static size_t bwd_smem(const AttnArgs& p) { return (size_t)(7 * p.K + 2 * p.Ts) * sizeof(float); }

void attention_fwd(AttnArgs p, const float* s, const float* W_s, const float* b_s, void* ws, cudaStream_t st) {
  p.s_tr = static_cast<float*>(ws);
  gemm_f32(false, false, p.B, p.K, p.H, 1.f, s, p.H, W_s, p.K, 0.f, p.s_tr, p.K, b_s, st);  // s_tr = s W_s + b_s
  const size_t smem = fwd_smem(p);
  SL_REQUIRE(smem <= 227 * 1024, SL_ERR_UNSUPPORTED, "attention: key_dim / src_time too large");
  SL_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  Phase ph(st, "k8_attention_fwd", 0.0, 4.0 * p.B * p.Ts * (double)(p.K + p.E));
  attn_fwd_kernel<<<p.B, kThreads, smem, st>>>(p);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void attention_bwd(AttnArgs p, const float* s, const float* W_s, const float* b_s, float* d_s, float* d_W_s,
                   float* d_b_s, void* ws, cudaStream_t st) {
  p.s_tr = static_cast<float*>(ws);
  p.d_s_tr = p.s_tr + (size_t)p.B * p.K;
  gemm_f32(false, false, p.B, p.K, p.H, 1.f, s, p.H, W_s, p.K, 0.f, p.s_tr, p.K, b_s, st);  // recompute s_tr
  if (!p.accumulate) {
    SL_CUDA_TRY(cudaMemsetAsync(p.d_W_fb, 0, sizeof(float) * p.K, st));
    SL_CUDA_TRY(cudaMemsetAsync(p.d_b_fb, 0, sizeof(float) * p.K, st));
    SL_CUDA_TRY(cudaMemsetAsync(p.d_v, 0, sizeof(float) * p.K, st));
    SL_CUDA_TRY(cudaMemsetAsync(p.d_b_v, 0, sizeof(float), st));
    if (d_b_s) SL_CUDA_TRY(cudaMemsetAsync(d_b_s, 0, sizeof(float) * p.K, st));
  }
  const size_t smem = bwd_smem(p);
  SL_REQUIRE(smem <= 227 * 1024, SL_ERR_UNSUPPORTED, "attention: key_dim / src_time too large");
  SL_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  {
    Phase ph(st, "k8_attention_bwd", 0.0, 4.0 * p.B * p.Ts * (double)(2 * p.K + 2 * p.E));
    attn_bwd_kernel<<<p.B, kThreads, smem, st>>>(p);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
  const float beta = p.accumulate ? 1.f : 0.f;
  if (d_s)  // d s = d s_tr W_s^T
    gemm_f32(false, true, p.B, p.H, p.K, 1.f, p.d_s_tr, p.K, W_s, p.K, beta, d_s, p.H, nullptr, st);
  if (d_W_s)  // d W_s = s^T d s_tr
    gemm_f32(true, false, p.H, p.K, p.B, 1.f, s, p.H, p.d_s_tr, p.K, beta, d_W_s, p.K, nullptr, st);
  if (d_b_s) {
    colsum_kernel<<<(unsigned)ceil_div(p.K, 256), 256, 0, st>>>(p.d_s_tr, p.B, p.K, d_b_s);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
}

}  // namespace sl
