// Fused optimizer step for the training loop around the hot path (SURVEY §8
// f3): global-norm gradient clipping followed by Adam, over one flat fp32
// parameter buffer (all layers' W, R, b back to back, as the encoder keeps
// them).  Reference semantics: SPEC.md trainer adam_step (SPEC.md:429-437,
// m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2;  bias-corrected m^, v^;
// theta <- theta - lr m^ / (sqrt(v^) + eps)) with the global-norm clip at 5.0
// applied before Adam.  The reference has no code for this op.
//
// Two HBM-bound passes: (1) sum of squares (a fixed-order, run-to-run
// deterministic reduction) + non-finite detection of the
// (already all-reduced) gradient, (2) the element-wise update, which reads
// the clip scale computed from (1) on the device — no host round trip.
// Bytes per parameter: 4 (pass 1) + 16 read + 12 written (pass 2).
#include <cstddef>

#include "adam.h"
#include "profile.h"

namespace sl {
namespace {

constexpr int kThreads = 512;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double part[kThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x % 32 == 0) part[threadIdx.x / 32] = v;
  __syncthreads();
  v = threadIdx.x < kThreads / 32 ? part[threadIdx.x] : 0.0;
  if (threadIdx.x < 32)
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kThreads) grad_sumsq_kernel(const float* __restrict__ g, int64_t n,
                                                               AdamScratch* sc) {
  float acc = 0.f;
  bool bad = false;
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kThreads) {
    const float4 x = __ldcs(g4 + i);
    acc = fmaf(x.x, x.x, acc);
    acc = fmaf(x.y, x.y, acc);
    acc = fmaf(x.z, x.z, acc);
    acc = fmaf(x.w, x.w, acc);
    bad |= !isfinite(x.x) || !isfinite(x.y) || !isfinite(x.z) || !isfinite(x.w);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    const float x = g[i];
    acc = fmaf(x, x, acc);
    bad |= !isfinite(x);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&sc->nonfinite, 1u);
  const double s = block_sum((double)acc);
  // deterministic total: every block leaves its partial, the last block to finish
  // adds them in block order (the same bits every run, unlike float atomics)
  __shared__ bool last;
  if (threadIdx.x == 0) {
    sc->part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kThreads) t += *((volatile double*)&sc->part[b]);
  t = block_sum(t);
  if (threadIdx.x == 0) {
    sc->sumsq = t;
    sc->ticket = 0;
  }
}

__global__ void __launch_bounds__(kThreads) adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                                                         float* __restrict__ m, float* __restrict__ v, int64_t n,
                                                         const AdamScratch* sc, AdamHyper h) {
  if (sc->nonfinite) return;  // SPEC: a non-finite gradient is an error; parameters stay untouched
  float scale = h.grad_scale;
  if (h.clip_norm > 0.f) {
    const float norm = (float)sqrt(sc->sumsq) * h.grad_scale;
    if (norm > h.clip_norm) scale *= h.clip_norm / norm;
  }
  const float b1 = h.beta1, b2 = h.beta2, c1 = 1.f - h.beta1, c2 = 1.f - h.beta2;
  // the step number lives on the device so a captured CUDA graph replays real steps
  const int t = h.step > 0 ? h.step : sc->t + 1;
  const float inv_bc1 = (float)(1.0 / (1.0 - pow((double)h.beta1, (double)t)));
  const float inv_bc2 = (float)(1.0 / (1.0 - pow((double)h.beta2, (double)t)));
  const float lr = h.lr, eps = h.eps;
  auto upd = [&](float& pp, float gg, float& mm, float& vv) {
    gg *= scale;
    mm = fmaf(b1, mm, c1 * gg);
    vv = fmaf(b2, vv, c2 * gg * gg);
    pp -= lr * (mm * inv_bc1) / (sqrtf(vv * inv_bc2) + eps);
  };
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kThreads) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    const float4 gg = __ldcs(reinterpret_cast<const float4*>(g) + i);
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    upd(pp.x, gg.x, mm.x, vv.x);
    upd(pp.y, gg.y, mm.y, vv.y);
    upd(pp.z, gg.z, mm.z, vv.z);
    upd(pp.w, gg.w, mm.w, vv.w);
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    upd(p[i], g[i], m[i], v[i]);
}

// after the update (stream order): report, and advance the device step counter
__global__ void adam_report_kernel(AdamScratch* sc, int32_t step, float grad_scale, float* norm_out,
                                   int32_t* bad_out) {
  if (norm_out) *norm_out = (float)sqrt(sc->sumsq) * grad_scale;
  if (bad_out) *bad_out = (int32_t)sc->nonfinite;
  if (!sc->nonfinite) sc->t = step > 0 ? step : sc->t + 1;
}

int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

void adam_step(int64_t n, float* params, const float* grads, float* m, float* v, const AdamHyper& h,
               AdamScratch* scratch, float* norm_out, int32_t* nonfinite_out, cudaStream_t stream) {
  SL_REQUIRE(n >= 0 && params && grads && m && v && scratch, SL_ERR_INVALID_ARGUMENT,
             "adam_step: null buffer");
  SL_REQUIRE(((uintptr_t)params | (uintptr_t)grads | (uintptr_t)m | (uintptr_t)v) % 16 == 0,
             SL_ERR_INVALID_ARGUMENT, "adam_step: buffers need 16 B alignment");
  SL_CUDA_TRY(cudaMemsetAsync(scratch, 0, offsetof(AdamScratch, t), stream));  // keep the step counter
  const int64_t n4 = (n + 3) / 4;
  const int grid = (int)std::min<int64_t>(std::min<int64_t>(std::max<int64_t>(1, (n4 + kThreads - 1) / kThreads),
                                                             4LL * sms()),
                                          kAdamMaxBlocks);
  {
    Phase ph(stream, "k6_grad_norm", 0.0, 4.0 * n);
    grad_sumsq_kernel<<<grid, kThreads, 0, stream>>>(grads, n, scratch);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
  {
    Phase ph(stream, "k6_adam", 0.0, 28.0 * n);
    adam_kernel<<<grid, kThreads, 0, stream>>>(params, grads, m, v, n, scratch, h);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
  adam_report_kernel<<<1, 1, 0, stream>>>(scratch, h.step, h.grad_scale, norm_out, nonfinite_out);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace sl
