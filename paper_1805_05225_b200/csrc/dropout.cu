// The reference's input dropout (Tape::dropout, tape.cpp:540-600, applied by
// eval_layer, compiler.cpp:554-562) on a [B, T, F] value keyed by its own Time
// coordinate: element (b, t, f) survives iff
//   u01(mix64(key, mix64(t + 2, b*F + f))) >= rate,   u01(h) = (splitmix64(h) >> 11) * 2^-53,
// with the counter-based hash of rng.hpp (splitmix64 / mix64), so the mask is a pure
// function of (key, position): bit-identical to the reference, recomputed in the
// backward instead of stored.  key = mix64(key0, batch_counter); the counter may be
// read on the device (e.g. the optimizer's step counter) so a captured CUDA graph
// draws a new mask every replay.
#include <cmath>

#include "dropout.h"
#include "profile.h"

namespace sl {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) {
  return splitmix64(a ^ (splitmix64(b) + 0x9e3779b97f4a7c15ull));
}

// out = in * inv_keep where the element survives, else 0 (the forward on x and the
// adjoint on dy are the same map)
// keep(h): u01(h) >= rate, with u01 = (splitmix64(h) >> 11) * 2^-53 exact in double, is
// the integer test (splitmix64(h) >> 11) >= thr53 for thr53 = ceil(rate * 2^53) (host).
// sidx = splitmix64(idx) does not depend on t: mix64(ct, idx) = splitmix64(ct ^ (sidx + C)).
__device__ __forceinline__ bool keep_s(uint64_t key, uint64_t ct, uint64_t sidx, uint64_t thr53) {
  return (splitmix64(mix64(key, splitmix64(ct ^ (sidx + 0x9e3779b97f4a7c15ull)))) >> 11) >= thr53;
}
__device__ __forceinline__ bool keep(uint64_t key, uint64_t ct, uint64_t idx, uint64_t thr53) {
  return keep_s(key, ct, splitmix64(idx), thr53);
}
__global__ void dropout_kernel(int B, int T, int F, uint64_t thr53, float inv_keep, uint64_t key0,
                               const int32_t* counter, int64_t counter_value, const float* __restrict__ in,
                               float* __restrict__ out) {
  const uint64_t key = mix64(key0, (uint64_t)(counter ? (int64_t)*counter : counter_value));
  const bool v4 = (F % 4) == 0 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (v4 && gridDim.y > 1) {
    // (b = blockIdx.y, four features per thread) over a slice of the steps (blockIdx.z):
    // splitmix64 of each feature's index once per slice — four hashes per element, not five
    const int b = blockIdx.y;
    const int f = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (f >= F) return;
    uint64_t sx[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) sx[u] = splitmix64((uint64_t)b * F + f + u);
    const int tper = (T + (int)gridDim.z - 1) / (int)gridDim.z;  // this block's slice of the steps
    const int t1 = min(T, ((int)blockIdx.z + 1) * tper);
    for (int t = (int)blockIdx.z * tper; t < t1; ++t) {
      const uint64_t ct = (uint64_t)(t + 2);
      const int64_t o = ((int64_t)b * T + t) * F + f;
      const float4 x = *reinterpret_cast<const float4*>(in + o);
      float4 y;
      y.x = keep_s(key, ct, sx[0], thr53) ? x.x * inv_keep : 0.f;
      y.y = keep_s(key, ct, sx[1], thr53) ? x.y * inv_keep : 0.f;
      y.z = keep_s(key, ct, sx[2], thr53) ? x.z * inv_keep : 0.f;
      y.w = keep_s(key, ct, sx[3], thr53) ? x.w * inv_keep : 0.f;
      *reinterpret_cast<float4*>(out + o) = y;
    }
    return;
  }
  // one CTA per (b, t) row: no 64-bit division per element
  for (int64_t r = blockIdx.x; r < (int64_t)B * T; r += gridDim.x) {
    const int b = (int)(r / T), t = (int)(r - (int64_t)b * T);
    const uint64_t ct = (uint64_t)(t + 2), i0 = (uint64_t)b * F;
    const float* src = in + r * F;
    float* dst = out + r * F;
    if (v4) {  // four elements per thread: 16 B loads / stores, four independent hash chains
      for (int f = threadIdx.x * 4; f < F; f += blockDim.x * 4) {
        const float4 x = *reinterpret_cast<const float4*>(src + f);
        float4 y;
        y.x = keep(key, ct, i0 + f, thr53) ? x.x * inv_keep : 0.f;
        y.y = keep(key, ct, i0 + f + 1, thr53) ? x.y * inv_keep : 0.f;
        y.z = keep(key, ct, i0 + f + 2, thr53) ? x.z * inv_keep : 0.f;
        y.w = keep(key, ct, i0 + f + 3, thr53) ? x.w * inv_keep : 0.f;
        *reinterpret_cast<float4*>(dst + f) = y;
      }
    } else {
      for (int f = threadIdx.x; f < F; f += blockDim.x)
        dst[f] = keep(key, ct, i0 + f, thr53) ? src[f] * inv_keep : 0.f;
    }
  }
}

}  // namespace

void dropout_apply(int B, int T, int F, float rate, uint64_t key0, const int32_t* counter, int64_t counter_value,
                   const float* in, float* out, cudaStream_t st) {
  const int64_t n = (int64_t)B * T * F;
  if (n == 0) return;
  const float inv_keep = 1.0f / (1.0f - rate);  // Real(1) / (Real(1) - rate), fp32 like the reference build
  Phase ph(st, "k11_dropout", 0.0, 8.0 * n);
  // u >= rate (doubles) <=> k >= rate * 2^53 for the integer k = u * 2^53 (exact scaling)
  const double r53 = std::ldexp((double)rate, 53);
  const uint64_t thr53 = r53 <= 0.0 ? 0ull : (uint64_t)std::ceil(r53);
  const bool v4 = (F % 4) == 0 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  if (v4 && B <= 65535) {  // per (b, feature group) over all t
    const dim3 grid((unsigned)ceil_div((int64_t)F / 4, 256), (unsigned)B, (unsigned)std::min(T, 8));
    dropout_kernel<<<grid, 256, 0, st>>>(B, T, F, thr53, inv_keep, key0, counter, counter_value, in, out);
  } else {
    const int grid = (int)std::min<int64_t>((int64_t)B * T, 148 * 16);
    dropout_kernel<<<grid, 256, 0, st>>>(B, T, F, thr53, inv_keep, key0, counter, counter_value, in, out);
  }
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace sl
