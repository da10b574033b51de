// The reference's input dropout (Tape::dropout, tape.cpp:540-600, applied by
// eval_layer, compiler.cpp:554-562) on a [B, T, F] value keyed by its own Time
// coordinate: element (b, t, f) survives iff
//   u01(mix64(key, mix64(t + 2, b*F + f))) >= rate,   u01(h) = (splitmix64(h) >> 11) * 2^-53,
// with the counter-based hash of rng.hpp (splitmix64 / mix64), so the mask is a pure
// function of (key, position): bit-identical to the reference, recomputed in the
// backward instead of stored.  key = mix64(key0, batch_counter); the counter may be
// read on the device (e.g. the optimizer's step counter) so a captured CUDA graph
// draws a new mask every replay.
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
__global__ void dropout_kernel(int B, int T, int F, float rate, float inv_keep, uint64_t key0,
                               const int32_t* counter, int64_t counter_value, const float* __restrict__ in,
                               float* __restrict__ out) {
  const uint64_t key = mix64(key0, (uint64_t)(counter ? (int64_t)*counter : counter_value));
  const double thr = (double)rate;
  // one CTA per (b, t) row: no 64-bit division per element
  for (int64_t r = blockIdx.x; r < (int64_t)B * T; r += gridDim.x) {
    const int b = (int)(r / T), t = (int)(r - (int64_t)b * T);
    const uint64_t ct = (uint64_t)(t + 2);
    const float* src = in + r * F;
    float* dst = out + r * F;
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      const uint64_t h = mix64(key, mix64(ct, (uint64_t)b * F + f));
      const double u = (double)(splitmix64(h) >> 11) * 0x1.0p-53;
      dst[f] = u >= thr ? src[f] * inv_keep : 0.f;
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
  const int grid = (int)std::min<int64_t>((int64_t)B * T, 148 * 16);
  dropout_kernel<<<grid, 256, 0, st>>>(B, T, F, rate, inv_keep, key0, counter, counter_value, in, out);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace sl
