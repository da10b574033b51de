// L2 residency across the decoder loop's access pattern (B200): per "step" read
// enc_ctx (61 MB fp32), then enc (123 MB), then the cell weight image (48 MB) —
// 232 MB per step against the 126 MB L2 — with (0) default loads, (1) enc_ctx
// loaded under an L2 evict_last policy and enc under evict_first, (2) enc_ctx and
// the weight image evict_last, enc evict_first.  Prints the per-kernel times.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2pb l2_policy_bench.cu
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int MODE>  // 0 default, 1 evict_last, 2 evict_first
__global__ void __launch_bounds__(256) readk(const float4* __restrict__ x, int64_t n, float* out) {
  float acc = 0.f;
  uint64_t pol = MODE == 1 ? pol_last() : pol_first();
  const int64_t stride = (int64_t)gridDim.x * 256;
  for (int64_t i0 = blockIdx.x * 256 + threadIdx.x; i0 < n; i0 += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= n) { v[u] = make_float4(0, 0, 0, 0); continue; }
      if (MODE == 0) {
        v[u] = __ldg(x + i);
      } else {
        asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                     : "l"(x + i), "l"(pol));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1.2345f) out[0] = acc;
}

template <int MODE>
void launch(const float* p, size_t bytes, float* out, cudaStream_t s) {
  readk<MODE><<<148 * 8, 256, 0, s>>>(reinterpret_cast<const float4*>(p), (int64_t)(bytes / 16), out);
}

int main() {
  const size_t nctx = 256ull * 60 * 1000 * 4, nenc = 256ull * 60 * 2000 * 4, nw = 3000ull * 4000 * 4;
  float *ctx, *enc, *w, *out;
  cudaMalloc(&ctx, nctx);
  cudaMalloc(&enc, nenc);
  cudaMalloc(&w, nw);
  cudaMalloc(&out, 4);
  cudaMemset(ctx, 0, nctx);
  cudaMemset(enc, 0, nenc);
  cudaMemset(w, 0, nw);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t ev[4];
  for (auto& e : ev) cudaEventCreate(&e);
  int maxp = 0, maxw = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  printf("max persisting L2 %.1f MB, max window %.1f MB\n", maxp / 1e6, maxw / 1e6);
  for (int variant = 0; variant < 5; ++variant) {
    if (variant == 3) {  // access policy window: enc_ctx persisting (carve-out at its maximum)
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp);
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = ctx;
      v.accessPolicyWindow.num_bytes = std::min<size_t>(nctx, maxw);
      v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)maxp / (float)v.accessPolicyWindow.num_bytes);
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      printf("window %.1f MB hitRatio %.2f: %s\n", v.accessPolicyWindow.num_bytes / 1e6,
             v.accessPolicyWindow.hitRatio,
             cudaGetErrorString(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v)));
    }
    float t[3] = {0, 0, 0};
    const int iters = 20;
    for (int it = 0; it < iters + 3; ++it) {
      cudaEventRecord(ev[0], s);
      if (variant == 0 || variant == 3) launch<0>(ctx, nctx, out, s);
      else launch<1>(ctx, nctx, out, s);
      cudaEventRecord(ev[1], s);
      if (variant == 0 || variant == 3) launch<0>(enc, nenc, out, s);
      else launch<2>(enc, nenc, out, s);
      cudaEventRecord(ev[2], s);
      if (variant == 2 || variant == 4) launch<1>(w, nw, out, s);
      else launch<0>(w, nw, out, s);
      cudaEventRecord(ev[3], s);
      cudaEventSynchronize(ev[3]);
      if (it >= 3)
        for (int k = 0; k < 3; ++k) {
          float ms;
          cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
          t[k] += ms;
        }
    }
    printf("variant %d: enc_ctx %.1f us (%.0f GB/s)  enc %.1f us (%.0f GB/s)  W %.1f us (%.0f GB/s)\n", variant,
           t[0] / iters * 1e3, nctx / (t[0] / iters * 1e-3) / 1e9, t[1] / iters * 1e3,
           nenc / (t[1] / iters * 1e-3) / 1e9, t[2] / iters * 1e3, nw / (t[2] / iters * 1e-3) / 1e9);
  }
  {  // L2-hot baseline: a 40 MB slice of enc_ctx read back to back
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
    const size_t n40 = 40ull << 20;
    float tt = 0;
    for (int it = 0; it < 23; ++it) {
      cudaEventRecord(ev[0], s);
      launch<0>(ctx, n40, out, s);
      cudaEventRecord(ev[1], s);
      cudaEventSynchronize(ev[1]);
      float ms;
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
      if (it >= 3) tt += ms;
    }
    printf("L2-hot 40 MB: %.1f us (%.0f GB/s)\n", tt / 20 * 1e3, n40 / (tt / 20 * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
