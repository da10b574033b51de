// Can enc_ctx (61 MB) stay in the 126 MB L2 across the decoder's steps while
// enc (123 MB) streams through it, with per-load eviction hints instead of a
// persisting carve-out?  Per "step": read A (61 MB) then B (123 MB); A with
// L2::evict_last, B with L2::evict_first — against plain loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 l2_hint_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int HINT>  // 0 plain, 1 evict_last, 2 evict_first
__global__ void rd(const float* __restrict__ x, int64_t n8, float* out) {
  float acc = 0.f;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i < n8; i += st) {
    float f[8];
    const float* p = x + i * 8;
    if (HINT == 1)
      asm volatile("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]), "=f"(f[6]), "=f"(f[7]) : "l"(p));
    else if (HINT == 2)
      asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]), "=f"(f[6]), "=f"(f[7]) : "l"(p));
    else
      asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]), "=f"(f[6]), "=f"(f[7]) : "l"(p));
    acc += f[0] + f[7];
  }
  if (acc == 1.2345f) out[0] = acc;
}
// normal-priority writes of W bytes (the per-step GEMM partials / states)
__global__ void wr(float4* y, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = make_float4(1.f, 2.f, 3.f, (float)i);
}

int main() {
  const int64_t nA = 256LL * 60 * 1000, nB = 256LL * 60 * 2000, nW = 32LL << 20;  // floats (W: 128 MB... / 4)
  float *A, *B, *W, *out;
  cudaMalloc(&A, nA * 4);
  cudaMalloc(&B, nB * 4);
  cudaMalloc(&W, nW);
  cudaMalloc(&out, 64);
  cudaMemset(A, 0, nA * 4);
  cudaMemset(B, 0, nB * 4);
  cudaEvent_t ev[4];
  for (auto& e : ev) cudaEventCreate(&e);
  for (int mode = 0; mode < 3; ++mode) {
    for (int wbytes : {0, 16, 32}) {  // extra normal-priority writes per step (MB)
      float ta = 0, tb = 0;
      const int steps = 20;
      for (int s = 0; s < steps + 2; ++s) {
        cudaEventRecord(ev[0]);
        if (mode == 0) rd<0><<<1184, 256>>>(A, nA / 8, out);
        else rd<1><<<1184, 256>>>(A, nA / 8, out);
        cudaEventRecord(ev[1]);
        if (mode == 0) rd<0><<<1184, 256>>>(B, nB / 8, out);
        else if (mode == 1) rd<2><<<1184, 256>>>(B, nB / 8, out);
        else rd<0><<<1184, 256>>>(B, nB / 8, out);
        cudaEventRecord(ev[2]);
        if (wbytes) wr<<<1184, 256>>>(reinterpret_cast<float4*>(W), (int64_t)wbytes * (1 << 20) / 16);
        cudaEventSynchronize(ev[2]);
        float a, b;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        if (s >= 2) ta += a, tb += b;
      }
      printf("mode %s  writes %2d MB/step: A (61 MB) %6.2f us  B (123 MB) %6.2f us  sum %6.2f\n",
             mode == 0 ? "plain               " : mode == 1 ? "A last, B first     " : "A last, B plain     ", wbytes,
             ta / steps * 1e3, tb / steps * 1e3, (ta + tb) / steps * 1e3);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
