// Microbenchmark: tcgen05.mma (kind::f16, SS operands, cta_group::1, M=128)
// throughput per SM vs N, with operands resident in shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1805_05225_b200/csrc
//      scripts/mma_rate_bench.cu -o scripts/mma_rate_bench.bin
#include <cstdio>

#include "tc.cuh"

using namespace sl;

template <int N>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, int chunks, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tmem_sh;
  const uint32_t base = (tc::smem_u32(raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    tc::mbar_init(&done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<256>(&tmem_sh);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_sh;
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc = tc::make_idesc(128, N, 1, false, false);
    const uint32_t a_bytes = 128 * 128, b_bytes = N * 128;  // one 64-wide K chunk each
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int it = 0; it < iters; ++it) {
      for (int c = 0; c < chunks; ++c) {
        const uint32_t sa = base + (c % 4) * a_bytes;
        const uint32_t sb = base + 4 * a_bytes + (c % 4) * b_bytes;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_f16(tmem, tc::make_sdesc(sa + k * 32, 0, 1024), tc::make_sdesc(sb + k * 32, 0, 1024),
                      idesc, (c | k) != 0);
      }
    }
    tc::mma_commit(&done);
    tc::mbar_wait(&done, 0);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

template <int N>
void run(int ctas) {
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  const int smem = 4 * 128 * 128 + 4 * N * 128 + 1024;
  cudaFuncSetAttribute(mma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 200, chunks = 16;
  mma_kernel<N><<<ctas, 128, smem>>>(iters, chunks, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("err %s\n", cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, out, ctas * 8, cudaMemcpyDeviceToHost);
  unsigned long long worst = 0;
  for (int i = 0; i < ctas; ++i) worst = h[i] > worst ? h[i] : worst;
  const double mmas = (double)iters * chunks * 4;
  const double ns = (double)worst / mmas;
  printf("N=%3d ctas=%3d : %.1f ns per MMA (%.0f clk @1.92GHz), %.0f TFLOP/s per SM-equivalent chip %.0f\n", N,
         ctas, ns, ns * 1.92, 2.0 * 128 * N * 16 / ns / 1e3, 2.0 * 128 * N * 16 / ns / 1e3 * 148);
  cudaFree(out);
}

int main() {
  for (int ctas : {1, 128}) {
    run<16>(ctas);
    run<32>(ctas);
    run<64>(ctas);
    run<128>(ctas);
    run<256>(ctas);
  }
  return 0;
}
