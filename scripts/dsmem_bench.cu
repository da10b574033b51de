// Microbenchmark: DSMEM (distributed shared memory) transfer rate within a
// 2-CTA cluster: (a) 256 threads x st.shared::cluster.v4 (16 B per store),
// (b) one thread issuing cp.async.bulk.shared::cluster.shared::cta (bulk copy
// engine) of 16 KB chunks completing on the peer's mbarrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1805_05225_b200/csrc
//      scripts/dsmem_bench.cu -o scripts/dsmem_bench.bin
#include <cstdio>

#include "tc.cuh"

using namespace sl;

__device__ __forceinline__ uint32_t mapa_(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// mode 0: thread stores, mode 1: bulk copies.  Each CTA sends `bytes` to its peer `reps` times.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    dsmem_kernel(int mode, int bytes, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const uint32_t peer = rank ^ 1;
  uint8_t* src = smem;          // [bytes]
  uint8_t* dst = smem + bytes;  // [bytes] receive area
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) reinterpret_cast<float*>(src)[i] = i;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  csync();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const uint32_t rdst = mapa_(tc::smem_u32(dst), peer);
  const uint32_t rbar = mapa_(tc::smem_u32(&bar), peer);
  for (int r = 0; r < reps; ++r) {
    if (mode == 0) {
      for (int off = threadIdx.x * 16; off < bytes; off += blockDim.x * 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + off);
        asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rdst + off), "r"(v.x),
                     "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
      }
      __syncthreads();
      csync();  // all stores of this rep visible at the peer
    } else {
      if (threadIdx.x == 0) {
        tc::mbar_arrive_expect_tx(&bar, bytes);  // my barrier receives the peer's bytes
      }
      csync();  // both barriers armed before any copy lands
      if (threadIdx.x == 0) {
        for (int off = 0; off < bytes; off += 16384) {
          const int n = bytes - off < 16384 ? bytes - off : 16384;
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  rdst + off),
              "r"(tc::smem_u32(src + off)), "r"(n), "r"(rbar)
              : "memory");
        }
        tc::mbar_wait(&bar, r & 1);
      }
      __syncthreads();
    }
  }
  csync();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  for (int mode : {0, 1})
    for (int bytes : {16384, 32768, 65536})
      for (int ctas : {2, 128}) {
        const int smem = 2 * bytes + 1024;
        cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int reps = 200;
        dsmem_kernel<<<ctas, 256, smem>>>(mode, bytes, reps, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("err %s\n", cudaGetErrorString(e));
          return 1;
        }
        unsigned long long h[148];
        cudaMemcpy(h, out, ctas * 8, cudaMemcpyDeviceToHost);
        unsigned long long worst = 0;
        for (int i = 0; i < ctas; ++i) worst = h[i] > worst ? h[i] : worst;
        const double us_per_rep = worst / 1e3 / reps;
        printf("%s bytes=%6d ctas=%3d : %.2f us per transfer, %.1f GB/s per CTA (incl. cluster sync per rep)\n",
               mode ? "bulk  " : "thread", bytes, ctas, us_per_rep, bytes / us_per_rep / 1e3);
      }
  return 0;
}
