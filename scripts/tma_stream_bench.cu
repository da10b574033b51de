// Microbenchmark: per-SM TMA streaming rate for the recurrence's access pattern.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1805_05225_b200/csrc
//      tma_stream_bench.cu -o /tmp/tsb -lcuda
// Each CTA streams `reps` passes over a [rows x K] bf16 matrix in boxes of
// {64, box_rows} through a `stages`-deep mbarrier ring (a consumer thread
// frees slots as soon as they land).  Modes: shared (all CTAs read the same
// matrix) or private (CTA i reads its own copy).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

#include "tc.cuh"

using namespace sl;

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int rows,
                                                       int K, int box_rows, int stages, int reps,
                                                       int private_mode, unsigned long long* out,
                                                       int kb) {
  extern __shared__ uint8_t raw[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const uint32_t base = (tc::smem_u32(raw) + 1023u) & ~1023u;
  uint8_t* smem = raw + (base - tc::smem_u32(raw));
  const uint32_t box_bytes = 64 * box_rows * 2 * kb;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::fence_barrier_init();
  }
  __syncthreads();
  const int nk = K / 64 / kb, nr = rows / box_rows;
  const int total = reps * nk * nr;
  const int z = private_mode ? blockIdx.x : 0;
  unsigned long long t0 = 0;
  if (threadIdx.x == 0) {  // producer
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int st = 0;
    uint32_t ph = 0;
    for (int i = 0; i < total; ++i) {
      tc::mbar_wait(&empty[st], ph ^ 1);
      tc::mbar_arrive_expect_tx(&full[st], box_bytes);
      const int kc = (i + blockIdx.x) % nk, rr = (i / nk) % nr;
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(tc::smem_u32(smem + st * box_bytes)),
          "l"(&tm), "r"(0), "r"(rr * box_rows), "r"(kc * kb), "r"(z), "r"(tc::smem_u32(&full[st]))
          : "memory");
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {  // consumer
    int st = 0;
    uint32_t ph = 0;
    for (int i = 0; i < total; ++i) {
      tc::mbar_wait(&full[st], ph);
      tc::mbar_arrive(&empty[st]);
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[blockIdx.x * 2 + 1] = t1;
  }
  if (threadIdx.x == 0) out[blockIdx.x * 2] = t0;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int rows = 256, K = 1024, reps = 40;
  const int max_ctas = 148;
  __nv_bfloat16* buf;
  cudaMalloc(&buf, (size_t)rows * K * 2 * max_ctas);
  cudaMemset(buf, 0, (size_t)rows * K * 2 * max_ctas);
  unsigned long long* out;
  cudaMalloc(&out, 2 * max_ctas * 8);
  for (int private_mode = 0; private_mode < 1; ++private_mode)
    for (int box_rows : {128, 256})
      for (int kb : {1, 2, 4})
        for (int stages : {3, 6})
          for (int ctas : {64, 126, 148}) {
            CUtensorMap tm;
            // 4-D view of row-major [z][rows][K]: {k_in 64, rows, k_chunk, z}
            cuuint64_t dims[4] = {64, (cuuint64_t)rows, (cuuint64_t)K / 64, (cuuint64_t)max_ctas};
            cuuint64_t strides[3] = {(cuuint64_t)K * 2, 128, (cuuint64_t)K * 2 * rows};
            cuuint32_t box[4] = {64, (cuuint32_t)box_rows, (cuuint32_t)kb, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) { printf("encode failed kb=%d rows=%d (%d)\n", kb, box_rows, (int)cr); continue; }
            const int smem = stages * 64 * box_rows * 2 * kb + 1024;
            if (smem > 227 * 1024) continue;
            cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            stream_kernel<<<ctas, 64, smem>>>(tm, rows, K, box_rows, stages, reps, private_mode, out, kb);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
              printf("error %s\n", cudaGetErrorString(e));
              return 1;
            }
            std::vector<unsigned long long> h(2 * ctas);
            cudaMemcpy(h.data(), out, 2 * ctas * 8, cudaMemcpyDeviceToHost);
            double worst = 0;
            for (int i = 0; i < ctas; ++i) worst = std::max(worst, (double)(h[2 * i + 1] - h[2 * i]));
            const double bytes = (double)reps * rows * K * 2;
            printf("shared box_rows=%3d kb=%d (%3d KB) stages=%d ctas=%3d : per-SM %.1f GB/s, aggregate %.2f TB/s\n",
                   box_rows, kb, 128 * box_rows * kb / 1024, stages, ctas, bytes / worst, bytes * ctas / worst / 1e3);
          }
  return 0;
}
