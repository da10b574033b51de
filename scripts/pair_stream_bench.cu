// Microbenchmark: the forward recurrence's h stream in isolation.
// 128 CTAs in clusters of 2 each stream 256 KB per "step" (8 boxes of
// 128 rows x 128 K bf16 = 32 KB) through a 3-slot ring, 200 steps.
// Variants (argv): slot release by the consumer thread with a plain mbarrier
// arrive vs by tcgen05.commit (how the MMA issuer frees a slot); and solo
// (each CTA's TMA completes on its own barrier) vs pair (.cta_group::2 TMA
// completing on the leader's barrier, release multicast to both CTAs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1805_05225_b200/csrc
//      scripts/pair_stream_bench.cu -o scripts/pair_stream_bench.bin -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <algorithm>
#include <vector>

#include "rec_tc_common.cuh"

using namespace sl;
using namespace sl::rtc;

constexpr int kSlots = 3;
__device__ __forceinline__ int kg_of(int s, int g) { return (g + (int)blockIdx.x / 2) % 8; }
constexpr uint32_t kBox = 128 * 128 * 2;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
    stream_kernel(const __grid_constant__ CUtensorMap tm, int steps, int pair_mode, int commit_release,
                  int do_mma, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  __shared__ __align__(8) uint64_t full[kSlots], empty[kSlots];
  __shared__ uint32_t tmem_sh;
  const uint32_t base = (tc::smem_u32(raw) + 1023u) & ~1023u;
  uint8_t* smem = raw + (base - tc::smem_u32(raw));
  const uint32_t r = cluster_rank();
  const bool leader = r == 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<128>(&tmem_sh);
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();
  tc::fence_after_sync();
  unsigned long long t0 = gtimer();
  if (warp == 0 && lane == 0) {  // producer
    int st = 0;
    uint32_t ph = 0;
    for (int s = 0; s < steps; ++s)
      for (int g = 0; g < 8; ++g) {
        tc::mbar_wait(&empty[st], ph ^ 1);
        const int kg = (g + blockIdx.x / 2) % 8;
        if (pair_mode) {
          if (leader) tc::mbar_arrive_expect_tx(&full[st], 2 * kBox);
          tma_load_4d_pair(smem + st * kBox, &tm, mapa(tc::smem_u32(&full[st]), 0), 0, r * 128, kg * 2, 0);
        } else {
          tc::mbar_arrive_expect_tx(&full[st], kBox);
          tma_load_4d(smem + st * kBox, &tm, &full[st], 0, r * 128, kg * 2, 0);
        }
        if (++st == kSlots) {
          st = 0;
          ph ^= 1;
        }
      }
  } else if (warp == 1 && lane == 0 && (leader || !pair_mode)) {  // consumer
    int st = 0;
    uint32_t ph = 0;
    for (int s = 0; s < steps; ++s)
      for (int g = 0; g < 8; ++g) {
        tc::mbar_wait(&full[st], ph);
        if (do_mma) {  // the recurrence's per-slot work: 8 x (M256 N128 K16), B = a resident 128 KB slice
          tc::fence_after_sync();
          constexpr uint32_t idesc = tc::make_idesc(256, 128, 1, false, false);
          const uint32_t rbase = base + kSlots * kBox;
          for (int j = 0; j < 2; ++j)
            for (int k = 0; k < 4; ++k)
              mma_f16_pair(tmem_sh, tc::make_sdesc(base + st * kBox + j * 16384 + k * 32, 0, 1024),
                           tc::make_sdesc(rbase + (uint32_t)(kg_of(s, g) * 2 + j) * 8192 + k * 32, 0, 1024), idesc,
                           (g | j | k) != 0);
        }
        if (commit_release) {
          if (pair_mode) mma_commit_pair(&empty[st]);
          else tc::mma_commit(&empty[st]);
        } else {
          tc::mbar_arrive(&empty[st]);
          if (pair_mode) mbar_arrive_remote(mapa(tc::smem_u32(&empty[st]), 1), 1);
        }
        if (++st == kSlots) {
          st = 0;
          ph ^= 1;
        }
      }
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out[blockIdx.x] = ((gtimer() - t0) << 8) | smid;  // time << 8 | SM id
  }
  if (warp == 1) tmem_dealloc_pair<128>(tmem_sh);
}

int main() {
  const int rows = 256, K = 1024, steps = 200, ctas = 128;
  __nv_bfloat16* buf;
  cudaMalloc(&buf, (size_t)rows * K * 2);
  cudaMemset(buf, 0, (size_t)rows * K * 2);
  unsigned long long* out;
  cudaMalloc(&out, ctas * 8);
  cuuint64_t dims[4] = {64, (cuuint64_t)rows, (cuuint64_t)K / 64, 1};
  cuuint64_t strides[3] = {(cuuint64_t)K * 2, 128, (cuuint64_t)K * 2 * rows};
  cuuint32_t box[4] = {64, 128, 2, 1};
  const CUtensorMap tm = tmap(buf, 4, dims, strides, box);
  const int smem = kSlots * kBox + 128 * 1024 + 1024;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int variant = 0; variant < 5; ++variant) {
      const int pair_mode = variant >= 2, commit = variant != 2, do_mma = variant >= 3;
      if (variant == 4) cudaMemset(buf, 0x3f, (size_t)rows * K * 2);  // nonzero operands
      stream_kernel<<<ctas, 64, smem>>>(tm, steps, pair_mode, commit, do_mma && pair_mode, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      std::vector<unsigned long long> h(ctas);
      cudaMemcpy(h.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
      unsigned long long worst = 0, best = ~0ull;
      std::vector<std::pair<unsigned long long, int>> per;
      for (auto v : h) {
        const unsigned long long tt = v >> 8;
        worst = tt > worst ? tt : worst;
        best = tt < best ? tt : best;
        per.push_back({tt, (int)(v & 255)});
      }
      std::sort(per.begin(), per.end());
      const double us_step = worst / 1e3 / steps;
      printf("   per-CTA us/step: min %.2f median %.2f max %.2f; slowest SMs:", best / 1e3 / steps,
             per[per.size() / 2].first / 1e3 / steps, us_step);
      for (int i = (int)per.size() - 1; i >= (int)per.size() - 6; --i) printf(" %d", per[i].second);
      printf("\n");
      printf("%s release=%s%s : %.2f us per 256 KB step, %.1f GB/s per CTA\n", pair_mode ? "pair" : "solo",
             commit ? "tcgen05.commit" : "mbarrier.arrive", do_mma ? (variant == 4 ? " +MMA(nonzero)" : " +MMA") : "",
             us_step, 256.0 * 1024 / us_step / 1e3);
    }
  return 0;
}
