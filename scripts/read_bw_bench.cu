// How fast can one kernel stream a 123 MB fp32 buffer (the decoder's enc,
// [256 x 60 x 2000]) once?  (a) grid-stride 16 B / 32 B loads at several grid
// sizes, (b) per-(row, column-slice) CTAs like attn_context_kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 read_bw_bench.cu -o /tmp/rbw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void flat16(const float4* __restrict__ x, int64_t n, float* out) {
  float acc = 0.f;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i + 3 * st < n; i += 4 * st) {
    float4 v0 = __ldg(x + i), v1 = __ldg(x + i + st), v2 = __ldg(x + i + 2 * st), v3 = __ldg(x + i + 3 * st);
    acc += v0.x + v1.y + v2.z + v3.w;
  }
  for (; i < n; i += st) acc += __ldg(x + i).x;
  if (acc == 1.2345f) out[0] = acc;
}

__global__ void flat32(const float* __restrict__ x, int64_t n8, float* out) {
  float acc = 0.f;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i + st < n8; i += 2 * st) {
    float f[16];
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]), "=f"(f[6]), "=f"(f[7])
                 : "l"(x + i * 8));
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(f[8]), "=f"(f[9]), "=f"(f[10]), "=f"(f[11]), "=f"(f[12]), "=f"(f[13]), "=f"(f[14]), "=f"(f[15])
                 : "l"(x + (i + st) * 8));
    acc += f[0] + f[9];
  }
  if (acc == 1.2345f) out[0] = acc;
}

// bulk copies global -> shared (cp.async.bulk), a ring of NS x 16 KB per CTA, persistent
template <int NS>
__global__ void __launch_bounds__(128, 1) bulk(const char* __restrict__ x, int64_t bytes, float* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[NS];
  constexpr int CH = 16384;
  const int64_t nch = bytes / CH;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  float acc = 0.f;
  int64_t c = blockIdx.x;
  int issued = 0;
  // prime
  if (threadIdx.x == 0)
    for (int s = 0; s < NS && c + (int64_t)s * gridDim.x < nch; ++s) {
      const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CH));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(sm + s * CH)),
                   "l"(x + (c + (int64_t)s * gridDim.x) * CH), "r"(CH), "r"(b)
                   : "memory");
    }
  int s = 0;
  unsigned ph = 0;
  for (int64_t k = c; k < nch; k += gridDim.x) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(b), "r"(ph));
    acc += reinterpret_cast<const float*>(sm + s * CH)[threadIdx.x * 32];
    __syncthreads();
    const int64_t kn = k + (int64_t)NS * gridDim.x;
    if (threadIdx.x == 0 && kn < nch) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CH));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(sm + s * CH)),
                   "l"(x + kn * CH), "r"(CH), "r"(b)
                   : "memory");
    }
    if (++s == NS) s = 0, ph ^= 1;
  }
  (void)issued;
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const int64_t n = 256LL * 60 * 2000;  // floats
  const int64_t bytes = n * 4;
  float *x, *out, *flush;
  cudaMalloc(&x, bytes + 1024);
  cudaMalloc(&out, 64);
  const size_t fb = 512ull << 20;
  cudaMalloc(&flush, fb);
  cudaMemset(x, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    float best = 1e9, sum = 0;
    for (int r = 0; r < 12; ++r) {
      cudaMemsetAsync(flush, r, fb);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
    }
    printf("%-36s best %7.2f us (%6.0f GB/s)  avg %7.2f us\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9, sum / 10 * 1e3);
  };
  for (int g : {148, 296, 592, 1184, 2368}) {
    char nm[64];
    snprintf(nm, 64, "flat16 grid %d x 256", g);
    run(nm, [&] { flat16<<<g, 256>>>(reinterpret_cast<const float4*>(x), n / 4, out); });
    snprintf(nm, 64, "flat32 grid %d x 256", g);
    run(nm, [&] { flat32<<<g, 256>>>(x, n / 8, out); });
  }
  cudaFuncSetAttribute(bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaFuncSetAttribute(bulk<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
  run("bulk 16KBx8 ring, 148 CTAs", [&] { bulk<8><<<148, 128, 8 * 16384>>>((const char*)x, bytes, out); });
  run("bulk 16KBx12 ring, 148 CTAs", [&] { bulk<12><<<148, 128, 12 * 16384>>>((const char*)x, bytes, out); });
  run("bulk 16KBx8 ring, 296 CTAs", [&] { bulk<8><<<296, 128, 8 * 16384>>>((const char*)x, bytes, out); });
  // 61 MB (enc_ctx)
  const int64_t n2 = 256LL * 60 * 1000;
  for (int g : {296, 1184}) {
    char nm[64];
    snprintf(nm, 64, "61MB flat32 grid %d", g);
    float best = 1e9;
    for (int r = 0; r < 12; ++r) {
      cudaMemsetAsync(flush, r, fb);
      cudaEventRecord(e0);
      flat32<<<g, 256>>>(x, n2 / 8, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) best = ms < best ? ms : best;
    }
    printf("%-36s best %7.2f us (%6.0f GB/s)\n", nm, best * 1e3, n2 * 4 / (best * 1e-3) / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
