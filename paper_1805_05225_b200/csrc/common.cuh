// Shared helpers for the sm_100a LSTM kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/seqloom_cuda.h"

namespace sl {

// Thread-local error message behind sl_last_error().
void set_error(const std::string& msg);

struct Error {
  int code;
  std::string msg;
};

#define SL_CUDA_TRY(expr)                                                            \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw ::sl::Error{SL_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

#define SL_REQUIRE(cond, code, msg)                  \
  do {                                               \
    if (!(cond)) throw ::sl::Error{(code), (msg)};   \
  } while (0)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Reference tape.cpp:846 — source time of processing step s under per-sequence reversal.
__device__ __forceinline__ int src_time(int s, int len, int dir) {
  return (dir > 0 || s >= len) ? s : len - 1 - s;
}

// Reference tape.cpp:1119-1126 uses 1/(1+exp(-z)) and std::tanh.  expf/tanhf
// (full-precision, not the __ intrinsics) keep fp32 parity at ~1 ulp.
__device__ __forceinline__ float sigmoidf_(float z) { return 1.0f / (1.0f + expf(-z)); }

// ---- grid-scope flag barrier (one counter per direction) -------------------
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// several counters after ONE release fence: fence_acq_rel_gpu(); red_relaxed_gpu(...) x n
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_gpu(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// All threads of the CTA call this.  `target` = CTAs in the group * (episode+1).
__device__ __forceinline__ void group_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    red_release_gpu(ctr, 1u);
    while (ld_acquire_gpu(ctr) < target) {
    }
  }
  __syncthreads();
}

}  // namespace sl
