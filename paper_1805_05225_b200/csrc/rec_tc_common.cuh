// Helpers shared by the tensor-core recurrence kernels (rec_tc.cu, rec_tc_bwd.cu).
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc.cuh"

namespace sl {
namespace rtc {

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(tc::smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(tc::smem_u32(bar))
      : "memory");
}

// 4-D tile load: {k_in, rows, k_chunk, slot} view of a [slot][rows][K] ring,
// so one op can carry several 64-wide K chunks (bigger boxes stream faster).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(tc::smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SL_TRACE(k)                                                          \
  do {                                                                       \
    if (a.trace && blockIdx.x == a.trace_cta) a.trace[s * 16 + (k)] = gtimer(); \
  } while (0)

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Row-segment loads/stores of a CTA's unit slice: 16 B vectors for every full
// chunk (partial slices too: the last CTA of a layer whose H is not a
// multiple of U must not fall off the fast path — it would straggle every
// step), scalar only for the ragged tail.  `vec` = the row pitch allows
// vector access at all (the base alignment is checked here).
__device__ __forceinline__ uint4 pack8_bf16(const float* v) {
  uint4 w;
  __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]), p1 = __floats2bfloat162_rn(v[2], v[3]);
  __nv_bfloat162 p2 = __floats2bfloat162_rn(v[4], v[5]), p3 = __floats2bfloat162_rn(v[6], v[7]);
  w.x = *reinterpret_cast<uint32_t*>(&p0);
  w.y = *reinterpret_cast<uint32_t*>(&p1);
  w.z = *reinterpret_cast<uint32_t*>(&p2);
  w.w = *reinterpret_cast<uint32_t*>(&p3);
  return w;
}
__device__ __forceinline__ void unpack8_bf16(uint4 w, float* v) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ws[k]));
    v[2 * k] = f.x;
    v[2 * k + 1] = f.y;
  }
}

template <int U>
__device__ __forceinline__ void store_f32(float* dst, const float* v, int nu) {
  int done = 0;
  if ((U % 4) == 0 && ((uintptr_t)dst & 15) == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 4)
      if (i + 4 <= nu) {
        *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        done = i + 4;
      }
  }
  for (int i = done; i < nu; ++i) dst[i] = v[i];
}
template <int U>
__device__ __forceinline__ void store_bf16(__nv_bfloat16* dst, const float* v, int nu) {
  int done = 0;
  if ((U % 8) == 0 && ((uintptr_t)dst & 15) == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 8)
      if (i + 8 <= nu) {
        *reinterpret_cast<uint4*>(dst + i) = pack8_bf16(v + i);
        done = i + 8;
      }
  } else if ((U % 4) == 0 && ((uintptr_t)dst & 7) == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 4)
      if (i + 4 <= nu) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(v[i], v[i + 1]);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(v[i + 2], v[i + 3]);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&p0);
        w.y = *reinterpret_cast<uint32_t*>(&p1);
        *reinterpret_cast<uint2*>(dst + i) = w;
        done = i + 4;
      }
  }
  for (int i = done; i < nu; ++i) dst[i] = __float2bfloat16_rn(v[i]);
}

template <int U>
__device__ __forceinline__ void load_f32(const float* src, float* v, int nu, bool vec) {
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = 0.f;
  int done = 0;
  if (vec && (U % 4) == 0 && ((uintptr_t)src & 15) == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 4)
      if (i + 4 <= nu) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(src + i));
        v[i] = x.x;
        v[i + 1] = x.y;
        v[i + 2] = x.z;
        v[i + 3] = x.w;
        done = i + 4;
      }
  }
  for (int i = done; i < nu; ++i) v[i] = __ldg(src + i);
}

template <int U>
__device__ __forceinline__ void load_bf16(const __nv_bfloat16* src, float* v, int nu, bool vec) {
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = 0.f;
  int done = 0;
  if (vec && (U % 8) == 0 && ((uintptr_t)src & 15) == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 8)
      if (i + 8 <= nu) {
        unpack8_bf16(__ldg(reinterpret_cast<const uint4*>(src + i)), v + i);
        done = i + 8;
      }
  }
  for (int i = done; i < nu; ++i) v[i] = __bfloat162float(src[i]);
}

template <int n>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float (&v)[n]) {
  if constexpr (n == 8) {
    tc::tmem_ld_32x32b_x8(taddr, v);
  } else if constexpr (n == 4) {
    tc::tmem_ld_32x32b_x4(taddr, v);
  } else if constexpr (n == 16) {
    tc::tmem_ld_32x32b_x16(taddr, v);
  } else {
    static_assert(n == 2, "unsupported tmem load width");
    tc::tmem_ld_32x32b_x2(taddr, v);
  }
}


// ---- host: TMA descriptors (bf16, SWIZZLE_128B unless stated)
inline PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    SL_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    SL_REQUIRE(q == cudaDriverEntryPointSuccess && f, SL_ERR_CUDA, "cuTensorMapEncodeTiled missing");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

inline CUtensorMap tmap(const void* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                 const cuuint32_t* box) {
  CUtensorMap m;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SL_REQUIRE(r == CUDA_SUCCESS, SL_ERR_CUDA, "cuTensorMapEncodeTiled failed (recurrence)");
  return m;
}


}  // namespace rtc
}  // namespace sl

namespace sl {
namespace rtc {

// ---- thread-block-cluster / DSMEM primitives
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cta address -> the same variable's shared::cluster address in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}
// n floats (n % 4 == 0) to a 16 B aligned shared::cluster address
template <int n>
__device__ __forceinline__ void st_cluster_vec(uint32_t addr, const float* v) {
#pragma unroll
  for (int i = 0; i < n; i += 4) st_cluster_v4(addr + i * 4, v[i], v[i + 1], v[i + 2], v[i + 3]);
}
// arrive (release, cluster scope) on an mbarrier of another CTA of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr, uint32_t count) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(count)
               : "memory");
}
// wait with cluster-scope acquire (sees DSMEM writes released by peers)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(tc::smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace rtc
}  // namespace sl
