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

// 256-bit global accesses (sm_100: one request per 32 B; the recurrence
// epilogues are request-rate bound, not byte bound)
__device__ __forceinline__ void st256(void* p, uint4 a, uint4 b) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
__device__ __forceinline__ void ld256_nc(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void ld256(const void* p, uint4& a, uint4& b) {  // coherent (data of this kernel)
  asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p)
               : "memory");
}

// Row-segment loads / stores of a thread's unit slice [0, nu) of U values.
// Granule cascade: 32 B accesses where aligned, then 16 B, 8 B, scalar for the
// ragged remainder — a partial slice (the last CTA of a layer whose H is not a
// multiple of the slice) must stay on wide accesses or it straggles every
// step.  All register indexing is static (no local-memory arrays).
__device__ __forceinline__ bool aligned_to(const void* p, int bytes) {
  return ((uintptr_t)p & (uintptr_t)(bytes - 1)) == 0;
}

template <int U>
__device__ __forceinline__ void store_f32(float* dst, const float* v, int nu) {
  int done = 0;
  if constexpr (U % 8 == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 8)
      if (i == done && i + 8 <= nu && aligned_to(dst + i, 32)) {
        st256(dst + i, make_uint4(__float_as_uint(v[i]), __float_as_uint(v[i + 1]), __float_as_uint(v[i + 2]),
                                  __float_as_uint(v[i + 3])),
              make_uint4(__float_as_uint(v[i + 4]), __float_as_uint(v[i + 5]), __float_as_uint(v[i + 6]),
                         __float_as_uint(v[i + 7])));
        done = i + 8;
      }
  }
  if constexpr (U % 4 == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 4)
      if (i == done && i + 4 <= nu && aligned_to(dst + i, 16)) {
        *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        done = i + 4;
      }
  }
#pragma unroll
  for (int i = 0; i < U; ++i)
    if (i >= done && i < nu) dst[i] = v[i];
}

template <int U>
__device__ __forceinline__ void store_bf16(__nv_bfloat16* dst, const float* v, int nu) {
  int done = 0;
  if constexpr (U % 16 == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 16)
      if (i == done && i + 16 <= nu && aligned_to(dst + i, 32)) {
        st256(dst + i, pack8_bf16(v + i), pack8_bf16(v + i + 8));
        done = i + 16;
      }
  }
  if constexpr (U % 8 == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 8)
      if (i == done && i + 8 <= nu && aligned_to(dst + i, 16)) {
        *reinterpret_cast<uint4*>(dst + i) = pack8_bf16(v + i);
        done = i + 8;
      }
  }
  if constexpr (U % 4 == 0) {
#pragma unroll
    for (int i = 0; i < U; i += 4)
      if (i == done && i + 4 <= nu && aligned_to(dst + i, 8)) {
        const __nv_bfloat162 p0 = __floats2bfloat162_rn(v[i], v[i + 1]);
        const __nv_bfloat162 p1 = __floats2bfloat162_rn(v[i + 2], v[i + 3]);
        *reinterpret_cast<uint2*>(dst + i) =
            make_uint2(*reinterpret_cast<const uint32_t*>(&p0), *reinterpret_cast<const uint32_t*>(&p1));
        done = i + 4;
      }
  }
#pragma unroll
  for (int i = 0; i < U; ++i)
    if (i >= done && i < nu) dst[i] = __float2bfloat16_rn(v[i]);
}

// v as its split-bf16 image: hi at dst, lo (v - bf16(v)) lo_off elements further on
template <int U>
__device__ __forceinline__ void store_split(__nv_bfloat16* dst, int64_t lo_off, const float* v, int nu) {
  float l[U];
#pragma unroll
  for (int u = 0; u < U; ++u) l[u] = v[u] - __bfloat162float(__float2bfloat16_rn(v[u]));
  store_bf16<U>(dst, v, nu);
  store_bf16<U>(dst + lo_off, l, nu);
}

// zero-filled beyond nu; vec = the row pitch allows vector access at all
template <int U>
__device__ __forceinline__ void load_f32(const float* src, float* v, int nu, bool vec) {
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = 0.f;
  int done = 0;
  if constexpr (U % 4 == 0) {
    if (vec) {
#pragma unroll
      for (int i = 0; i < U; i += 4)
        if (i == done && i + 4 <= nu && aligned_to(src + i, 16)) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(src + i));
          v[i] = x.x;
          v[i + 1] = x.y;
          v[i + 2] = x.z;
          v[i + 3] = x.w;
          done = i + 4;
        }
    }
  }
#pragma unroll
  for (int i = 0; i < U; ++i)
    if (i >= done && i < nu) v[i] = __ldg(src + i);
}

template <int U>
__device__ __forceinline__ void load_bf16(const __nv_bfloat16* src, float* v, int nu, bool vec) {
#pragma unroll
  for (int i = 0; i < U; ++i) v[i] = 0.f;
  int done = 0;
  if constexpr (U % 8 == 0) {
    if (vec) {
#pragma unroll
      for (int i = 0; i < U; i += 8)
        if (i == done && i + 8 <= nu && aligned_to(src + i, 16)) {
          unpack8_bf16(__ldg(reinterpret_cast<const uint4*>(src + i)), v + i);
          done = i + 8;
        }
    }
  }
#pragma unroll
  for (int i = 0; i < U; ++i)
    if (i >= done && i < nu) v[i] = __bfloat162float(src[i]);
}

// U bf16 values kept packed in registers (U/2 words): halves the register
// cost of operands prefetched a whole step ahead.  All indexing is static.
template <int U>
struct Bf16Vec {
  static_assert(U % 4 == 0, "Bf16Vec: multiple of 4");
  uint32_t w[U / 2];
  __device__ __forceinline__ float operator[](int i) const {
    const uint32_t x = w[i / 2];
    return __uint_as_float((i & 1) ? (x & 0xffff0000u) : (x << 16));
  }
  __device__ __forceinline__ void pack(const float* v) {
#pragma unroll
    for (int i = 0; i < U; i += 2) {
      const __nv_bfloat162 p = __floats2bfloat162_rn(v[i], v[i + 1]);
      w[i / 2] = *reinterpret_cast<const uint32_t*>(&p);
    }
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < U / 2; ++i) w[i] = 0u;
  }
  __device__ __forceinline__ void store(__nv_bfloat16* dst, int nu) const {
    int done = 0;
    if constexpr (U % 16 == 0) {
#pragma unroll
      for (int i = 0; i < U; i += 16)
        if (i == done && i + 16 <= nu && aligned_to(dst + i, 32)) {
          st256(dst + i, make_uint4(w[i / 2], w[i / 2 + 1], w[i / 2 + 2], w[i / 2 + 3]),
                make_uint4(w[i / 2 + 4], w[i / 2 + 5], w[i / 2 + 6], w[i / 2 + 7]));
          done = i + 16;
        }
    }
    if constexpr (U % 8 == 0) {
#pragma unroll
      for (int i = 0; i < U; i += 8)
        if (i == done && i + 8 <= nu && aligned_to(dst + i, 16)) {
          *reinterpret_cast<uint4*>(dst + i) = make_uint4(w[i / 2], w[i / 2 + 1], w[i / 2 + 2], w[i / 2 + 3]);
          done = i + 8;
        }
    }
#pragma unroll
    for (int i = 0; i < U; i += 4)
      if (i == done && i + 4 <= nu && aligned_to(dst + i, 8)) {
        *reinterpret_cast<uint2*>(dst + i) = make_uint2(w[i / 2], w[i / 2 + 1]);
        done = i + 4;
      }
    unsigned short* d16 = reinterpret_cast<unsigned short*>(dst);
#pragma unroll
    for (int i = 0; i < U; ++i)
      if (i >= done && i < nu) d16[i] = (unsigned short)((i & 1) ? (w[i / 2] >> 16) : (w[i / 2] & 0xffffu));
  }
  // full slice from shared memory (generic loads; 8 B / 16 B aligned)
  __device__ __forceinline__ void load_shared(const __nv_bfloat16* src) {
    if constexpr (U % 8 == 0) {
#pragma unroll
      for (int i = 0; i < U; i += 8) {
        const uint4 q = *reinterpret_cast<const uint4*>(src + i);
        w[i / 2] = q.x;
        w[i / 2 + 1] = q.y;
        w[i / 2 + 2] = q.z;
        w[i / 2 + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < U; i += 4) {
        const uint2 q = *reinterpret_cast<const uint2*>(src + i);
        w[i / 2] = q.x;
        w[i / 2 + 1] = q.y;
      }
    }
  }
  // zero-filled beyond nu; vec = the row pitch allows vector access at all
  __device__ __forceinline__ void load(const __nv_bfloat16* src, int nu, bool vec) {
    zero();
    int done = 0;
    if (vec) {
      if constexpr (U % 16 == 0) {
#pragma unroll
        for (int i = 0; i < U; i += 16)
          if (i == done && i + 16 <= nu && aligned_to(src + i, 32)) {
            uint4 q0, q1;
            ld256_nc(src + i, q0, q1);
            w[i / 2] = q0.x;
            w[i / 2 + 1] = q0.y;
            w[i / 2 + 2] = q0.z;
            w[i / 2 + 3] = q0.w;
            w[i / 2 + 4] = q1.x;
            w[i / 2 + 5] = q1.y;
            w[i / 2 + 6] = q1.z;
            w[i / 2 + 7] = q1.w;
            done = i + 16;
          }
      }
      if constexpr (U % 8 == 0) {
#pragma unroll
        for (int i = 0; i < U; i += 8)
          if (i == done && i + 8 <= nu && aligned_to(src + i, 16)) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(src + i));
            w[i / 2] = q.x;
            w[i / 2 + 1] = q.y;
            w[i / 2 + 2] = q.z;
            w[i / 2 + 3] = q.w;
            done = i + 8;
          }
      }
#pragma unroll
      for (int i = 0; i < U; i += 4)
        if (i == done && i + 4 <= nu && aligned_to(src + i, 8)) {
          const uint2 q = __ldg(reinterpret_cast<const uint2*>(src + i));
          w[i / 2] = q.x;
          w[i / 2 + 1] = q.y;
          done = i + 4;
        }
    }
    const unsigned short* s16 = reinterpret_cast<const unsigned short*>(src);
#pragma unroll
    for (int i = 0; i < U; ++i)
      if (i >= done && i < nu) w[i / 2] |= (uint32_t)__ldg(s16 + i) << ((i & 1) * 16);
  }
};

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
                 const cuuint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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
// relaxed remote arrive: pure signalling (e.g. "I have read the accumulator" /
// "your slot in my buffer is free"), no wait for this thread's earlier global
// stores to drain the way a .release arrive must
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_addr, uint32_t count) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(count)
               : "memory");
}
// DSMEM store that completes `bytes` of transaction count on the DESTINATION
// CTA's mbarrier (the receiver arms it with expect_tx): no release fence
__device__ __forceinline__ void st_async_v4(uint32_t addr, uint4 v, uint32_t bar_cl) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   addr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(bar_cl)
               : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t addr, uint2 v, uint32_t bar_cl) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "r"(v.x), "r"(v.y), "r"(bar_cl)
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


// ---- paired fp32 math (sm_100 FFMA2 / FMUL2 / FADD2: two lanes per instruction)
// The recurrence epilogues are instruction-issue bound (16 warps on 4
// schedulers do the per-unit gate math at once), so units are processed in pairs.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2s(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 tanh2(float2 x) { return f2(tc::tanh_approx(x.x), tc::tanh_approx(x.y)); }
// sigmoid(x) = 0.5 tanh(x / 2) + 0.5
__device__ __forceinline__ float2 sigmoid2(float2 x) {
  return fma2(f2s(0.5f), tanh2(mul2(f2s(0.5f), x)), f2s(0.5f));
}
// the two bf16 of one packed word as (low, high) floats
__device__ __forceinline__ float2 bf16x2_f2(uint32_t w) {
  return f2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// Bulk L2 prefetch by the TMA engine (no registers, no LSU requests): pulls a
// contiguous range into L2 ahead of the epilogue's loads.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- CTA-pair (cta_group::2) primitives
// TMA into this CTA's smem whose completion is signalled on the barrier at
// shared::cluster address `bar_cl` (the pair leader's)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cl, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(tc::smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(bar_cl)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cl, int c0,
                                                 int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(tc::smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_cl)
      : "memory");
}
// D[tmem] (+)= A . B for the pair: M = 256 (128 rows of A per CTA), N split
// over the two CTAs' B halves; issued by the leader only
__device__ __forceinline__ void mma_f16_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                             bool acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)acc)
      : "memory");
}
// arrive once on the barrier at this smem offset in BOTH CTAs of the pair when
// the issuing thread's prior MMAs complete
// (mask = the pair's two cluster ranks; 0x3 for a 2-CTA cluster)
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask = 0x3) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(tc::smem_u32(bar)),
      "h"(mask)
      : "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem) {  // whole warp, both CTAs
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   tc::smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

}  // namespace rtc
}  // namespace sl
