// BF16 tensor-core GEMM for sm_100a: TMA -> shared (SWIZZLE_128B) -> tcgen05.mma
// -> TMEM -> fused epilogue.  Used by the SL_PREC_BF16 path for
//   K1  XW[B*T, 8H]  = X . [W_fw | W_bw] + b          (A K-major,  B N-major)
//   K4  dX[B*T, D]  (+)= DZ . [W_fw | W_bw]^T         (A K-major,  B K-major)
//       dW[D, 8H]   (+)= X^T . DZ                     (A M-major,  B N-major)
//       dR[H, 4H]   (+)= Hprev^T . DZ_d               (A M-major,  B N-major)
// i.e. the reference's per-step Eigen products (tape.cpp:1103, 1174-1203)
// hoisted into one GEMM each over all B*T rows.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: 4-stage ring of {A 128x64, B BNx64} bf16 tiles
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> alpha*acc + bias + beta*C -> fp32 global
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile i overlap the
// MMAs of tile i+1.  Operand majorness is a compile-time switch so the same
// kernel serves X.W, DZ.W^T and X^T.DZ without any transpose pass.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "gemm.h"
#include "profile.h"
#include "tc.cuh"

namespace sl {
namespace {

constexpr int BM = 128, BK = 64, kStages = 4, kThreads = 192;
constexpr uint32_t kBoxBytes = 64 * 64 * 2;  // one 64(MN) x 64(K) bf16 box = 8 KB

struct Params {
  int M, N, K;
  int nm, nn, nk;
  float* C;
  int64_t ldc;
  float alpha, beta;
  const float* bias;
  int m_split;
  float* C2;
  int64_t ldc2;
  __nv_bfloat16* Cb;  // bf16 output instead of C (beta must be 0)
  int a_blk3d, b_blk3d;  // MN-major operand loaded as ONE 3-D box per stage
};

__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                     int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(tc::smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(tc::smem_u32(bar))
      : "memory");
}

template <int BN>
struct Smem {
  static constexpr uint32_t kA = BM * BK * 2;  // 16 KB
  static constexpr uint32_t kB = BN * BK * 2;  // 16 / 32 KB
  static constexpr uint32_t kStage = kA + kB;
  static constexpr uint32_t kBytes = kStages * kStage + 1024;  // + alignment slack
};

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, Params p) {
  using S = Smem<BN>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  const uint32_t base = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - tc::smem_u32(smem_raw));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr uint32_t kTmemCols = 2 * BN;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull_bar[a], 1);
      tc::mbar_init(&tempty_bar[a], 128);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(&tmem_base_sh);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base_sh;
  const int ntiles = p.nm * p.nn;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t % p.nm) * BM, n0 = (t / p.nm) * BN;
        for (int kb = 0; kb < p.nk; ++kb) {
          tc::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::kStage;
          uint8_t* sb = sa + S::kA;
          tc::mbar_arrive_expect_tx(&full_bar[stage], S::kStage);
          const int k0 = kb * BK;
          if (A_MN) {
            if (p.a_blk3d) {  // {mn_in 64, k rows 64, mn blocks}: the whole stage in one op
              tma3(sa, &tmA, &full_bar[stage], 0, k0, m0 / 64);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tc::tma_load_2d(sa + j * kBoxBytes, &tmA, &full_bar[stage], m0 + 64 * j, k0);
            }
          } else {
            tc::tma_load_2d(sa, &tmA, &full_bar[stage], k0, m0);
          }
          if (B_MN) {
            if (p.b_blk3d) {
              tma3(sb, &tmB, &full_bar[stage], 0, k0, n0 / 64);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tc::tma_load_2d(sb + j * kBoxBytes, &tmB, &full_bar[stage], n0 + 64 * j, k0);
            }
          } else {
            tc::tma_load_2d(sb, &tmB, &full_bar[stage], k0, n0);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = tc::make_idesc(BM, BN, 1, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t use = (uint32_t)(it >> 1);
        tc::mbar_wait(&tempty_bar[acc], (use & 1) ^ 1);
        tc::fence_after_sync();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int kb = 0; kb < p.nk; ++kb) {
          tc::mbar_wait(&full_bar[stage], phase);
          tc::fence_after_sync();
          const uint32_t sa = base + stage * S::kStage;
          const uint32_t sb = sa + S::kA;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: advance 16 elems = 32 B inside the 128 B swizzle row.
            // MN-major: advance 16 K-rows = 2 KB; MN blocks 8 KB apart (LBO).
            const uint64_t ad = A_MN ? tc::make_sdesc(sa + k * 2048, kBoxBytes, 1024)
                                     : tc::make_sdesc(sa + k * 32, 0, 1024);
            const uint64_t bd = B_MN ? tc::make_sdesc(sb + k * 2048, kBoxBytes, 1024)
                                     : tc::make_sdesc(sb + k * 32, 0, 1024);
            tc::mma_f16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          tc::mma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs finish
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc::mma_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {  // ---------------- epilogue (warps 2..5 -> TMEM lane quarters 2,3,0,1)
    const int q = warp & 3;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t use = (uint32_t)(it >> 1);
      const int m0 = (t % p.nm) * BM, n0 = (t / p.nm) * BN;
      tc::mbar_wait(&tfull_bar[acc], use & 1);
      tc::fence_after_sync();
      const int row = m0 + 32 * q + lane;
      const bool second = row >= p.m_split;
      float* crow = second ? p.C2 + (int64_t)(row - p.m_split) * p.ldc2 : p.C + (int64_t)row * p.ldc;
      const bool vec = second ? (p.ldc2 % 4) == 0 && ((uintptr_t)p.C2 & 15) == 0
                              : (p.ldc % 4) == 0 && ((uintptr_t)p.C & 15) == 0;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tc::tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + acc * BN + c, v);
        const int col0 = n0 + c;
        if (p.Cb) {  // bf16 output (K1's XW): alpha * acc + bias, rounded
          if (row >= p.M) continue;
          __nv_bfloat16* brow = p.Cb + (int64_t)row * p.ldc + col0;
          if (col0 + 32 <= p.N && (p.ldc % 8) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              float o[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = p.alpha * v[j + i] + (p.bias ? p.bias[col0 + j + i] : 0.f);
              uint4 w;
              __nv_bfloat162 t0 = __floats2bfloat162_rn(o[0], o[1]), t1 = __floats2bfloat162_rn(o[2], o[3]);
              __nv_bfloat162 t2 = __floats2bfloat162_rn(o[4], o[5]), t3 = __floats2bfloat162_rn(o[6], o[7]);
              w.x = *reinterpret_cast<uint32_t*>(&t0);
              w.y = *reinterpret_cast<uint32_t*>(&t1);
              w.z = *reinterpret_cast<uint32_t*>(&t2);
              w.w = *reinterpret_cast<uint32_t*>(&t3);
              *reinterpret_cast<uint4*>(brow + j) = w;
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j)
              brow[j] = __float2bfloat16_rn(p.alpha * v[j] + (p.bias ? p.bias[col0 + j] : 0.f));
          }
          continue;
        }
        if (row >= p.M || (second ? p.C2 : p.C) == nullptr) continue;
        if (vec && col0 + 32 <= p.N) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o;
            o.x = p.alpha * v[j];
            o.y = p.alpha * v[j + 1];
            o.z = p.alpha * v[j + 2];
            o.w = p.alpha * v[j + 3];
            if (p.bias) {
              const float4 bb = *reinterpret_cast<const float4*>(p.bias + col0 + j);
              o.x += bb.x;
              o.y += bb.y;
              o.z += bb.z;
              o.w += bb.w;
            }
            float4* dst = reinterpret_cast<float4*>(crow + col0 + j);
            if (p.beta != 0.f) {
              const float4 old = *dst;
              o.x += p.beta * old.x;
              o.y += p.beta * old.y;
              o.z += p.beta * old.z;
              o.w += p.beta * old.w;
            }
            *dst = o;
          }
        } else {
          for (int j = 0; j < 32 && col0 + j < p.N; ++j) {
            float o = p.alpha * v[j];
            if (p.bias) o += p.bias[col0 + j];
            float* dst = crow + col0 + j;
            if (p.beta != 0.f) o += p.beta * *dst;
            *dst = o;
          }
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&tempty_bar[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<kTmemCols>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  SL_REQUIRE(fn != nullptr, SL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// Row-major bf16 matrix [outer, inner] with leading dimension ld (elements),
// boxes of 64 (inner, = one 128 B swizzle row) x box_outer.
CUtensorMap tmap_bf16(const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  SL_REQUIRE(((uintptr_t)ptr & 15) == 0 && (ld * 2) % 16 == 0, SL_ERR_INVALID_ARGUMENT,
             "gemm_bf16_tc: operands need 16 B aligned base and leading dimension % 8 == 0");
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SL_REQUIRE(r == CUDA_SUCCESS, SL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

// MN-major operand stored [K, MN] (ld) as a 3-D map {64 (mn within block),
// K rows, MN blocks of 64}: one box = `nblk` 64x64 blocks laid out block after
// block (8 KB apart = the UMMA descriptor's LBO).  Reads whole 64-wide blocks,
// so the caller must guarantee round_up(MN, 64) readable elements per row.
CUtensorMap tmap_bf16_mn3(const void* ptr, int64_t mn, int64_t k, int64_t ld, int nblk) {
  SL_REQUIRE(((uintptr_t)ptr & 15) == 0 && (ld * 2) % 16 == 0, SL_ERR_INVALID_ARGUMENT,
             "gemm_bf16_tc: operands need 16 B aligned base and leading dimension % 8 == 0");
  CUtensorMap m;
  cuuint64_t dims[3] = {64, (cuuint64_t)k, (cuuint64_t)ceil_div(mn, 64)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), 128};
  cuuint32_t box[3] = {64, 64, (cuuint32_t)nblk};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SL_REQUIRE(r == CUDA_SUCCESS, SL_ERR_CUDA, "cuTensorMapEncodeTiled failed (mn3)");
  return m;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int BN, bool A_MN, bool B_MN>
void launch(const CUtensorMap& a, const CUtensorMap& b, const Params& p, cudaStream_t s) {
  auto kern = gemm_bf16_tc_kernel<BN, A_MN, B_MN>;
  static bool configured = false;
  if (!configured) {
    SL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Smem<BN>::kBytes));
    configured = true;
  }
  const int tiles = p.nm * p.nn;
  const int grid = std::min(tiles, num_sms());
  kern<<<grid, kThreads, Smem<BN>::kBytes, s>>>(a, b, p);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace

void gemm_bf16_tc(const TcGemm& g, cudaStream_t stream) {
  if (g.M <= 0 || g.N <= 0) return;
  constexpr bool one_cta = false;  // (the single-CTA form stays for operands the pair GEMM cannot load)
  SL_REQUIRE(!g.sm_part || gemm_bf16_tc2_ok(g), SL_ERR_UNSUPPORTED,
             "gemm_bf16_tc: softmax partials need the CTA-pair GEMM");
  if ((!one_cta || g.sm_part) && gemm_bf16_tc2_ok(g)) {
    SL_REQUIRE(!g.Cb || g.beta == 0.f, SL_ERR_INVALID_ARGUMENT, "gemm_bf16_tc: bf16 output needs beta = 0");
    gemm_bf16_tc2(g, stream);
    return;
  }
  SL_REQUIRE(g.ksplit <= 1, SL_ERR_UNSUPPORTED, "gemm_bf16_tc: split-K needs the CTA-pair GEMM");
  SL_REQUIRE(!g.A_lo && !g.B_lo, SL_ERR_UNSUPPORTED, "gemm_bf16_tc: x3 operands need the CTA-pair GEMM");
  SL_REQUIRE(g.kchunk <= 0, SL_ERR_UNSUPPORTED, "gemm_bf16_tc: chunked accumulation needs the CTA-pair GEMM");
  constexpr int BN = 256;
  Params p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.nm = (int)ceil_div(g.M, BM);
  p.nn = (int)ceil_div(g.N, BN);
  p.nk = (int)ceil_div(g.K, BK);
  p.C = g.C;
  p.ldc = g.ldc;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.bias = g.bias;
  p.m_split = g.m_split;
  p.C2 = g.C2;
  p.ldc2 = g.ldc2;
  p.Cb = g.Cb;
  SL_REQUIRE(!g.Cb || g.beta == 0.f, SL_ERR_INVALID_ARGUMENT, "gemm_bf16_tc: bf16 output needs beta = 0");
  // A: K-major stored [M, K]; MN-major stored [K, M].  B: K-major stored [N, K]; MN-major [K, N].
  // one 3-D box per stage for MN-major operands when whole 64-blocks are readable
  // (the LSTM's buffers are padded so; callers offsetting into a row, like
  // DZ's per-direction column blocks, keep offset + round_up(MN, 64) <= ld)
  p.a_blk3d = g.a_mn && g.lda >= round_up(g.M, 64);
  p.b_blk3d = g.b_mn && g.ldb >= round_up(g.N, 64);
  const CUtensorMap ta = g.a_mn ? (p.a_blk3d ? tmap_bf16_mn3(g.A, g.M, g.K, g.lda, BM / 64)
                                             : tmap_bf16(g.A, g.M, g.K, g.lda, 64))
                                : tmap_bf16(g.A, g.K, g.M, g.lda, BM);
  const CUtensorMap tb = g.b_mn ? (p.b_blk3d ? tmap_bf16_mn3(g.B, g.N, g.K, g.ldb, BN / 64)
                                             : tmap_bf16(g.B, g.N, g.K, g.ldb, 64))
                                : tmap_bf16(g.B, g.K, g.N, g.ldb, BN);
  if (!g.a_mn && g.b_mn) launch<BN, false, true>(ta, tb, p, stream);
  else if (!g.a_mn && !g.b_mn) launch<BN, false, false>(ta, tb, p, stream);
  else if (g.a_mn && g.b_mn) launch<BN, true, true>(ta, tb, p, stream);
  else launch<BN, true, false>(ta, tb, p, stream);
}

}  // namespace sl
