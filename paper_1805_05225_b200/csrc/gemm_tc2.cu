// 2-CTA (CTA-pair) BF16 tensor-core GEMM: tcgen05.mma.cta_group::2, M = 256.
//
// The same operation as gemm_tc.cu (C = alpha op(A) op(B) + beta C + bias,
// K-/MN-major operands, fp32 / bf16 / split-C epilogues) with the Blackwell
// CTA-pair datapath: a cluster of two CTAs on one TPC computes a 256 x 256
// tile; each CTA TMA-loads its 128 rows of A and its 128 columns of B per
// K-block (32 KB per stage instead of 48 KB for a 128 x 256 single-CTA tile),
// the leader issues one M=256 N=256 K=16 MMA for both, and each CTA's TMEM
// receives its 128 rows of the accumulator.  Both CTAs' TMA loads complete on
// the LEADER's full barrier (.cta_group::2), MMA completion is multicast to
// both CTAs' empty / tmem-full barriers, and both epilogues release the
// accumulator on the leader's tmem-empty barrier.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "gemm.h"
#include "profile.h"
#include "tc.cuh"

namespace sl {
namespace {

// warps: 0 TMA producer, 1 MMA issuer, 2..9 epilogue (two warps per TMEM lane
// quarter, each draining half of the 256 accumulator columns: the epilogue of a
// tile must hide under the next tile's mainloop, which for short K it did not
// with one warp per quarter)
constexpr int BMP = 256, BNP = 256, BK = 64, kStages = 6, kEpiWarps = 8, kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kHalf = 128 * 64 * 2;  // 16 KB: 128 rows (or cols) x 64 K of bf16
constexpr uint32_t kStage = 2 * kHalf;    // A half + B half per CTA
// + per epilogue warp one 32 x 32 fp32 block: the plain-output epilogue's transpose
// staging (coalesced row-segment stores)
constexpr uint32_t kEpiBlock = 32 * 32 * 4;
constexpr uint32_t kSmem = kStages * kStage + 1024 + kEpiWarps * kEpiBlock;
// X3 (fp32-class) mode: a stage holds A_hi, B_hi, A_lo, B_lo of one 64-wide K block
// (64 KB per CTA, 3 stages in the same shared memory) and feeds three MMAs per
// 16-wide K step: A_hi B_hi + A_lo B_hi + A_hi B_lo
template <bool X3> __host__ __device__ constexpr int n_stages() { return X3 ? 3 : kStages; }
template <bool X3> __host__ __device__ constexpr uint32_t stage_bytes() { return X3 ? 2 * kStage : kStage; }
static_assert(3 * 2 * kStage <= kStages * kStage, "X3 stages fit the shared memory of the bf16 ones");

struct P2 {
  int M, N, K, nm, nn, nk;
  float* C;
  int64_t ldc;
  float alpha, beta;
  const float* bias;
  int m_split;
  float* C2;
  int64_t ldc2;
  __nv_bfloat16* Cb;

  float4* sm_part;  // softmax partials (gemm.h TcGemm::sm_part)
  int sm_ld;
  const int32_t* sm_targets;
  int ksplit, kb_per;    // split-K: work unit t -> tile t % tiles, K blocks [z kb_per, (z + 1) kb_per), z = t / tiles
  int64_t split_stride;  // ... written to C + z * split_stride
  int kchunk;            // CHUNK kernels: K blocks per accumulation chunk
  int group_m;           // rasterisation group (tile_mn)
};

// Output tile of a tile index: grouped rasterisation — consecutive indices walk GM
// M-tiles (p.group_m) before the next N-tile, so the ~74 tiles in flight at once share
// GM A row-blocks and ~74/GM B column-blocks and their operands stay L2-resident
// (M-fastest over all nm M-tiles re-streamed A from HBM once per N-tile).
__device__ __forceinline__ void tile_mn(const P2& p, int tile, int& mi, int& ni) {
  const int gm = p.group_m;
  const int per_group = gm * p.nn;
  const int g = tile / per_group, l = tile % per_group;
  const int rows = min(gm, p.nm - g * gm);  // the last group may be narrower
  mi = g * gm + l % rows;
  ni = l / rows;
}

// K-block range of work unit t (split-K; ksplit == 1: the whole K)
__device__ __forceinline__ void unit_kb(const P2& p, int t, int& tile, int& kb0, int& kb1, int& z) {
  const int tiles = p.nm * p.nn;
  tile = t % tiles;
  z = t / tiles;
  kb0 = z * p.kb_per;
  kb1 = min(p.nk, kb0 + p.kb_per);
}


__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ float fast_ex2(float x) {  // 2^x, MUFU (ex2.approx.ftz)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// TMA into this CTA's smem, completing on the (possibly peer) barrier `bar_cl`
__device__ __forceinline__ void tma2d_pair(uint32_t dst, const CUtensorMap* m, uint32_t bar_cl, int c0,
                                          int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(bar_cl)
      : "memory");
}
__device__ __forceinline__ void tma3d_pair(uint32_t dst, const CUtensorMap* m, uint32_t bar_cl, int c0,
                                          int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cl)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// arrive on the barrier at this smem offset in BOTH CTAs of the pair when the
// issuing thread's prior MMAs complete
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(tc::smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t bar_cl, uint32_t count) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cl),
               "r"(count)
               : "memory");
}

// debug timeline (sl_debug_gemm_trace): per CTA 8 globaltimer stamps (entry, after the
// prologue, first TMA issued, last MMA committed, accumulator ready in the epilogue,
// epilogue done, final cluster sync, TMEM released)
__device__ unsigned long long* g_gemm_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GT(i)                                                           \
  do {                                                                  \
    if (g_gemm_trace) g_gemm_trace[(size_t)blockIdx.x * 8 + (i)] = gtimer(); \
  } while (0)

// fp32 output of 32 accumulator columns of one row (alpha, bias, beta; 32 B / 16 B / scalar stores)
__device__ __forceinline__ void store_row32(const P2& p, float* crow, int col0, const float (&v)[32], bool vec) {
  if (vec && col0 + 32 <= p.N && p.beta == 0.f && !p.bias && (p.ldc % 8) == 0 && ((uintptr_t)crow & 31) == 0) {
    // plain fp32 tile (split-K partials, plain outputs): 32 B vector stores — full
    // sectors and half the store requests of float4 (the epilogue is request-bound)
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      float* dst = crow + col0 + j;
      asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "f"(p.alpha * v[j]),
                   "f"(p.alpha * v[j + 1]), "f"(p.alpha * v[j + 2]), "f"(p.alpha * v[j + 3]), "f"(p.alpha * v[j + 4]),
                   "f"(p.alpha * v[j + 5]), "f"(p.alpha * v[j + 6]), "f"(p.alpha * v[j + 7])
                   : "memory");
    }
  } else if (vec && col0 + 32 <= p.N) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      float4 o = make_float4(p.alpha * v[j], p.alpha * v[j + 1], p.alpha * v[j + 2], p.alpha * v[j + 3]);
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
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col0 + j >= p.N) break;
      float o = p.alpha * v[j];
      if (p.bias) o += p.bias[col0 + j];
      float* dst = crow + col0 + j;
      if (p.beta != 0.f) o += p.beta * *dst;
      *dst = o;
    }
  }
}

template <bool A_MN, bool B_MN, bool CHUNK, bool X3, bool SMX>
__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    gemm_bf16_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmAl, const __grid_constant__ CUtensorMap tmBl, P2 p) {
  // the softmax-statistics epilogue exists only in the SMX instantiations (the logits
  // GEMM), so its registers do not weigh on every other GEMM's epilogue
  float4* const smp = SMX ? p.sm_part : nullptr;
  constexpr int NST = n_stages<X3>();
  constexpr uint32_t SB = stage_bytes<X3>();
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_sh;
  const uint32_t base = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t r = cta_rank();
  const bool leader = r == 0;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (threadIdx.x == 0) GT(0);
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    if (X3) {
      tc::prefetch_tmap(&tmAl);
      tc::prefetch_tmap(&tmBl);
    }
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull_bar[a], 1);
      tc::mbar_init(&tempty_bar[a], 2 * 32 * kEpiWarps);  // both CTAs' epilogue threads (leader's copy)
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) {  // same warp id in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_sh)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x == 0) GT(1);
  tc::fence_after_sync();
  const uint32_t tmem = tmem_sh;
  const int ntiles = p.nm * p.nn * p.ksplit;  // work units

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int st = 0;
      uint32_t ph = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        int tile, kb0, kb1, z;
        unit_kb(p, t, tile, kb0, kb1, z);
        int mi, ni;
        tile_mn(p, tile, mi, ni);
        const int m0 = mi * BMP + r * 128, n0 = ni * BNP + r * 128;
        for (int kb = kb0; kb < kb1; ++kb) {
          tc::mbar_wait(&empty_bar[st], ph ^ 1);
          const uint32_t sa = base + st * SB, sb = sa + kHalf;
          const uint32_t fb = mapa_u32(tc::smem_u32(&full_bar[st]), 0);  // leader's barrier
          if (leader) tc::mbar_arrive_expect_tx(&full_bar[st], 2 * SB);
          const int k0 = kb * BK;
          if (A_MN) tma3d_pair(sa, &tmA, fb, 0, k0, m0 / 64);
          else tma2d_pair(sa, &tmA, fb, k0, m0);
          if (kb == kb0 && t == pair) GT(2);
          if (B_MN) tma3d_pair(sb, &tmB, fb, 0, k0, n0 / 64);
          else tma2d_pair(sb, &tmB, fb, k0, n0);
          if (X3) {  // the lo halves of both operands
            if (A_MN) tma3d_pair(sa + 2 * kHalf, &tmAl, fb, 0, k0, m0 / 64);
            else tma2d_pair(sa + 2 * kHalf, &tmAl, fb, k0, m0);
            if (B_MN) tma3d_pair(sa + 3 * kHalf, &tmBl, fb, 0, k0, n0 / 64);
            else tma2d_pair(sa + 3 * kHalf, &tmBl, fb, k0, n0);
          }
          if (++st == NST) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ---------------- MMA issuer (leader only)
      constexpr uint32_t idesc = tc::make_idesc(BMP, BNP, 1, A_MN, B_MN);
      int st = 0;
      uint32_t ph = 0;
      int it = 0;  // accumulator uses: one per unit, or (CHUNK) one per K chunk
      for (int t = pair; t < ntiles; t += npairs) {
        int tile, kb0, kb1, z;
        unit_kb(p, t, tile, kb0, kb1, z);
        const int step = CHUNK ? p.kchunk : (kb1 - kb0);
        for (int c0 = kb0; c0 < kb1; c0 += step, ++it) {
          const int c1 = min(kb1, c0 + step);
          const int acc = it & 1;
          tc::mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
          tc::fence_after_sync();
          for (int kb = c0; kb < c1; ++kb) {
            tc::mbar_wait(&full_bar[st], ph);
            tc::fence_after_sync();
            const uint32_t sa = base + st * SB, sb = sa + kHalf;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = A_MN ? tc::make_sdesc(sa + k * 2048, 8192, 1024)
                                       : tc::make_sdesc(sa + k * 32, 0, 1024);
              const uint64_t bd = B_MN ? tc::make_sdesc(sb + k * 2048, 8192, 1024)
                                       : tc::make_sdesc(sb + k * 32, 0, 1024);
              mma_pair(tmem + acc * BNP, ad, bd, idesc, (kb != c0 || k != 0) ? 1u : 0u);
              if (X3) {  // + A_lo B_hi + A_hi B_lo
                const uint32_t sal = sa + 2 * kHalf, sbl = sa + 3 * kHalf;
                const uint64_t adl = A_MN ? tc::make_sdesc(sal + k * 2048, 8192, 1024)
                                          : tc::make_sdesc(sal + k * 32, 0, 1024);
                const uint64_t bdl = B_MN ? tc::make_sdesc(sbl + k * 2048, 8192, 1024)
                                          : tc::make_sdesc(sbl + k * 32, 0, 1024);
                mma_pair(tmem + acc * BNP, adl, bd, idesc, 1u);
                mma_pair(tmem + acc * BNP, ad, bdl, idesc, 1u);
              }
            }
            commit_pair(&empty_bar[st]);  // frees the slot in both CTAs
            if (++st == NST) {
              st = 0;
              ph ^= 1;
            }
          }
          commit_pair(&tfull_bar[acc]);
          GT(3);
        }
      }
    }
  } else {  // ---------------- epilogue (warps 2..9 -> TMEM lane quarters 2,3,0,1, x2 column halves)
    const int q = warp & 3;
    const int half = (warp - 2) / 4;
    const uint32_t tempty_leader[2] = {mapa_u32(tc::smem_u32(&tempty_bar[0]), 0),
                                       mapa_u32(tc::smem_u32(&tempty_bar[1]), 0)};
    int it = 0;
    if constexpr (CHUNK) {  // ---- chunked accumulation: fp32 C only
      for (int t = pair; t < ntiles; t += npairs) {
        int tile, kb0, kb1, z;
        unit_kb(p, t, tile, kb0, kb1, z);
        int mi, ni;
        tile_mn(p, tile, mi, ni);
        const int m0 = mi * BMP + r * 128, n0 = ni * BNP;
        float sum[128];  // this thread's row x the warp's 128 columns, summed over the chunks in fp32
#pragma unroll
        for (int j = 0; j < 128; ++j) sum[j] = 0.f;
        for (int c0 = kb0; c0 < kb1; c0 += p.kchunk, ++it) {
          const int acc = it & 1;
          tc::mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
          tc::fence_after_sync();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float v[32];
            tc::tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + acc * BNP + half * 128 + c * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) sum[c * 32 + j] += v[j];
          }
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) arrive_remote(tempty_leader[acc], 32);  // this chunk's accumulator is free again
        }
        const int row = m0 + 32 * q + lane;
        if (row >= p.M) continue;
        const bool second = row >= p.m_split;
        float* crow = second ? p.C2 + (int64_t)(row - p.m_split) * p.ldc2
                             : p.C + z * p.split_stride + (int64_t)row * p.ldc;
        if (crow == nullptr || (second ? p.C2 : p.C) == nullptr) continue;
        const bool vec = second ? (p.ldc2 % 4) == 0 && ((uintptr_t)p.C2 & 15) == 0
                                : (p.ldc % 4) == 0 && ((uintptr_t)p.C & 15) == 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = sum[c * 32 + j];
          store_row32(p, crow, n0 + half * 128 + c * 32, v, vec);
        }
      }
    } else
    for (int t = pair; t < ntiles; t += npairs, ++it) {
      const int acc = it & 1;
      int tile, kb0, kb1, z;
      unit_kb(p, t, tile, kb0, kb1, z);
      int mi, ni;
      tile_mn(p, tile, mi, ni);
      const int m0 = mi * BMP + r * 128, n0 = ni * BNP;
      tc::mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      if (warp == 2 && lane == 0 && it == 0) GT(4);
      tc::fence_after_sync();
      const int row = m0 + 32 * q + lane;
      const bool second = row >= p.m_split;
      float* crow = second ? p.C2 + (int64_t)(row - p.m_split) * p.ldc2
                           : p.C + z * p.split_stride + (int64_t)row * p.ldc;
      const bool vec = second ? (p.ldc2 % 4) == 0 && ((uintptr_t)p.C2 & 15) == 0
                              : (p.ldc % 4) == 0 && ((uintptr_t)p.C & 15) == 0;
      constexpr int kColsPerWarp = BNP / (kEpiWarps / 4);
      static_assert(kColsPerWarp == 128, "softmax partials are per 128-column block");
      // online softmax statistics of this row over the warp's 128 columns
      float sm_m = -INFINITY, sm_s = 0.f, sm_t = 0.f, sm_y = 0.f;
      const int sm_tgt = (smp && row < p.M) ? p.sm_targets[row] : -1;
      // plain fp32 tile (split-K partials, plain outputs): two TMEM loads in flight per
      // wait, each warp's 32 x 32 blocks transposed through shared memory (16 B chunks
      // XOR-swizzled: conflict-free both ways) and stored as 128 B row segments, four
      // rows per instruction — a quarter of the requests of one 32 B store per row
      const bool plain_tile = !p.Cb && !smp && p.beta == 0.f && p.C != nullptr &&
                              n0 + (half + 1) * kColsPerWarp <= p.N && (p.ldc % 4) == 0 &&
                              ((uintptr_t)p.C & 15) == 0 && (p.split_stride % 4) == 0 &&
                              ((uintptr_t)p.bias & 15) == 0 && __all_sync(0xffffffffu, row < p.M && !second);
      // plain bf16 tile (bf16 outputs without statistics): the same transpose, 64 B row
      // segments (four lanes per row, eight rows per instruction)
      const bool plain_bf16 = !plain_tile && p.Cb != nullptr && n0 + (half + 1) * kColsPerWarp <= p.N &&
                              (p.ldc % 8) == 0 && ((uintptr_t)p.Cb & 15) == 0 && (p.split_stride % 8) == 0 &&
                              ((uintptr_t)p.bias & 15) == 0 && __all_sync(0xffffffffu, row < p.M);
      if (plain_bf16) {
        uint32_t* blk = reinterpret_cast<uint32_t*>(smem_raw + (base - tc::smem_u32(smem_raw)) + NST * SB) +
                        (warp - 2) * 1024;
        __nv_bfloat16* c0p = p.Cb + z * p.split_stride + (int64_t)(m0 + 32 * q) * p.ldc + n0 + half * kColsPerWarp;
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + acc * BNP + half * kColsPerWarp;
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          float v[32];
          tc::tmem_ld_32x32b_x32(ta + cc * 32, v);
          const int col0 = n0 + half * kColsPerWarp + cc * 32;
          float zr[32];  // the stored (bf16-rounded) values, for the softmax statistics
          // row `lane`: 32 bf16 = four 16 B chunks, XOR-swizzled by bits 1-2 of the row
          // (conflict-free for both the row writes and the 8-row reads)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float o[8];
            if (p.bias) {
              const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + 8 * j));
              const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + 8 * j + 4));
              const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = fmaf(p.alpha, v[8 * j + i], bb[i]);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = p.alpha * v[8 * j + i];
            }
            __nv_bfloat162 t0 = __floats2bfloat162_rn(o[0], o[1]), t1 = __floats2bfloat162_rn(o[2], o[3]);
            __nv_bfloat162 t2 = __floats2bfloat162_rn(o[4], o[5]), t3 = __floats2bfloat162_rn(o[6], o[7]);
            *reinterpret_cast<uint4*>(blk + lane * 16 + ((j ^ ((lane >> 1) & 3)) * 4)) =
                make_uint4(*reinterpret_cast<uint32_t*>(&t0), *reinterpret_cast<uint32_t*>(&t1),
                           *reinterpret_cast<uint32_t*>(&t2), *reinterpret_cast<uint32_t*>(&t3));
            zr[8 * j] = __low2float(t0), zr[8 * j + 1] = __high2float(t0), zr[8 * j + 2] = __low2float(t1);
            zr[8 * j + 3] = __high2float(t1), zr[8 * j + 4] = __low2float(t2), zr[8 * j + 5] = __high2float(t2);
            zr[8 * j + 6] = __low2float(t3), zr[8 * j + 7] = __high2float(t3);
          }
          if (smp) {  // statistics of the stored values, one rescale per 32 columns
            float mx[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) mx[i] = fmaxf(fmaxf(zr[i], zr[i + 8]), fmaxf(zr[i + 16], zr[i + 24]));
#pragma unroll
            for (int w = 4; w >= 1; w /= 2)
#pragma unroll
              for (int i = 0; i < w; ++i) mx[i] = fmaxf(mx[i], mx[i + w]);
            const float mn = fmaxf(sm_m, mx[0]);
            constexpr float kL2e = 1.4426950408889634f;
            const float ms = mn * kL2e;
            float es[4] = {0.f, 0.f, 0.f, 0.f}, ts[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              es[j & 3] += fast_ex2(fmaf(zr[j], kL2e, -ms));
              ts[j & 3] += zr[j];
              if (col0 + j == sm_tgt) sm_y = zr[j];
            }
            sm_s = fmaf(sm_s, fast_ex2(fmaf(sm_m, kL2e, -ms)), (es[0] + es[1]) + (es[2] + es[3]));
            sm_t += (ts[0] + ts[1]) + (ts[2] + ts[3]);
            sm_m = mn;
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = 8 * i + lane / 4, ch = lane & 3;
            const uint4 t = *reinterpret_cast<const uint4*>(blk + rr * 16 + ((ch ^ ((rr >> 1) & 3)) * 4));
            *reinterpret_cast<uint4*>(c0p + (int64_t)rr * p.ldc + cc * 32 + ch * 8) = t;
          }
          __syncwarp();
        }
        if (smp)
          smp[(int64_t)row * p.sm_ld + (n0 + half * kColsPerWarp) / 128] = make_float4(sm_m, sm_s, sm_t, sm_y);
      } else if (SMX && !p.Cb && smp && p.beta == 0.f && p.C != nullptr && n0 + (half + 1) * kColsPerWarp <= p.N &&
                 (p.ldc % 4) == 0 && ((uintptr_t)p.C & 15) == 0 && ((uintptr_t)p.bias & 15) == 0 &&
                 __all_sync(0xffffffffu, row < p.M && !second)) {
        // fp32 logits with their softmax statistics: outputs and statistics per row (lane),
        // then the coalesced transpose store of the plain tile
        float* blk = reinterpret_cast<float*>(smem_raw + (base - tc::smem_u32(smem_raw)) + NST * SB) +
                     (warp - 2) * 1024;
        float* c0p = p.C + (int64_t)(m0 + 32 * q) * p.ldc + n0 + half * kColsPerWarp;
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + acc * BNP + half * kColsPerWarp;
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          float o[32];  // the accumulator columns, then (in place) the stored outputs
          tc::tmem_ld_32x32b_x32(ta + cc * 32, o);
          const int col0 = n0 + half * kColsPerWarp + cc * 32;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 bb = p.bias ? __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            o[j] = fmaf(p.alpha, o[j], bb.x), o[j + 1] = fmaf(p.alpha, o[j + 1], bb.y);
            o[j + 2] = fmaf(p.alpha, o[j + 2], bb.z), o[j + 3] = fmaf(p.alpha, o[j + 3], bb.w);
          }
          float mx[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) mx[i] = fmaxf(fmaxf(o[i], o[i + 8]), fmaxf(o[i + 16], o[i + 24]));
#pragma unroll
          for (int w = 4; w >= 1; w /= 2)
#pragma unroll
            for (int i = 0; i < w; ++i) mx[i] = fmaxf(mx[i], mx[i + w]);
          const float mn = fmaxf(sm_m, mx[0]);
          constexpr float kL2e = 1.4426950408889634f;
          const float ms = mn * kL2e;
          float es[4] = {0.f, 0.f, 0.f, 0.f}, ts[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            es[j & 3] += fast_ex2(fmaf(o[j], kL2e, -ms));
            ts[j & 3] += o[j];
            if (col0 + j == sm_tgt) sm_y = o[j];
          }
          sm_s = fmaf(sm_s, fast_ex2(fmaf(sm_m, kL2e, -ms)), (es[0] + es[1]) + (es[2] + es[3]));
          sm_t += (ts[0] + ts[1]) + (ts[2] + ts[3]);
          sm_m = mn;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(blk + lane * 32 + ((j ^ (lane & 7)) * 4)) =
                make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = 4 * i + lane / 8, ch = lane & 7;
            const float4 t = *reinterpret_cast<const float4*>(blk + rr * 32 + ((ch ^ (rr & 7)) * 4));
            *reinterpret_cast<float4*>(c0p + (int64_t)rr * p.ldc + cc * 32 + ch * 4) = t;
          }
          __syncwarp();
        }
        smp[(int64_t)row * p.sm_ld + (n0 + half * kColsPerWarp) / 128] = make_float4(sm_m, sm_s, sm_t, sm_y);
      } else if (plain_tile) {
        float* blk = reinterpret_cast<float*>(smem_raw + (base - tc::smem_u32(smem_raw)) + NST * SB) +
                     (warp - 2) * 1024;
        float* c0p = p.C + z * p.split_stride + (int64_t)(m0 + 32 * q) * p.ldc + n0 + half * kColsPerWarp;
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + acc * BNP + half * kColsPerWarp;
        auto put = [&](const uint32_t(&rv)[32], int cc) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(blk + lane * 32 + ((j ^ (lane & 7)) * 4)) =
                make_float4(p.alpha * __uint_as_float(rv[4 * j]), p.alpha * __uint_as_float(rv[4 * j + 1]),
                            p.alpha * __uint_as_float(rv[4 * j + 2]), p.alpha * __uint_as_float(rv[4 * j + 3]));
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = 4 * i + lane / 8, ch = lane & 7;
            float4 t = *reinterpret_cast<const float4*>(blk + rr * 32 + ((ch ^ (rr & 7)) * 4));
            if (p.bias) {  // this lane's four columns of the bias
              const float4 bb = __ldg(reinterpret_cast<const float4*>(p.bias + n0 + half * kColsPerWarp + cc * 32 + ch * 4));
              t.x += bb.x, t.y += bb.y, t.z += bb.z, t.w += bb.w;
            }
            *reinterpret_cast<float4*>(c0p + (int64_t)rr * p.ldc + cc * 32 + ch * 4) = t;
          }
          __syncwarp();
        };
        {  // all four 32-column loads in flight, one wait
          uint32_t r0[32], r1[32], r2[32], r3[32];
          tc::tmem_ld_32x32b_x32_nw(ta, r0);
          tc::tmem_ld_32x32b_x32_nw(ta + 32, r1);
          tc::tmem_ld_32x32b_x32_nw(ta + 64, r2);
          tc::tmem_ld_32x32b_x32_nw(ta + 96, r3);
          tc::tmem_wait_ld_dep(r0);
          tc::reg_dep(r1);
          tc::reg_dep(r2);
          tc::reg_dep(r3);
          put(r0, 0);
          put(r1, 1);
          put(r2, 2);
          put(r3, 3);
        }
      } else
#pragma unroll 1
      for (int c = half * kColsPerWarp; c < (half + 1) * kColsPerWarp; c += 32) {
        float v[32];
        tc::tmem_ld_32x32b_x32(tmem + ((uint32_t)(32 * q) << 16) + acc * BNP + c, v);
        const int col0 = n0 + c;
        if (p.Cb) {
          if (row >= p.M) continue;
          __nv_bfloat16* brow = p.Cb + z * p.split_stride + (int64_t)row * p.ldc + col0;
          if (col0 + 32 <= p.N && (p.ldc % 8) == 0) {
            const bool bvec = p.bias && ((uintptr_t)(p.bias + col0) & 15) == 0;
            // 32 B stores (two 8-column groups per request) when the row segment allows:
            // the epilogue's uncoalesced per-row stores are request-bound
            const bool v32 = ((uintptr_t)brow & 31) == 0;
            uint4 wlo = make_uint4(0, 0, 0, 0);
            float zr[32];  // the stored (bf16-rounded) values, for the statistics
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              float o[8];
              if (bvec) {  // bias as two 16 B loads per 8 columns (L1-resident across rows)
                const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j));
                const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j + 4));
                const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = fmaf(p.alpha, v[j + i], bb[i]);
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = p.alpha * v[j + i] + (p.bias ? p.bias[col0 + j + i] : 0.f);
              }
              uint4 w;
              __nv_bfloat162 t0 = __floats2bfloat162_rn(o[0], o[1]), t1 = __floats2bfloat162_rn(o[2], o[3]);
              __nv_bfloat162 t2 = __floats2bfloat162_rn(o[4], o[5]), t3 = __floats2bfloat162_rn(o[6], o[7]);
              w.x = *reinterpret_cast<uint32_t*>(&t0);
              w.y = *reinterpret_cast<uint32_t*>(&t1);
              w.z = *reinterpret_cast<uint32_t*>(&t2);
              w.w = *reinterpret_cast<uint32_t*>(&t3);
              if (!v32) {
                *reinterpret_cast<uint4*>(brow + j) = w;
              } else if ((j & 8) == 0) {
                wlo = w;
              } else {
                asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(brow + j - 8),
                             "r"(wlo.x), "r"(wlo.y), "r"(wlo.z), "r"(wlo.w), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w)
                             : "memory");
              }
              zr[j] = __low2float(t0), zr[j + 1] = __high2float(t0), zr[j + 2] = __low2float(t1);
              zr[j + 3] = __high2float(t1), zr[j + 4] = __low2float(t2), zr[j + 5] = __high2float(t2);
              zr[j + 6] = __low2float(t3), zr[j + 7] = __high2float(t3);
            }
            if (smp) {  // statistics of the stored (bf16) values: one rescale per 32 columns
              float mx[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) mx[i] = fmaxf(fmaxf(zr[i], zr[i + 8]), fmaxf(zr[i + 16], zr[i + 24]));
#pragma unroll
              for (int w = 4; w >= 1; w /= 2)
#pragma unroll
                for (int i = 0; i < w; ++i) mx[i] = fmaxf(mx[i], mx[i + w]);
              const float mn = fmaxf(sm_m, mx[0]);
              constexpr float kL2e = 1.4426950408889634f;
              const float ms = mn * kL2e;
              float es[4] = {0.f, 0.f, 0.f, 0.f}, ts[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                es[j & 3] += fast_ex2(fmaf(zr[j], kL2e, -ms));
                ts[j & 3] += zr[j];
                if (col0 + j == sm_tgt) sm_y = zr[j];
              }
              sm_s = fmaf(sm_s, fast_ex2(fmaf(sm_m, kL2e, -ms)), (es[0] + es[1]) + (es[2] + es[3]));
              sm_t += (ts[0] + ts[1]) + (ts[2] + ts[3]);
              sm_m = mn;
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) {
              const __nv_bfloat16 zb = __float2bfloat16_rn(p.alpha * v[j] + (p.bias ? p.bias[col0 + j] : 0.f));
              brow[j] = zb;
              if (smp) {
                const float z = __bfloat162float(zb);
                const float mn = fmaxf(sm_m, z);
                sm_s = sm_s * exp2f((sm_m - mn) * 1.4426950408889634f) + exp2f((z - mn) * 1.4426950408889634f);
                sm_m = mn;
                sm_t += z;
                if (col0 + j == sm_tgt) sm_y = z;
              }
            }
          }
          if (smp && c + 32 == (half + 1) * kColsPerWarp && n0 + half * kColsPerWarp < p.N)
            smp[(int64_t)row * p.sm_ld + (n0 + half * kColsPerWarp) / 128] =
                make_float4(sm_m, sm_s, sm_t, sm_y);
          continue;
        }
        if (row >= p.M || (second ? p.C2 : p.C) == nullptr) continue;
        if (smp) {  // fp32 output: statistics of the stored values (alpha v + bias; beta = 0)
          // the outputs once (bias as 16 B loads), their max as a tree, the exp sum in four
          // independent partial sums (ex2.approx on log2e-scaled values): the statistics stay
          // cheaper than the tile's MMAs, so the epilogue hides under the next tile
          const bool full = col0 + 32 <= p.N;
          float o[32];
          if (full && (!p.bias || ((uintptr_t)(p.bias + col0) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 bb = p.bias ? __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
              o[j] = fmaf(p.alpha, v[j], bb.x);
              o[j + 1] = fmaf(p.alpha, v[j + 1], bb.y);
              o[j + 2] = fmaf(p.alpha, v[j + 2], bb.z);
              o[j + 3] = fmaf(p.alpha, v[j + 3], bb.w);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              o[j] = col0 + j < p.N ? p.alpha * v[j] + (p.bias ? __ldg(p.bias + col0 + j) : 0.f) : -INFINITY;
          }
          float mx[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) mx[i] = fmaxf(fmaxf(o[i], o[i + 8]), fmaxf(o[i + 16], o[i + 24]));
#pragma unroll
          for (int w = 4; w >= 1; w /= 2)
#pragma unroll
            for (int i = 0; i < w; ++i) mx[i] = fmaxf(mx[i], mx[i + w]);
          const float mn = fmaxf(sm_m, mx[0]);
          if (mn != -INFINITY) {
            constexpr float kL2e = 1.4426950408889634f;
            const float ms = mn * kL2e;
            float es[4] = {0.f, 0.f, 0.f, 0.f}, ts[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (full || col0 + j < p.N) {
                es[j & 3] += fast_ex2(fmaf(o[j], kL2e, -ms));
                ts[j & 3] += o[j];
                if (col0 + j == sm_tgt) sm_y = o[j];
              }
            }
            sm_s = fmaf(sm_s, fast_ex2(fmaf(sm_m, kL2e, -ms)), (es[0] + es[1]) + (es[2] + es[3]));
            sm_t += (ts[0] + ts[1]) + (ts[2] + ts[3]);
            sm_m = mn;
          }
          if (c + 32 == (half + 1) * kColsPerWarp && n0 + half * kColsPerWarp < p.N)
            smp[(int64_t)row * p.sm_ld + (n0 + half * kColsPerWarp) / 128] = make_float4(sm_m, sm_s, sm_t, sm_y);
          float* dst = crow + col0;
          if (full && vec && (p.ldc % 8) == 0 && ((uintptr_t)dst & 31) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 8)
              asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + j), "f"(o[j]),
                           "f"(o[j + 1]), "f"(o[j + 2]), "f"(o[j + 3]), "f"(o[j + 4]), "f"(o[j + 5]), "f"(o[j + 6]),
                           "f"(o[j + 7])
                           : "memory");
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < p.N) dst[j] = o[j];
          }
          continue;
        }
        if (vec && col0 + 32 <= p.N && p.beta == 0.f && !p.bias && (p.ldc % 8) == 0 &&
            ((uintptr_t)crow & 31) == 0) {
          // plain fp32 tile (split-K partials, plain outputs): 32 B vector stores — full
          // sectors and half the store requests of float4 (the epilogue is request-bound)
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            float* dst = crow + col0 + j;
            asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst),
                         "f"(p.alpha * v[j]), "f"(p.alpha * v[j + 1]), "f"(p.alpha * v[j + 2]),
                         "f"(p.alpha * v[j + 3]), "f"(p.alpha * v[j + 4]), "f"(p.alpha * v[j + 5]),
                         "f"(p.alpha * v[j + 6]), "f"(p.alpha * v[j + 7])
                         : "memory");
          }
        } else if (vec && col0 + 32 <= p.N) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o = make_float4(p.alpha * v[j], p.alpha * v[j + 1], p.alpha * v[j + 2],
                                   p.alpha * v[j + 3]);
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
      __syncwarp();
      if (lane == 0) arrive_remote(tempty_leader[acc], 32);  // release the accumulator (leader's barrier)
      if (warp == 2 && lane == 0) GT(5);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs / arrivals are done before TMEM goes away
  if (threadIdx.x == 0) GT(6);
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    if (lane == 0) GT(7);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 enc2() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    SL_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

CUtensorMap tm2d(const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  SL_REQUIRE(enc2()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS,
             SL_ERR_CUDA, "cuTensorMapEncodeTiled failed (gemm2 2d)");
  return m;
}
CUtensorMap tm3d_mn(const void* ptr, int64_t mn, int64_t k, int64_t ld) {
  CUtensorMap m;
  cuuint64_t dims[3] = {64, (cuuint64_t)k, (cuuint64_t)ceil_div(mn, 64)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), 128};
  cuuint32_t box[3] = {64, 64, 2};
  cuuint32_t es[3] = {1, 1, 1};
  SL_REQUIRE(enc2()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS,
             SL_ERR_CUDA, "cuTensorMapEncodeTiled failed (gemm2 3d)");
  return m;
}

int sms2() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <bool A_MN, bool B_MN, bool CHUNK, bool X3, bool SMX = false>
void launch2(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& al, const CUtensorMap& bl, const P2& p,
             cudaStream_t s) {
  auto kern = gemm_bf16_tc2_kernel<A_MN, B_MN, CHUNK, X3, SMX>;
  static bool configured = false;
  if (!configured) {
    SL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    configured = true;
  }
  const int tiles = p.nm * p.nn * p.ksplit;
  const int pairs = std::min(tiles, sms2() / 2);
  kern<<<2 * pairs, kThreads, kSmem, s>>>(a, b, al, bl, p);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

}  // namespace

void gemm_tc2_set_trace(unsigned long long* buf) {
  SL_CUDA_TRY(cudaMemcpyToSymbol(g_gemm_trace, &buf, sizeof(buf)));
}

int gemm_tc2_ksplit(int M, int N, int K) {
  const int tiles = (int)(ceil_div(M, BMP) * ceil_div(N, BNP));
  const int nk = (int)ceil_div(K, BK);
  // fill the SM pairs, keeping >= 4 K blocks per unit so the 6-stage pipeline still streams;
  // only for a handful of output tiles — beyond that the partials' extra HBM round trip and
  // the reduction cost more than the idle SMs
  if (tiles > 8) return 1;
  const int want = std::max(1, std::min(sms2() / 2 / tiles, nk / 4));
  return (int)ceil_div(nk, ceil_div(nk, want));  // the count gemm_bf16_tc2 actually runs (no empty units)
}

template <bool X3>
void dispatch2(const TcGemm& g, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tal,
               const CUtensorMap& tbl, const P2& p, cudaStream_t st) {
  const bool ch = g.kchunk > 0;
#define SL_L2(AM, BM)                                                   \
  do {                                                                  \
    if (ch) launch2<AM, BM, true, X3>(ta, tb, tal, tbl, p, st);         \
    else if (p.sm_part) launch2<AM, BM, false, X3, true>(ta, tb, tal, tbl, p, st); \
    else launch2<AM, BM, false, X3>(ta, tb, tal, tbl, p, st);           \
  } while (0)
  if (!g.a_mn && g.b_mn) SL_L2(false, true);
  else if (!g.a_mn && !g.b_mn) SL_L2(false, false);
  else if (g.a_mn && g.b_mn) SL_L2(true, true);
  else SL_L2(true, false);
#undef SL_L2
}

bool gemm_bf16_tc2_ok(const TcGemm& g) {
  // MN-major operands must be loadable as whole 64-wide blocks (3-D boxes)
  return (!g.a_mn || g.lda >= round_up(g.M, 64)) && (!g.b_mn || g.ldb >= round_up(g.N, 64));
}

void gemm_bf16_tc2(const TcGemm& g, cudaStream_t stream) {
  P2 p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.nm = (int)ceil_div(g.M, BMP);
  p.nn = (int)ceil_div(g.N, BNP);
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
  p.ksplit = 1;
  p.kb_per = p.nk;
  p.split_stride = 0;
  if (g.ksplit > 1) {  // fp32 partial products only (the caller reduces them)
    SL_REQUIRE(!g.bias && g.beta == 0.f && g.m_split >= g.M && !g.sm_part, SL_ERR_INVALID_ARGUMENT,
               "gemm_bf16_tc2: split-K writes plain (fp32 or bf16) partials");
    p.kb_per = (int)ceil_div(p.nk, g.ksplit);
    p.ksplit = (int)ceil_div(p.nk, p.kb_per);  // no empty units
    SL_REQUIRE(p.ksplit == g.ksplit, SL_ERR_INVALID_ARGUMENT,
               "gemm_bf16_tc2: split count must be one gemm_tc2_ksplit returns (every partial written)");
    p.split_stride = g.split_stride;
  }
  SL_REQUIRE(((uintptr_t)g.A & 15) == 0 && ((uintptr_t)g.B & 15) == 0 && (g.lda * 2) % 16 == 0 &&
                 (g.ldb * 2) % 16 == 0,
             SL_ERR_INVALID_ARGUMENT, "gemm_bf16_tc2: operands need 16 B alignment");
  const CUtensorMap ta = g.a_mn ? tm3d_mn(g.A, g.M, g.K, g.lda) : tm2d(g.A, g.K, g.M, g.lda, 128);
  const CUtensorMap tb = g.b_mn ? tm3d_mn(g.B, g.N, g.K, g.ldb) : tm2d(g.B, g.K, g.N, g.ldb, 128);
  // bulk-tensor output stores when the output is written (not accumulated) and
  // its rows are 16 B aligned; the per-row path stays for beta != 0
  p.sm_part = g.sm_part;
  p.sm_ld = g.sm_ld;
  p.sm_targets = g.sm_targets;
  SL_REQUIRE(!g.sm_part || (g.sm_targets && g.beta == 0.f && g.m_split >= g.M && g.kchunk == 0 && g.ksplit <= 1),
             SL_ERR_INVALID_ARGUMENT, "gemm: softmax partials need the targets and a plain single-pass output");
  p.kchunk = g.kchunk;
  p.group_m = std::max(1, std::min(p.nm, 8));
  if (g.kchunk > 0)
    SL_REQUIRE(!g.Cb && !g.sm_part, SL_ERR_INVALID_ARGUMENT, "gemm_bf16_tc2: chunked accumulation writes fp32 C");
  const bool x3 = g.A_lo != nullptr;
  SL_REQUIRE(x3 == (g.B_lo != nullptr), SL_ERR_INVALID_ARGUMENT, "gemm_bf16_tc2: x3 mode needs both lo operands");
  if (x3) {
    SL_REQUIRE(((uintptr_t)g.A_lo & 15) == 0 && ((uintptr_t)g.B_lo & 15) == 0 && !g.Cb, SL_ERR_INVALID_ARGUMENT,
               "gemm_bf16_tc2: x3 operands need 16 B alignment and fp32 C");
    const CUtensorMap tal = g.a_mn ? tm3d_mn(g.A_lo, g.M, g.K, g.lda) : tm2d(g.A_lo, g.K, g.M, g.lda, 128);
    const CUtensorMap tbl = g.b_mn ? tm3d_mn(g.B_lo, g.N, g.K, g.ldb) : tm2d(g.B_lo, g.K, g.N, g.ldb, 128);
    dispatch2<true>(g, ta, tb, tal, tbl, p, stream);
  } else {
    dispatch2<false>(g, ta, tb, ta, tb, p, stream);
  }
}

}  // namespace sl
