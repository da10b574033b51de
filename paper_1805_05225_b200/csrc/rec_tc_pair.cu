// K2, CTA-pair form — persistent tensor-core forward recurrence on the
// Blackwell CTA-pair datapath (tcgen05 .cta_group::2).
//
// Why a pair: the per-step product h_{s-1} [B x H] . R [H x 4H] is a skinny
// GEMM that must be spread over ~128 SMs, so each SM can only keep a 64-column
// slice of R (128 KB bf16) resident.  A single-CTA M = 128 x N = 64 MMA runs at
// half the tensor-core rate (it costs as much as N = 128), and each CTA must
// stream all B rows of h_{s-1} through its shared memory.  A CTA pair instead
// issues M = 256 (the two 128-row batch tiles, one per CTA) x N = 128 (both
// CTAs' R slices) MMAs: full rate, and each CTA streams only its own 128 rows.
//
// Pair (leader rank 0, peer rank 1) = PU hidden units of one direction; CTA r
// holds R^T rows [r*2PU, r*2PU+2PU) of the pair's 4PU gate columns (ordered
// gate-major: column g*PU + j = gate g of unit j) and finalizes batch tile r
// (rows b0 + 128 r ...) for all PU units.  Per step s:
//   warp 0 (both)   waits on the step counter of ITS batch tile (every pair
//                   published its units of h_{s-1} for that tile), then
//                   TMA-streams its 128 rows of h_{s-1} from the L2 ring into
//                   its own smem, completing on the LEADER's stage barrier;
//   warp 1 (leader) issues the M=256 x N=4PU x K=16 MMAs; commits multicast to
//                   both CTAs' stage-free and accumulator-full barriers;
//   warps 2..9      2 threads per batch row x PU/2 units: tcgen05.ld the row's
//                   gate pre-activations, add x W + b (K1), sigmoid / tanh,
//                   update the fp32 cell in registers, write h_s to the ring,
//                   publish, then write y and the saved activations.
// Two instantiations:
//   X3 = false (SL_PREC_BF16): PU = 32, bf16 R / h / x W / saves, both
//                directions in one launch, fast SFU activations;
//   X3 = true  (SL_PREC_FP32, fp32-class on the tensor cores): PU = 16, R^T
//                resident as hi and lo bf16 slices (R = R_hi + R_lo), h as hi
//                and lo rings, z = h_hi R_hi + h_lo R_hi + h_hi R_lo (the
//                dropped h_lo R_lo is ~2^-18 relative) accumulated in fp32
//                TMEM; fp32 x W, saves and outputs, expf / tanhf activations;
//                one direction per launch.
// Semantics as rec_tc.cu: layers.cpp:27-33, tape.cpp:1103-1135 (step),
// tape.cpp:797 (mask), tape.cpp:846 (reversal).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "profile.h"
#include "rec_tc.h"
#include "rec_tc_common.cuh"
#include "fastmath.cuh"

namespace sl {
namespace {
using namespace rtc;

// kBF16: bf16 path; kX3: fp32-class, one direction per launch, R hi + lo resident;
// kX3C: fp32-class, both directions concurrently, R_hi and R_lo streamed through
// the ring with h (a stage = [h_hi | h_lo | R_lo | R_hi] of one K chunk): with no
// resident R the shared memory holds 4 such stages instead of 2
// kBF16N: the bf16 path with 16 units per pair (narrow layers: one direction, or H small
// enough that 32-unit pairs would leave half the SMs idle), x W loaded per row
enum Mode { kBF16 = 0, kX3 = 1, kX3C = 2, kBF16N = 3 };
template <int M>
struct PairCfg {
  static constexpr bool X3 = M == kX3 || M == kX3C;
  static constexpr int kPU = M == kX3 || M == kBF16N ? 16 : 32;  // hidden units per pair
  static constexpr int kN = 4 * kPU;                       // MMA N (both CTAs' R slices)
  static constexpr int kNHalf = kN / 2;                    // R^T rows held per CTA (per precision part)
  static constexpr bool kStreamR = M != kX3;                // R (x3: hi and lo) streamed with h
  static constexpr int kRParts = M == kX3 ? 2 : 0;           // resident R copies (kX3: hi + lo)
  static constexpr int kHParts = X3 ? 2 : 1;               // h copies per stage (hi, + lo)
  static constexpr uint32_t kRloBytes = M == kX3C ? kNHalf * 128 : 0;  // streamed R_lo per 64-K chunk
  static constexpr uint32_t kRhiBytes = kStreamR ? kNHalf * 128 : 0;   // streamed R_hi per 64-K chunk
  static constexpr int kSplit = M == kX3C ? 4 : 2;         // epilogue threads per batch row
  static constexpr int kEpi = 128 * kSplit;                // epilogue threads
  static constexpr int kThreads = 64 + kEpi;
  static constexpr int kUT = kPU / kSplit;                 // units per epilogue thread
};
constexpr int kMaxStages = 8;
constexpr uint32_t kChunk = 128 * 64 * 2;   // 128 rows x 64 K bf16
constexpr uint32_t kXwGate = 128 * 32 * 2;  // x W tile of one gate: 128 rows x 32 units bf16
constexpr uint32_t kSmemMax = 227 * 1024;
constexpr int kGrpCtrs = 32;                // step counters per (direction, batch tile): one per K group

template <int M>
__host__ __device__ inline uint32_t stage_bytes_of(int kb) {
  using Cfg = PairCfg<M>;
  return (uint32_t)(Cfg::kHParts * kChunk + Cfg::kRloBytes + Cfg::kRhiBytes) * kb;
}
template <int M>
uint32_t pair_smem(int Kp, int stages, int kb) {
  using Cfg = PairCfg<M>;
  return (uint32_t)Cfg::kRParts * Cfg::kNHalf * Kp * 2 + stages * stage_bytes_of<M>(kb) + 1024;
}

#ifdef SL_EXPERIMENTS
#define TR(k)                                          \
  do {                                                 \
    if (trace) trace[s * tstride + (k)] = gtimer();    \
  } while (0)
#else
#define TR(k) \
  do {        \
  } while (0)
#endif


template <int MODE>
__global__ void __launch_bounds__(PairCfg<MODE>::kThreads, 1)
    rec_fwd_pair_kernel(const __grid_constant__ CUtensorMap tmR0, const __grid_constant__ CUtensorMap tmR1,
                        const __grid_constant__ CUtensorMap tmH0, const __grid_constant__ CUtensorMap tmH1,
                        const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmX1,
                        TcRecFwdArgs a) {
  using Cfg = PairCfg<MODE>;
  constexpr bool X3 = Cfg::X3;
  constexpr int kPU = Cfg::kPU, kN = Cfg::kN, kNHalf = Cfg::kNHalf;
  constexpr int kUT = Cfg::kUT, kEpi = Cfg::kEpi;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t r_bar, tfull_bar, tempty_bar;
  __shared__ __align__(8) uint64_t xw_full[kMaxStages];  // ring slots carrying an x W tile
  __shared__ uint32_t tmem_sh;
  __shared__ int tmax_sh, tmin_sh;

  const int pr = blockIdx.x / 2;        // pair index over the launch's directions
  const int d = pr / a.P;               // a.P = pairs per direction
  const int pair = pr % a.P;
  const int r = (int)cluster_rank();    // 0 = leader; also the batch tile
  const bool leader = r == 0;
  const int u0 = pair * kPU;
  // X3: tmH* = the hi ring, tmX* = the lo ring (x W is fp32, read by the epilogue)
  const CUtensorMap* tmR = d == 0 ? &tmR0 : &tmR1;
  const CUtensorMap* tmH = d == 0 ? &tmH0 : &tmH1;
  const CUtensorMap* tmX = d == 0 ? &tmX0 : &tmX1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t base = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - tc::smem_u32(smem_raw));
  const int nkc = a.Kp / 64;
  const uint32_t r_bytes = (uint32_t)Cfg::kRParts * kNHalf * a.Kp * 2;
  uint8_t* sR = smem;
  uint8_t* sH = smem + r_bytes;
  const uint32_t part_bytes = kChunk * a.kb;             // one precision part of h in a stage
  const uint32_t stage_bytes = stage_bytes_of<MODE>(a.kb);
  // streamed R_hi chunks sit after h (and, kX3C, after R_lo) in a stage
  const uint32_t rhi_off = Cfg::kHParts * part_bytes + a.kb * Cfg::kRloBytes;

  if (threadIdx.x == 0) {
    tmax_sh = 0;
    tmin_sh = 1 << 30;
    tc::prefetch_tmap(tmR);
    tc::prefetch_tmap(tmH);
    if (X3 || a.xw_tma) tc::prefetch_tmap(tmX);
    for (int s = 0; s < a.stages; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
      tc::mbar_init(&xw_full[s], 1);
    }
    tc::mbar_init(&r_bar, 1);
    tc::mbar_init(&tfull_bar, 1);
    tc::mbar_init(&tempty_bar, 2 * kEpi);  // both CTAs' epilogue threads (leader's copy used)
    tc::fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<kN>(&tmem_sh);
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();
  tc::fence_after_sync();
  {
    int m = 0, mn = 1 << 30;
    for (int i = threadIdx.x; i < a.B; i += blockDim.x) {
      m = max(m, (int)a.lens[i]);
      mn = min(mn, (int)a.lens[i]);
    }
    atomicMax(&tmax_sh, m);
    atomicMin(&tmin_sh, mn);
  }
  __syncthreads();
  const int Tmax = tmax_sh;
  // Equal lengths (bf16 only): step s is the same time index for every row, so
  // a step's x W rows form one TMA box per gate; it rides the h ring as one
  // extra slot per step (loaded before the step counter is even polled,
  // consumed by the epilogue) instead of 4 x 128 scattered 32 B loads.
  const bool xw_tma = !X3 && a.xw_tma && tmin_sh == Tmax;
  const int dir = a.dirsign[d];
  const uint32_t tmem = tmem_sh;
#ifdef SL_EXPERIMENTS
  // debug trace: one CTA (trace_cta >= 0) or every CTA (trace_cta < 0, buffer [grid][T][48])
  const bool trace_on = a.trace && (a.trace_cta < 0 || (int)blockIdx.x == a.trace_cta);
  const int tstride = a.trace_cta < 0 ? 48 : 16;
  unsigned long long* trace =
      trace_on ? a.trace + (a.trace_cta < 0 ? (size_t)blockIdx.x * a.T * tstride : 0) : nullptr;
#endif
  // Step counters per (direction, batch tile, K group of kb*64 hidden units):
  // a pair publishes its units of h_s to its group's counter, and a consumer
  // streams each K group as soon as THAT group is complete — the stream
  // overlaps the stragglers instead of waiting for the slowest pair.
  const int ngrp = nkc / a.kb;
  const int gunits = a.kb * 64;
  const int kc_off = pair % ngrp;
  unsigned* ctr = a.bar + (d * 2 + r) * kGrpCtrs;
  auto group_pairs = [&](int g) {  // pairs publishing into K group g
    return max(0, min(gunits / kPU, a.P - g * (gunits / kPU)));
  };

  if (warp == 0) {  // ------------------------------------------------ producer (both CTAs)
    if (lane == 0) {
      const uint32_t r_bar_l = mapa(tc::smem_u32(&r_bar), 0);
      if (leader) tc::mbar_arrive_expect_tx(&r_bar, 2 * r_bytes);
      for (int kc = 0; kc < (Cfg::kStreamR ? 0 : nkc); ++kc) {  // (kBF16 / kX3C stream R with h)
        tma_load_2d_pair(sR + (size_t)kc * kNHalf * 128, tmR, r_bar_l, kc * 64, pair * kN + r * kNHalf);
        if constexpr (MODE == kX3)  // the lo rows follow the P * kN hi rows
          tma_load_2d_pair(sR + (size_t)(nkc + kc) * kNHalf * 128, tmR, r_bar_l, kc * 64,
                           a.P * kN + pair * kN + r * kNHalf);
      }
    }
    int st = 0;  // ring position, tracked by every lane (only lane 0 issues)
    uint32_t ph = 0;
    auto advance = [&]() {
      if (++st == a.stages) {
        st = 0;
        ph ^= 1;
      }
    };
    const int kg_lane = (lane + kc_off) % ngrp;  // lane k polls the k-th group in issue order
    for (int s = 0; s < Tmax; ++s) {
      if (xw_tma) {  // this step's x W tile: 4 gate boxes [128 rows x 32 units]
        if (lane == 0) {
          tc::mbar_wait(&empty_bar[st], ph ^ 1);
          // the slot's stage-full barrier (the leader's) must still complete one
          // phase per ring pass, or the MMA issuer's parity drifts
          if (leader) tc::mbar_arrive(&full_bar[st]);
          tc::mbar_arrive_expect_tx(&xw_full[st], 4 * kXwGate);
          const int t = src_time(s, Tmax, dir);
#pragma unroll
          for (int g = 0; g < 4; ++g)
            tma_load_3d(sH + st * stage_bytes + g * kXwGate, tmX, &xw_full[st], g * a.H + u0, t,
                        a.b0 + r * 128);
        }
        advance();
      }
      const unsigned target = (unsigned)group_pairs(kg_lane) * (unsigned)s;
      bool rdy = lane >= ngrp || s == 0;
      int done = 0;
      while (done < ngrp) {
        if (!rdy) rdy = ld_acquire(ctr + kg_lane) >= target;
        const unsigned m = __ballot_sync(0xffffffffu, rdy);
        while (done < ngrp && ((m >> done) & 1u)) {
          if (lane == 0) {
            if (done == 0) TR(0);
            const int kg = (done + kc_off) % ngrp;
            tc::fence_proxy_async_global();  // the group's h (generic-proxy stores) -> TMA reads
            tc::mbar_wait(&empty_bar[st], ph ^ 1);
            if (leader) tc::mbar_arrive_expect_tx(&full_bar[st], 2 * stage_bytes);
            const uint32_t fb = mapa(tc::smem_u32(&full_bar[st]), 0);
            if constexpr (Cfg::kStreamR)  // this group's R chunks (no dependency on the step)
              for (int j = 0; j < a.kb; ++j) {
                if constexpr (MODE == kX3C)
                  tma_load_2d_pair(sH + st * stage_bytes + 2 * part_bytes + j * Cfg::kRloBytes, tmR, fb,
                                   (kg * a.kb + j) * 64, a.P * kN + pair * kN + r * kNHalf);
                tma_load_2d_pair(sH + st * stage_bytes + rhi_off + j * Cfg::kRhiBytes, tmR, fb,
                                 (kg * a.kb + j) * 64, pair * kN + r * kNHalf);
              }
            tma_load_4d_pair(sH + st * stage_bytes, tmH, fb, 0, (a.b0 + r * 128) / 8, kg * a.kb * 8, s & 1);
            if constexpr (X3)
              tma_load_4d_pair(sH + st * stage_bytes + part_bytes, tmX, fb, 0, (a.b0 + r * 128) / 8,
                               kg * a.kb * 8, s & 1);
          }
          advance();
          ++done;
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ------------------------------------ MMA issuer (leader)
      constexpr uint32_t idesc = tc::make_idesc(256, kN, 1, false, false);
      tc::mbar_wait(&r_bar, 0);
      int st = 0;
      uint32_t ph = 0;
      for (int s = 0; s < Tmax; ++s) {
        if (xw_tma && ++st == a.stages) {  // the x W slot belongs to the epilogue
          st = 0;
          ph ^= 1;
        }
        tc::mbar_wait(&tempty_bar, (s & 1) ^ 1);
        tc::fence_after_sync();
        for (int kq = 0; kq < ngrp; ++kq) {
          const int kg = (kq + kc_off) % ngrp;
          tc::mbar_wait(&full_bar[st], ph);
          tc::fence_after_sync();
          if (kq == 0) TR(1);
          for (int j = 0; j < a.kb; ++j) {
            const int kc = kg * a.kb + j;
            const uint32_t sa = base + r_bytes + st * stage_bytes + j * kChunk;
            // R_hi: resident, or (kX3C) the stage's chunk (same SW128 rows)
            const uint32_t sb = Cfg::kStreamR ? base + r_bytes + st * stage_bytes + rhi_off + j * Cfg::kRhiBytes
                                              : base + (uint32_t)kc * kNHalf * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ah = tc::make_sdesc_noswz(sa + k * 2 * 2048, 2048, 128);
              const uint64_t bh = tc::make_sdesc(sb + k * 32, 0, 1024);
              mma_f16_pair(tmem, ah, bh, idesc, (kq | j | k) != 0);
              if constexpr (X3) {
                const uint64_t al = tc::make_sdesc_noswz(sa + part_bytes + k * 2 * 2048, 2048, 128);
                const uint32_t sbl = MODE == kX3C
                                         ? base + r_bytes + st * stage_bytes + 2 * part_bytes + j * Cfg::kRloBytes
                                         : sb + (uint32_t)nkc * kNHalf * 128;
                const uint64_t bl = tc::make_sdesc(sbl + k * 32, 0, 1024);
                mma_f16_pair(tmem, al, bh, idesc, true);  // h_lo R_hi
                mma_f16_pair(tmem, ah, bl, idesc, true);  // h_hi R_lo
              }
            }
          }
          mma_commit_pair(&empty_bar[st]);
          if (++st == a.stages) {
            st = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair(&tfull_bar);
      }
    }
  } else {  // ------------------------------------------------------ epilogue (both CTAs)
    const int e = warp - 2;
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int part = e / 4;          // which kUT-unit slice of the pair's units
    const int rl = q * 32 + lane;
    const int row = a.b0 + r * 128 + rl;
    const bool valid_row = row < a.B;
    const int len = valid_row ? a.lens[row] : 0;
    const int H = a.H, T = a.T;
    const int lo = part * kUT;
    const int ut0 = u0 + lo;
    const int nu = max(0, min(kUT, H - ut0));
    const int gdir = X3 ? a.dir0 + d : d;  // global direction: y columns, final-state rows
    __nv_bfloat16* hb = a.hbuf[d];
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + lo;
    const uint32_t tempty_l = mapa(tc::smem_u32(&tempty_bar), 0);
    const bool vec = (H % 8) == 0 && (a.xw_ld % 8) == 0;
    float cst[kUT], hst[kUT];
#pragma unroll
    for (int u = 0; u < kUT; ++u) cst[u] = hst[u] = 0.f;

    // x W + b (K1 output) of a step, prefetched one step ahead
    uint32_t xw_par = 0;  // per ring slot: parity of its next x W use
    Bf16Vec<kUT> xv[4];   // bf16 path
    float xf[4][kUT];     // x3 path
    auto load_xw = [&](int st) {
      if constexpr (X3) {
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int u = 0; u < kUT; ++u) xf[g][u] = 0.f;
        if (valid_row && st < len) {
          const float* xr = a.xwf[d] + ((size_t)row * T + src_time(st, len, dir)) * a.xw_ld + ut0;
          const bool v4 = (H % 4) == 0 && (a.xw_ld % 4) == 0;
#pragma unroll
          for (int g = 0; g < 4; ++g) load_f32<kUT>(xr + (size_t)g * H, xf[g], nu, v4);
        }
      } else {
        if (xw_tma) {
          const int slot = (int)(((int64_t)st * (ngrp + 1)) % a.stages);
          tc::mbar_wait(&xw_full[slot], (xw_par >> slot) & 1);
          xw_par ^= 1u << slot;
          const uint8_t* tile = sH + slot * stage_bytes + rl * 64;
          const uint32_t sw = (rl >> 1) & 3;  // SWIZZLE_64B: 16 B chunk ^= address bits [7:8]
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint4 q0 = *reinterpret_cast<const uint4*>(tile + g * kXwGate + ((2 * part) ^ sw) * 16);
            const uint4 q1 = *reinterpret_cast<const uint4*>(tile + g * kXwGate + ((2 * part + 1) ^ sw) * 16);
            xv[g].w[0] = q0.x, xv[g].w[1] = q0.y, xv[g].w[2] = q0.z, xv[g].w[3] = q0.w;
            xv[g].w[4] = q1.x, xv[g].w[5] = q1.y, xv[g].w[6] = q1.z, xv[g].w[7] = q1.w;
          }
          named_sync(2, kEpi);  // every epilogue thread has its slice: the slot is free
          if (e == 0 && lane == 0) tc::mbar_arrive(&empty_bar[slot]);
          return;
        }
        if (valid_row && st < len) {
          const __nv_bfloat16* xr = a.xw[d] + ((size_t)row * T + src_time(st, len, dir)) * a.xw_ld + ut0;
#pragma unroll
          for (int g = 0; g < 4; ++g) xv[g].load(xr + g * H, nu, vec);
        }
      }
    };
    load_xw(0);
    for (int s = 0; s < Tmax; ++s) {
      const bool active = valid_row && s < len;
      const int t = active ? src_time(s, len, dir) : s;
      const size_t pos = (size_t)row * T + t;
      if (lane == 0) tc::mbar_wait_sleep(&tfull_bar, s & 1);  // one poller per warp
      __syncwarp();
      tc::fence_after_sync();
      float z[4 * kUT];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float v[kUT];
        tmem_ld_cols<kUT>(tbase + g * kPU, v);
#pragma unroll
        for (int u = 0; u < kUT; ++u) z[g * kUT + u] = v[u];
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote_relaxed(tempty_l, 32);  // accumulator may be overwritten

      if (valid_row) {
        if (active) {
          if constexpr (X3) {  // 1/(1+exp(-z)), tanh (tape.cpp:1119-1135): two-MUFU forms, paired fp32
#pragma unroll
            for (int u = 0; u < kUT; u += 2) {
              using fm::add2;
              const float2 gi = fm::sigmoid2(add2(f2(z[u], z[u + 1]), f2(xf[0][u], xf[0][u + 1])));
              const float2 gf = fm::sigmoid2(add2(f2(z[kUT + u], z[kUT + u + 1]), f2(xf[1][u], xf[1][u + 1])));
              const float2 gg = fm::tanh2(add2(f2(z[2 * kUT + u], z[2 * kUT + u + 1]), f2(xf[2][u], xf[2][u + 1])));
              const float2 go = fm::sigmoid2(add2(f2(z[3 * kUT + u], z[3 * kUT + u + 1]), f2(xf[3][u], xf[3][u + 1])));
              z[u] = gi.x, z[u + 1] = gi.y;
              z[kUT + u] = gf.x, z[kUT + u + 1] = gf.y;
              z[2 * kUT + u] = gg.x, z[2 * kUT + u + 1] = gg.y;
              z[3 * kUT + u] = go.x, z[3 * kUT + u + 1] = go.y;
              const float2 cn = fm::fma2(gf, f2(cst[u], cst[u + 1]), fm::mul2(gi, gg));  // c = f c + i g
              cst[u] = cn.x, cst[u + 1] = cn.y;
              const float2 h = fm::mul2(go, fm::tanh2(cn));                              // h = o tanh(c)
              hst[u] = h.x, hst[u + 1] = h.y;
            }
          } else {
#pragma unroll
            for (int u = 0; u < kUT; u += 2) {  // two units per paired-fp32 instruction
              const float2 gi = sigmoid2(add2(f2(z[u], z[u + 1]), bf16x2_f2(xv[0].w[u / 2])));
              const float2 gf = sigmoid2(add2(f2(z[kUT + u], z[kUT + u + 1]), bf16x2_f2(xv[1].w[u / 2])));
              const float2 gg = tanh2(add2(f2(z[2 * kUT + u], z[2 * kUT + u + 1]), bf16x2_f2(xv[2].w[u / 2])));
              const float2 go = sigmoid2(add2(f2(z[3 * kUT + u], z[3 * kUT + u + 1]), bf16x2_f2(xv[3].w[u / 2])));
              z[u] = gi.x, z[u + 1] = gi.y;
              z[kUT + u] = gf.x, z[kUT + u + 1] = gf.y;
              z[2 * kUT + u] = gg.x, z[2 * kUT + u + 1] = gg.y;
              z[3 * kUT + u] = go.x, z[3 * kUT + u + 1] = go.y;
              const float2 cn = fma2(gf, f2(cst[u], cst[u + 1]), mul2(gi, gg));  // c = f c + i g
              cst[u] = cn.x, cst[u + 1] = cn.y;
              const float2 h = mul2(go, tanh2(cn));                             // h = o tanh(c)
              hst[u] = h.x, hst[u + 1] = h.y;
            }
          }
        }
        // only h_s is on the cross-CTA critical path
        // h ring in the interleaved layout (rec_tc.h dz_ring_off): 8-unit chunks of
        // consecutive rows are contiguous, so each warp store covers 512 B
#pragma unroll
        for (int c = 0; c < kUT; c += 8) {
          const size_t off = dz_ring_off((s + 1) & 1, row, ut0 + c, dz_ring_bp(a.B), a.Kp);
          store_bf16<8>(hb + off, hst + c, max(0, min(8, nu - c)));
          if constexpr (X3) {  // h_lo = h - bf16(h): exact in fp32, rounded to bf16
            float hl[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) hl[u] = hst[c + u] - __bfloat162float(__float2bfloat16_rn(hst[c + u]));
            store_bf16<8>(a.hbuf_lo[d] + off, hl, max(0, min(8, nu - c)));
          }
        }
      }
      named_sync(1, kEpi);
      if (e == 0 && lane == 0) {
        tc::fence_proxy_async_global();
        red_release_gpu(ctr + u0 / gunits, 1u);  // my K group's counter
        TR(6);
      }
      // take the next step's x W tile out of its ring slot now (before the
      // saves): a slot held through the saves starves this CTA's next h
      // stream of a stage, and a late CTA would fall further behind each step
      if (s + 1 < Tmax) load_xw(s + 1);
      if (valid_row) {
        float zero[kUT];
#pragma unroll
        for (int u = 0; u < kUT; ++u) zero[u] = 0.f;
        if (active) {
          if constexpr (X3) {
            if (a.gatesf[d]) {
#pragma unroll
              for (int g = 0; g < 4; ++g)
                store_f32<kUT>(a.gatesf[d] + gate_save_off(s, g, row, a.B, H, ut0), z + g * kUT, nu);
            }
            if (a.y) store_f32<kUT>(a.y + pos * a.y_ld + (size_t)gdir * H + ut0, hst, nu);
            if (a.yimg) store_split<kUT>(a.yimg + pos * a.yimg_ld + (size_t)gdir * H + ut0, a.yimg_lo, hst, nu);
            if (a.gatesf[d]) {  // the saved (c, h)_{prev} of each step, off the critical path
              if (s == 0) {
                store_f32<kUT>(a.cprevf[d] + cprev_save_off(0, row, a.B, H, ut0), zero, nu);
                store_split<kUT>(a.hprevi[d] + pos * a.hprev_ld + ut0, a.hprevi_lo, zero, nu);
              }
              if (s + 1 < len) {
                const size_t pn = (size_t)row * T + src_time(s + 1, len, dir);
                store_f32<kUT>(a.cprevf[d] + cprev_save_off(s + 1, row, a.B, H, ut0), cst, nu);
                store_split<kUT>(a.hprevi[d] + pn * a.hprev_ld + ut0, a.hprevi_lo, hst, nu);
              }
            }
          } else {
            const bool save = a.gates[d] != nullptr;
            if (save) {
#pragma unroll
              for (int g = 0; g < 4; ++g)
                store_bf16<kUT>(a.gates[d] + gate_save_off(s, g, row, a.B, H, ut0), z + g * kUT, nu);
            }
            if (a.y) store_f32<kUT>(a.y + pos * a.y_ld + (size_t)d * H + ut0, hst, nu);
            if (a.ybf) store_bf16<kUT>(a.ybf + pos * a.ybf_ld + (size_t)d * H + ut0, hst, nu);
            if (save) {  // the saved (c, h)_{prev} of each step, written off the critical path:
              // zeros at the first step, (c_s, h_s) at the position of step s + 1
              if (s == 0) {
                store_bf16<kUT>(a.cprev[d] + cprev_save_off(0, row, a.B, H, ut0), zero, nu);
                store_bf16<kUT>(a.hprev[d] + pos * a.hprev_ld + ut0, zero, nu);
              }
              if (s + 1 < len) {
                const size_t pn = (size_t)row * T + src_time(s + 1, len, dir);
                store_bf16<kUT>(a.cprev[d] + cprev_save_off(s + 1, row, a.B, H, ut0), cst, nu);
                store_bf16<kUT>(a.hprev[d] + pn * a.hprev_ld + ut0, hst, nu);
              }
            }
          }
        } else {  // padded position t == s: zero output (tape.cpp:797), frozen state
          if (a.y) store_f32<kUT>(a.y + pos * a.y_ld + (size_t)gdir * H + ut0, zero, nu);
          if constexpr (X3) {
            if (a.yimg) store_split<kUT>(a.yimg + pos * a.yimg_ld + (size_t)gdir * H + ut0, a.yimg_lo, zero, nu);
            if (a.gatesf[d]) store_split<kUT>(a.hprevi[d] + pos * a.hprev_ld + ut0, a.hprevi_lo, zero, nu);
          } else {
            if (a.ybf) store_bf16<kUT>(a.ybf + pos * a.ybf_ld + (size_t)d * H + ut0, zero, nu);
            if (a.gates[d]) store_bf16<kUT>(a.hprev[d] + pos * a.hprev_ld + ut0, zero, nu);
          }
        }
      }
    }
    if (valid_row) {  // positions beyond the longest sequence, final states
      float zero[kUT];
#pragma unroll
      for (int u = 0; u < kUT; ++u) zero[u] = 0.f;
      for (int s = Tmax; s < T; ++s) {
        const size_t pos = (size_t)row * T + s;
        if (a.y) store_f32<kUT>(a.y + pos * a.y_ld + (size_t)gdir * H + ut0, zero, nu);
        if constexpr (X3) {
          if (a.yimg) store_split<kUT>(a.yimg + pos * a.yimg_ld + (size_t)gdir * H + ut0, a.yimg_lo, zero, nu);
          if (a.gatesf[d]) store_split<kUT>(a.hprevi[d] + pos * a.hprev_ld + ut0, a.hprevi_lo, zero, nu);
        } else {
          if (a.ybf) store_bf16<kUT>(a.ybf + pos * a.ybf_ld + (size_t)d * H + ut0, zero, nu);
          if (a.gates[d]) store_bf16<kUT>(a.hprev[d] + pos * a.hprev_ld + ut0, zero, nu);
        }
      }
#pragma unroll
      for (int u = 0; u < kUT; ++u) {
        if (u >= nu) continue;
        if (a.h_last) a.h_last[((size_t)gdir * a.B + row) * H + ut0 + u] = hst[u];
        if (a.c_last) a.c_last[((size_t)gdir * a.B + row) * H + ut0 + u] = cst[u];
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();  // the peer's MMAs / arrivals are done before TMEM and smem go away
  if (warp == 1) tmem_dealloc_pair<kN>(tmem);
}
#undef TR

// RT rows [pair * 4UC + g * UC + j] = column g*H + pair*UC + j of R (the x3 pair
// kernels' order), lo rows at + P * 4UC: (R - bf16(R)) rounded to bf16.  One block
// per (pair, gate) x 64 k, 16 B stores along k; R is read once for both parts.
template <int UC>
__global__ void __launch_bounds__(256) pack_rt_x3_kernel(const float* __restrict__ R, int H, int Kp, int P,
                                                         __nv_bfloat16* __restrict__ RT) {
  __shared__ float tile[64][UC + 1];
  const int cg = blockIdx.x;  // (pair, gate)
  const int cta = cg / 4, g = cg % 4;
  const int k0 = blockIdx.y * 64;
  const int c0 = g * H + cta * UC;
  const int units_here = min(UC, H - cta * UC);
  for (int e = threadIdx.x; e < 64 * UC; e += 256) {
    const int i = e / UC, j = e % UC;
    const int k = k0 + i;
    tile[i][j] = (k < H && j < units_here) ? __ldg(R + (size_t)k * 4 * H + c0 + j) : 0.f;
  }
  __syncthreads();
  const size_t lo_off = (size_t)P * 4 * UC * Kp;
  for (int e = threadIdx.x; e < UC * 8; e += 256) {
    const int j = e / 8, kq = (e % 8) * 8;
    float f[8], l[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      f[u] = tile[kq + u][j];
      l[u] = f[u] - __bfloat162float(__float2bfloat16_rn(f[u]));
    }
    __nv_bfloat16* dst = RT + ((size_t)cta * 4 * UC + g * UC + j) * Kp + k0 + kq;
    *reinterpret_cast<uint4*>(dst) = pack8_bf16(f);
    *reinterpret_cast<uint4*>(dst + lo_off) = pack8_bf16(l);
  }
}

template <int MODE>
void launch_pair(const TcRecFwdArgs& a0, const CUtensorMap* tr, const CUtensorMap* th, const CUtensorMap* tx,
                 cudaStream_t stream) {
  TcRecFwdArgs a = a0;
  const uint32_t smem = pair_smem<MODE>(a.Kp, a.stages, a.kb);
  auto kern = rec_fwd_pair_kernel<MODE>;
  SL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CUtensorMap r0 = tr[0], r1 = tr[a.nd > 1 ? 1 : 0], h0 = th[0], h1 = th[a.nd > 1 ? 1 : 0];
  CUtensorMap x0 = tx[0], x1 = tx[a.nd > 1 ? 1 : 0];
  unsigned* bar0 = a.bar;
  for (int b0 = 0; b0 < a.B; b0 += 256) {  // batch chunks of up to two 128-row tiles
    a.b0 = b0;
    a.bar = bar0 + kBarPerChunk * (b0 / 256);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * a.P * a.nd);
    cfg.blockDim = dim3(PairCfg<MODE>::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident, or fail loudly
    attrs[1].val.cooperative = 1;
    cfg.attrs = attrs;
    // SL_NO_COOP=1 (ncu only: it cannot launch cooperative cluster kernels; the
    // grid of <= #SMs CTAs at 1 CTA/SM is still co-resident in practice)
    static const bool no_coop = getenv("SL_NO_COOP") != nullptr;
    cfg.numAttrs = no_coop ? 1 : 2;
    SL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, r0, r1, h0, h1, x0, x1, a));
    count_launch();
  }
}

// interleaved h ring {8 rows x 8 k, 8-row groups, K chunks of 8, slot}: 128 B TMA
// rows; a box is 128 rows x kb*64 K in the SWIZZLE_NONE core-matrix layout
CUtensorMap ring_map(const __nv_bfloat16* ring, int B, int Kp, int kb) {
  const int Bp = dz_ring_bp(B);
  cuuint64_t hd[4] = {64, (cuuint64_t)Bp / 8, (cuuint64_t)Kp / 8, 2};
  cuuint64_t hs[3] = {128, (cuuint64_t)Bp * 16, (cuuint64_t)Kp / 8 * Bp * 16};
  cuuint32_t hbx[4] = {64, 16, (cuuint32_t)kb * 8, 1};
  return tmap(ring, 4, hd, hs, hbx, CU_TENSOR_MAP_SWIZZLE_NONE);
}

}  // namespace

bool tc_rec_fwd_pair_fits(int H, int nd, int sms) {
  const int P = (int)ceil_div(H, PairCfg<kBF16>::kPU);
  const int Kp = (int)round_up(H, 64);
  return (int64_t)2 * P * nd <= sms && pair_smem<kBF16>(Kp, 2, 2) <= kSmemMax;
}

int tc_rec_fwd_pair_units(int H, int nd, int sms) {
  // 16 units per pair when 32-unit pairs would cover at most half the SMs and the
  // narrow grid still fits (e.g. one direction of H = 1024: 128 CTAs instead of 64);
  // small layers keep 32 (their steps are latency-, not MMA-bound)
  const int P16 = (int)ceil_div(H, PairCfg<kBF16N>::kPU);
  const int Kp = (int)round_up(H, 64);
  if (H >= 512 && (int64_t)2 * P16 * nd <= sms && pair_smem<kBF16N>(Kp, 2, 2) <= kSmemMax &&
      Kp / 64 / 2 <= kGrpCtrs)
    return 16;
  return 32;
}

void rec_fwd_pair(const TcRecFwdArgs& a0, const TcFwdShape& sh, __nv_bfloat16* const* RT,
                  cudaStream_t stream) {
  const bool narrow = sh.U == PairCfg<kBF16N>::kPU;
  const int kN = 4 * sh.U, kNHalf = kN / 2;
  TcRecFwdArgs a = a0;
  a.U = sh.U;
  a.P = sh.P;
  a.Kp = sh.Kp;
  CUtensorMap tr[2], th[2], tx[2];
  a.kb = (a.Kp / 64) % 2 == 0 ? 2 : 1;
  // x W tiles by TMA: 3-D view {columns, T, B} of the bf16 K1 output, one box
  // per gate of [128 rows x 32 units], 64 B swizzle (conflict-free epilogue reads);
  // the narrow kernel loads its 16-unit slices per row instead
  a.xw_tma = !narrow && kChunk * a.kb >= 4 * kXwGate && (a.xw_ld * 2) % 16 == 0;
  for (int k = 0; k < a.nd; ++k) a.xw_tma = a.xw_tma && ((uintptr_t)a.xw[k] & 15) == 0;
  for (int k = 0; k < a.nd; ++k) {
    if (a.xw_tma) {
      cuuint64_t xd[3] = {(cuuint64_t)a.xw_ld, (cuuint64_t)a.T, (cuuint64_t)a.B};
      cuuint64_t xs[2] = {(cuuint64_t)a.xw_ld * 2, (cuuint64_t)a.xw_ld * 2 * a.T};
      cuuint32_t xb[3] = {32, 1, 128};
      tx[k] = tmap(a.xw[k], 3, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_64B);
    } else {
      tx[k] = CUtensorMap{};
    }
    cuuint64_t rd[2] = {(cuuint64_t)a.Kp, (cuuint64_t)a.P * kN};
    cuuint64_t rs[1] = {(cuuint64_t)a.Kp * 2};
    cuuint32_t rb[2] = {64, (cuuint32_t)kNHalf};
    tr[k] = tmap(RT[k], 2, rd, rs, rb);
    th[k] = ring_map(a.hbuf[k], a.B, a.Kp, a.kb);
  }
  a.stages = 0;
  for (int st = kMaxStages; st >= 2 && !a.stages; --st)
    if ((narrow ? pair_smem<kBF16N>(a.Kp, st, a.kb) : pair_smem<kBF16>(a.Kp, st, a.kb)) <= kSmemMax) a.stages = st;
  SL_REQUIRE(a.stages >= 2, SL_ERR_UNSUPPORTED, "rec_fwd_pair: R slice does not fit in shared memory");
  SL_REQUIRE(a.Kp / 64 / a.kb <= kGrpCtrs && 4 * kGrpCtrs <= kBarPerChunk, SL_ERR_UNSUPPORTED,
             "rec_fwd_pair: too many K groups for the step counters");
  if (narrow) launch_pair<kBF16N>(a, tr, th, tx, stream);
  else launch_pair<kBF16>(a, tr, th, tx, stream);
}

TcFwdShape tc_rec_fwd_x3_shape(int H, int sms, int nd) {
  if (nd == 2) {  // both directions concurrently (R_lo streamed), when the grid fits
    using Cc = PairCfg<kX3C>;
    const int P = (int)ceil_div(H, Cc::kPU);
    const int Kp = (int)round_up(H, 64);
    if ((int64_t)4 * P <= sms && pair_smem<kX3C>(Kp, 2, 1) <= kSmemMax && Kp / 64 <= kGrpCtrs) {
      TcFwdShape sh{1, Cc::kPU, P, Kp};
      sh.pair = 2;  // kX3C
      return sh;
    }
  }
  using Cfg = PairCfg<kX3>;
  const int P = (int)ceil_div(H, Cfg::kPU);
  const int Kp = (int)round_up(H, 64);
  if ((int64_t)2 * P > sms || pair_smem<kX3>(Kp, 2, 1) > kSmemMax || Kp / 64 > kGrpCtrs)
    return TcFwdShape{0, 0, 0, 0};
  TcFwdShape sh{1, Cfg::kPU, P, Kp};
  sh.pair = 1;  // kX3: one direction per launch
  return sh;
}

size_t tc_rec_x3_pack_elems(const TcFwdShape& sh) { return (size_t)2 * sh.P * 4 * sh.U * sh.Kp; }

void tc_rec_x3_pack(const float* R, int H, const TcFwdShape& sh, __nv_bfloat16* RT, cudaStream_t stream) {
  const dim3 grid((unsigned)sh.P * 4, (unsigned)(sh.Kp / 64));
  if (sh.U == 32) pack_rt_x3_kernel<32><<<grid, 256, 0, stream>>>(R, H, sh.Kp, sh.P, RT);
  else pack_rt_x3_kernel<16><<<grid, 256, 0, stream>>>(R, H, sh.Kp, sh.P, RT);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

// x3: sh.pair == 1 -> one direction (a.nd == 1, RT[0]); sh.pair == 2 -> both (a.nd == 2)
void rec_fwd_pair_x3(const TcRecFwdArgs& a0, const TcFwdShape& sh, const __nv_bfloat16* const* RT,
                     cudaStream_t stream) {
  TcRecFwdArgs a = a0;
  const bool conc = sh.pair == 2;
  SL_REQUIRE(conc ? a.nd == 2 : a.nd == 1, SL_ERR_INVALID_ARGUMENT, "rec_fwd_pair_x3: direction count");
  a.U = sh.U;
  a.P = sh.P;
  a.Kp = sh.Kp;
  a.kb = 1;
  a.xw_tma = 0;
  const int kN = 4 * sh.U, kNHalf = kN / 2;
  CUtensorMap tr[2], th[2], tl[2];
  for (int k = 0; k < a.nd; ++k) {
    cuuint64_t rd[2] = {(cuuint64_t)a.Kp, (cuuint64_t)2 * a.P * kN};
    cuuint64_t rs[1] = {(cuuint64_t)a.Kp * 2};
    cuuint32_t rb[2] = {64, (cuuint32_t)kNHalf};
    tr[k] = tmap(RT[k], 2, rd, rs, rb);
    th[k] = ring_map(a.hbuf[k], a.B, a.Kp, a.kb);
    tl[k] = ring_map(a.hbuf_lo[k], a.B, a.Kp, a.kb);
  }
  a.stages = 0;
  for (int st = kMaxStages; st >= 2 && !a.stages; --st)
    if ((conc ? pair_smem<kX3C>(a.Kp, st, a.kb) : pair_smem<kX3>(a.Kp, st, a.kb)) <= kSmemMax) a.stages = st;
  SL_REQUIRE(a.stages >= 2, SL_ERR_UNSUPPORTED, "rec_fwd_pair_x3: R slice does not fit in shared memory");
  if (conc) launch_pair<kX3C>(a, tr, th, tl, stream);
  else launch_pair<kX3>(a, tr, th, tl, stream);
}

}  // namespace sl
