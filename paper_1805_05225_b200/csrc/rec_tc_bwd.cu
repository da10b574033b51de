// K3 — persistent tensor-core BPTT: the mirror of K2.
//
// One launch runs all T steps of the launch's directions backwards.  CTA c of
// direction d owns hidden units [c*U, c*U+U): it keeps R[units, :] (the rows
// of R feeding those units' h, all 4H gate columns, bf16, K-major) resident in
// shared memory, and per step s (descending):
//   warp 0      waits for every CTA of the direction to publish DZ_{s+1}, then
//               TMA-streams DZ_{s+1} [128-row batch tile x 64 gate cols] bf16
//               from the L2-resident ring buffer;
//   warp 1      tcgen05.mma: dh_rec[:, units] = DZ_{s+1} . R[units, :]^T
//               (tape.cpp:1182-1189, the per-step GEMM GH = DZ R^T);
//   warps 2..   one/two threads per batch row: gh = dy + dh_rec, the cell-gate
//               adjoint of tape.cpp:1157-1170 with the carried dc, writing
//               DZ_s to the ring (for the next step) and to the [B*T, 8H]
//               DZ matrix the hoisted K4 GEMMs consume.
// As in K2 the two 128-row batch tiles are independent recurrences with their
// own step counters, so one tile's epilogue overlaps the other's MMAs.
// Two instantiations:
//   X3 = false (SL_PREC_BF16): bf16 R / DZ / saves, both directions per launch;
//   X3 = true  (SL_PREC_FP32, fp32-class): R resident as hi and lo bf16 slices,
//              DZ as hi and lo rings, dh = DZ_hi R_hi^T + DZ_lo R_hi^T +
//              DZ_hi R_lo^T accumulated in fp32 TMEM, fp32 partial exchange
//              between the K-split CTAs, fp32 saves (K2 x3) and fp32 DZ for
//              K4; one direction per launch.
#include <cstdlib>
#include <type_traits>

#include "profile.h"
#include "rec_tc.h"
#include "rec_tc_common.cuh"
#include "fastmath.cuh"

namespace sl {
namespace {
using namespace rtc;

constexpr int kStages = 8;  // ring slots (kBF16 / kX3 use at most 6)
constexpr int kBoxCtrs = 128;  // step counters per (direction, batch tile): one per DZ box
constexpr uint32_t kTile = 128 * 64 * 2;  // 16 KB A tile
constexpr uint32_t kSmemMax = 227 * 1024;

__host__ __device__ constexpr int nb_of(int C, int U) { return C * U < 16 ? 16 : C * U; }

// kBF16: bf16 R / DZ, both directions per launch; kX3: fp32-class, one direction per
// launch, R hi + lo resident; kX3C: fp32-class, both directions per launch, R_hi and
// R_lo streamed with DZ (a stage = [DZ_hi | DZ_lo | R_lo | R_hi] of 32 K): with no
// resident R the shared memory holds 8 such stages, and the per-step stream (DZ of
// both tiles plus the CTA's R slice, ~1.5 MB) is no longer latency-bound on 3 slots
enum BwdMode { kBF16 = 0, kX3 = 1, kX3C = 2 };

// K elements of the DZ ring a stage carries: 64 * kb, or 32 for kX3C
__host__ __device__ inline int stage_k(int mode, int kb) { return mode == kX3C ? 32 : 64 * kb; }
// kBF16 and kX3C stream the CTA's R slice with DZ (kX3C: hi and lo); kX3 keeps it resident
__host__ __device__ inline bool stream_r(int mode) { return mode != kX3; }
__host__ __device__ inline uint32_t bwd_stage_bytes(int mode, int NB, int kb) {
  const int kk = stage_k(mode, kb);
  return (uint32_t)(mode == kBF16 ? 1 : 2) * 128 * kk * 2 + (stream_r(mode) ? (mode == kX3C ? 2u : 1u) * NB * kk * 2 : 0u);
}
uint32_t bwd_smem_m(int mode, int C, int U, int Kc, int stages, int kb) {
  const int NB = nb_of(C, U);
  const uint32_t rparts = mode == kX3 ? 2 : 0;  // resident R parts
  // [C-1 slots][128 rows][U] partials from the peers (bf16, x3: fp32): one buffer per
  // batch tile, or (kX3C) one buffer the two tiles use in turn
  const uint32_t recv = C > 1 ? (uint32_t)(mode == kX3C ? 1 : 2) * (C - 1) * U * 128 * (mode == kBF16 ? 2 : 4) : 0;
  return rparts * (uint32_t)NB * Kc * 2 + (uint32_t)stages * bwd_stage_bytes(mode, NB, kb) + recv + 1024;
}
// (bf16 shape probing: two 16 KB chunks per stage unit)
uint32_t bwd_smem(int C, int U, int Kc, int stages) { return bwd_smem_m(kBF16, C, U, Kc, stages, 2); }

// TMA descriptors of one launch, per direction: R (resident rows; kX3: hi then lo),
// the DZ ring (hi), the DZ_lo ring (x3), R_lo as 8-K core-matrix boxes (kX3C)
struct BwdMaps {
  CUtensorMap R[2], Z[2], Zlo[2], Rlo[2], Rhi[2];
};

// C   CTAs per cluster = K-split factor over the 4H gate columns of DZ
// U   hidden units each CTA finalizes (the cluster owns C*U units)
// MT  128-row batch tiles per launch
// SPLIT epilogue threads per batch row (UT = U / SPLIT units each).  (One
// thread per row for U = 16 — 32 B segments, half the requests — measured
// slower: the per-thread math and stores then sit on the critical path.)
constexpr int bwd_split(int U) { return U >= 8 ? 2 : 1; }

template <int C, int U, int MT, int MODE, int SPLIT = bwd_split(U), int UT = U / SPLIT>
__global__ void __launch_bounds__(64 + 128 * MT * SPLIT, 1)
    rec_bwd_tc_kernel(const __grid_constant__ BwdMaps mp, TcRecBwdArgs a) {
  constexpr bool X3 = MODE != kBF16;
  constexpr int NB = nb_of(C, U);  // MMA N: the cluster's units
  constexpr int kEpiTile = 128 * SPLIT;
  using RecvT = typename std::conditional<X3, float, __nv_bfloat16>::type;
  constexpr uint32_t kRecvBytes = (uint32_t)(C - 1) * 128 * U * sizeof(RecvT);  // per tile and use
  constexpr uint32_t kTmemCols = (MT * NB <= 32) ? 32 : (MT * NB <= 64) ? 64 : (MT * NB <= 128) ? 128 : 256;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t r_bar, tfull_bar[MT], tempty_bar[MT];
  __shared__ __align__(8) uint64_t recv_full[MT], free_bar[MT][C];
  __shared__ uint32_t tmem_sh;
  __shared__ int tmax_sh;

  const int d = blockIdx.x / a.P;
  const int cta = blockIdx.x % a.P;        // CTA index within the direction
  const int r = C > 1 ? (int)cluster_rank() : 0;  // K-slice of this CTA
  const int cl = cta / C;                  // cluster index within the direction
  const int u0 = cl * C * U + r * U;       // first unit this CTA finalizes
  const int Kc = a.Kz / C;
  const CUtensorMap* tmR = &mp.R[d];
  const CUtensorMap* tmZ = &mp.Z[d];
  const CUtensorMap* tmZl = &mp.Zlo[d];
  const CUtensorMap* tmRl = &mp.Rlo[d];
  const CUtensorMap* tmRh = &mp.Rhi[d];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t base = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - tc::smem_u32(smem_raw));
  const uint32_t r_part = (uint32_t)NB * Kc * 2;  // one precision part of the R slice
  const uint32_t r_bytes = r_part * (MODE == kX3 ? 2 : 0);  // resident R (kX3 only)
  uint8_t* sR = smem;
  uint8_t* sA = smem + r_bytes;
  const int kst = stage_k(MODE, a.kb);           // DZ columns per stage (= per TMA box)
  const uint32_t part_bytes = 128u * kst * 2;    // one precision part of DZ in a stage
  const uint32_t stage_bytes = bwd_stage_bytes(MODE, NB, a.kb);
  // the streamed R_hi rows follow DZ (and, kX3C, R_lo) in a stage
  const uint32_t rhi_off = (X3 ? 2 : 1) * part_bytes + (MODE == kX3C ? (uint32_t)NB * kst * 2 : 0u);
  // [MT][C-1 slots][128 rows][U] partials from the peers: one buffer per
  // batch tile (a shared buffer would couple the two tiles' recurrences through
  // its free/full handshake) and row-major, so each sender thread writes its
  // row's slice with 16 B DSMEM stores
  RecvT* recv = reinterpret_cast<RecvT*>(sA + a.stages * stage_bytes);
  const int nkc = Kc / 64;

  if (threadIdx.x == 0) {
    tmax_sh = 0;
    tc::prefetch_tmap(tmR);
    tc::prefetch_tmap(tmZ);
    if (X3) tc::prefetch_tmap(tmZl);
    if (MODE == kX3C) tc::prefetch_tmap(tmRl);
    if (MODE != kX3) tc::prefetch_tmap(tmRh);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    tc::mbar_init(&r_bar, 1);
    for (int m = 0; m < MT; ++m) {
      tc::mbar_init(&tfull_bar[m], 1);
      tc::mbar_init(&tempty_bar[m], kEpiTile);
    }
    for (int m = 0; m < MT; ++m) {
      // one arming arrive per use; the peers' st.async stores complete the bytes
      tc::mbar_init(&recv_full[m], 1);
      for (int p = 0; p < C; ++p) tc::mbar_init(&free_bar[m][p], kEpiTile);
    }
    tc::fence_barrier_init();
    if (C > 1)
      for (int m = 0; m < MT; ++m) tc::mbar_arrive_expect_tx(&recv_full[m], kRecvBytes);
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(&tmem_sh);
  tc::fence_before_sync();
  __syncthreads();
  if constexpr (C > 1) cluster_sync();  // peers' barriers are initialized before any remote arrive
  tc::fence_after_sync();
  {
    int m = 0;
    for (int i = threadIdx.x; i < a.B; i += blockDim.x) m = max(m, (int)a.lens[i]);
    atomicMax(&tmax_sh, m);
  }
  __syncthreads();
  const int Tmax = tmax_sh;
  const uint32_t tmem = tmem_sh;
#ifdef SL_EXPERIMENTS  // per-(CTA, iteration) stamps for scripts/trace_bwd.py (slot map there)
  unsigned long long* trace = a.trace ? a.trace + (size_t)blockIdx.x * a.T * 32 : nullptr;
#define TRB(it, k)                                           \
  do {                                                       \
    if (trace) trace[(size_t)(it) * 32 + (k)] = gtimer();    \
  } while (0)
#else
#define TRB(it, k) \
  do {             \
  } while (0)
#endif
  // Step counters per (direction, batch tile, DZ box of kb*64 ring columns): a
  // CTA publishes DZ_s of its units to every box its columns fall in (<= 2 per
  // gate), and a consumer streams each box of its K slice as soon as THAT box's
  // producers (a handful of CTAs) published — not the slowest of all P.
  const int bw = kst;
  unsigned* ctr = a.bar + d * 2 * kBoxCtrs;
  const int hq8c = dz_ring_hq(a.H);
  auto box_producers = [&](int gb) -> unsigned {  // CTAs whose DZ columns hit box gb
    const int lo = gb * bw, hi = lo + bw;
    unsigned n = 0;
    for (int c = 0; c < a.P; ++c) {
      const int ua = c * U, ub = min(ua + U, a.H);
      bool hit = false;
#pragma unroll
      for (int g = 0; g < 4; ++g) hit |= ua < ub && g * hq8c + ua < hi && g * hq8c + ub > lo;
      n += hit ? 1u : 0u;
    }
    return n;
  };
  const int ngrp = Kc / kst;  // TMA boxes per tile
  const int kc_off = cta % ngrp;

  if (warp == 0) {  // ---------------------------------------------- producer
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(&r_bar, r_bytes);
      for (int kc = 0; kc < (MODE == kX3 ? nkc : 0); ++kc) {  // (kBF16 / kX3C stream R with DZ)
        tc::tma_load_2d(sR + (size_t)kc * NB * 128, tmR, &r_bar, kc * 64, cta * NB);
        if constexpr (MODE == kX3)  // the lo rows follow the P * NB hi rows
          tc::tma_load_2d(sR + r_part + (size_t)kc * NB * 128, tmR, &r_bar, kc * 64, a.P * NB + cta * NB);
      }
    }
    int st = 0;  // ring position, tracked by every lane (lane 0 issues)
    uint32_t ph = 0;
    const int nst = a.stages;
    // the saved activations the epilogue reads this iteration: this CTA's
    // 16-unit chunk of the 4 gates and of c_{s-1}, all rows of the launch
    const int pf_u = (u0 / 16) * 16;
    const int pf_rows = min(a.B - a.b0, MT * 128);
    const bool pf = (X3 ? a.gatesf[d] != nullptr : a.gates[d] != nullptr) && u0 < a.H;
    const uint32_t pf_elem = X3 ? 4 : 2;
    // lane k polls the k-th box of this CTA's K slice in issue order
    const int kg_lane = (lane + kc_off) % ngrp;
    const int gb_lane = r * (Kc / bw) + kg_lane;
    const unsigned exp_lane = lane < ngrp ? box_producers(gb_lane) : 0u;
    for (int s = 0; s < Tmax; ++s) {  // s = iteration (processing step Tmax-1-s)
      const int slot = s & 1;          // ring slot holding DZ of the previous iteration
      if (pf && lane == 0) {
        const int ps = Tmax - 1 - s;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const size_t o = gate_save_off(ps, g, a.b0, a.B, a.H, pf_u);
          if constexpr (X3) prefetch_l2(a.gatesf[d] + o, pf_rows * 16 * pf_elem);
          else prefetch_l2(a.gates[d] + o, pf_rows * 16 * pf_elem);
        }
        const size_t o = cprev_save_off(ps, a.b0, a.B, a.H, pf_u);
        if constexpr (X3) prefetch_l2(a.cprevf[d] + o, pf_rows * 16 * pf_elem);
        else prefetch_l2(a.cprev[d] + o, pf_rows * 16 * pf_elem);
      }
      for (int mt = 0; mt < MT; ++mt) {
        const unsigned target = exp_lane * (unsigned)s;
        bool rdy = lane >= ngrp || s == 0;
        int done = 0;
        while (done < ngrp) {
          if (!rdy) rdy = ld_acquire(ctr + mt * kBoxCtrs + gb_lane) >= target;
          const unsigned m = __ballot_sync(0xffffffffu, rdy);
          while (done < ngrp && ((m >> done) & 1u)) {
            if (lane == 0) {
              if (done == 0) TRB(s, 3 * mt);
              const int kg = (done + kc_off) % ngrp;
              tc::fence_proxy_async_global();  // the box's DZ (generic-proxy stores) -> TMA reads
#ifdef SL_EXPERIMENTS
              const unsigned long long w0 = trace ? gtimer() : 0;
#endif
              tc::mbar_wait(&empty_bar[st], ph ^ 1);
#ifdef SL_EXPERIMENTS
              if (trace) {  // time the producer waited for a free ring slot, and the last issue
                trace[(size_t)s * 32 + 18 + mt] += gtimer() - w0;
                if (done == ngrp - 1) trace[(size_t)s * 32 + 16 + mt] = gtimer();
                if (done == ngrp / 2) trace[(size_t)s * 32 + 20 + mt] = gtimer();
              }
#endif
              tc::mbar_arrive_expect_tx(&full_bar[st], stage_bytes);
              const int kcol8 = (r * Kc + kg * kst) / 8;  // the box's first 8-column chunk of the ring
              if constexpr (MODE == kX3C)  // this box's R rows (no dependency on the step)
                tma_load_3d(sA + st * stage_bytes + 2 * part_bytes, tmRl, &full_bar[st], 0, (cta * NB) / 8,
                            (kg * kst) / 8);
              if constexpr (MODE != kX3)
                tma_load_3d(sA + st * stage_bytes + rhi_off, tmRh, &full_bar[st], 0, (cta * NB) / 8, (kg * kst) / 8);
              tma_load_4d(sA + st * stage_bytes, tmZ, &full_bar[st], 0, (a.b0 + mt * 128) / 8, kcol8, slot);
              if constexpr (X3)
                tma_load_4d(sA + st * stage_bytes + part_bytes, tmZl, &full_bar[st], 0, (a.b0 + mt * 128) / 8,
                            kcol8, slot);
            }
            if (++st == nst) {
              st = 0;
              ph ^= 1;
            }
            ++done;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // -------------------------------------------- MMA issuer
      constexpr uint32_t idesc = tc::make_idesc(128, NB, 1, false, false);
      tc::mbar_wait(&r_bar, 0);
      int st = 0;
      uint32_t ph = 0;
      const int nst = a.stages;
      for (int s = 0; s < Tmax; ++s) {
        for (int mt = 0; mt < MT; ++mt) {
          tc::mbar_wait(&tempty_bar[mt], (s & 1) ^ 1);
          tc::fence_after_sync();
          for (int kq = 0; kq < ngrp; ++kq) {
            const int kg = (kq + kc_off) % ngrp;
            tc::mbar_wait(&full_bar[st], ph);
            tc::fence_after_sync();
            if (kq == 0) TRB(s, 1 + 3 * mt);
            if (kq == ngrp - 1) TRB(s, 2 + 3 * mt);
            if (kq == ngrp / 2) TRB(s, 22 + mt);
            // A: the stage holds [kst / 8 K-chunks][128 rows][8] (SWIZZLE_NONE), 2 KB per chunk;
            // B_hi: the resident SW128 K-major R rows (128 B per 64-K chunk row)
            const uint32_t sa = base + r_bytes + st * stage_bytes;
            const int k0 = kg * kst;  // first K (gate column) of the box within the slice
#pragma unroll 1
            for (int k = 0; k < kst / 16; ++k) {
              const int kk = k0 + 16 * k;
              const uint32_t sb = base + (uint32_t)(kk / 64) * NB * 128 + (uint32_t)((kk % 64) / 16) * 32;
              const uint64_t ah = tc::make_sdesc_noswz(sa + k * 2 * 2048, 2048, 128);
              // B_hi: the stage's [kst / 8][NB rows][8] core matrices, or (kX3) resident SW128 rows
              const uint64_t bh = MODE != kX3 ? tc::make_sdesc_noswz(sa + rhi_off + k * 2 * NB * 16, NB * 16, 128)
                                              : tc::make_sdesc(sb, 0, 1024);
              tc::mma_f16(tmem + mt * NB, ah, bh, idesc, (kq | k) != 0);
              if constexpr (X3) {
                const uint64_t al = tc::make_sdesc_noswz(sa + part_bytes + k * 2 * 2048, 2048, 128);
                // R_lo: resident SW128 (kX3) or the stage's [kst / 8][NB rows][8] core matrices (kX3C)
                const uint64_t bl = MODE == kX3 ? tc::make_sdesc(sb + r_part, 0, 1024)
                                                : tc::make_sdesc_noswz(sa + 2 * part_bytes + k * 2 * NB * 16, NB * 16, 128);
                tc::mma_f16(tmem + mt * NB, al, bh, idesc, true);  // DZ_lo R_hi^T
                tc::mma_f16(tmem + mt * NB, ah, bl, idesc, true);  // DZ_hi R_lo^T
              }
            }
            tc::mma_commit(&empty_bar[st]);
            if (++st == nst) {
              st = 0;
              ph ^= 1;
            }
          }
          tc::mma_commit(&tfull_bar[mt]);
        }
      }
    }
  } else {  // ------------------------------------------------------ epilogue
    const int e = warp - 2;
    const int mt = e / (4 * SPLIT);
    const int half = (e / 4) % SPLIT;
    const int q = warp & 3;
    const int rl = q * 32 + lane;  // row within the tile
    const int row = a.b0 + mt * 128 + rl;
    const bool valid_row = row < a.B;
    const int len = valid_row ? a.lens[row] : 0;
    const int dir = a.dirsign[d];
    const int gdir = MODE == kX3 ? a.dir0 + d : d;  // global direction: dy / DZ columns, final-state rows
    const int H = a.H, T = a.T;
    const int lo = half * UT;
    const int ut0 = u0 + lo;
    const int nu = max(0, min(UT, H - ut0));
    __nv_bfloat16* zr = a.dzring[d];
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + mt * NB;
    float gcar[UT];
#pragma unroll
    for (int u = 0; u < UT; ++u) gcar[u] = 0.f;

    for (int it = 0; it < Tmax; ++it) {
      const int s = Tmax - 1 - it;  // processing step
      // uses of the exchange buffer: once per step per tile, or (kX3C: one buffer for both
      // tiles) MT it + mt — the senders of a use wait until the receiver consumed the
      // previous one (at most one use ahead: a sender's MMA input needed the receiver's
      // publish of the previous step, which follows its consumption)
      constexpr bool kShared = MODE == kX3C;
      const int use = kShared ? MT * it + mt : it;
      const int fb = kShared ? 0 : mt;             // free-barrier set
      const size_t rtile = kShared ? 0 : (size_t)mt;  // receive-buffer tile
      const bool active = valid_row && s < len;
      const int t = active ? src_time(s, len, dir) : s;
      const size_t pos = (size_t)row * T + t;
      // saved gates / c_{s-1} of this step: fp32 (x3) or packed bf16 (registers)
      typename std::conditional<X3, float[4][UT], Bf16Vec<UT>[4]>::type gv;
      typename std::conditional<X3, float[UT], Bf16Vec<UT>>::type cp;
      float dyv[UT];
#ifdef SL_EXPERIMENTS
      if (active && (a.debug_flags & 16)) {  // timing experiment: no saved-activation / dy loads
#pragma unroll
        for (int u = 0; u < UT; ++u) {
          if constexpr (X3) {
#pragma unroll
            for (int g = 0; g < 4; ++g) gv[g][u] = 0.5f;
            cp[u] = 0.1f;
          }
          dyv[u] = 0.01f;
        }
      } else
#endif
      if (active) {  // prefetch this step's saved activations and upstream grad
        const bool vec = nu == UT && (UT % 4) == 0 && (H % 4) == 0;
        if constexpr (X3) {
#pragma unroll
          for (int g = 0; g < 4; ++g) load_f32<UT>(a.gatesf[d] + gate_save_off(s, g, row, a.B, H, ut0), gv[g], nu, true);
          load_f32<UT>(a.cprevf[d] + cprev_save_off(s, row, a.B, H, ut0), cp, nu, true);
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g) gv[g].load(a.gates[d] + gate_save_off(s, g, row, a.B, H, ut0), nu, true);
          cp.load(a.cprev[d] + cprev_save_off(s, row, a.B, H, ut0), nu, true);
        }
        load_f32<UT>(a.dy + pos * a.dy_ld + (size_t)gdir * H + ut0, dyv, nu, vec && (a.dy_ld % 4) == 0);
      }
      float dh[UT];
      const bool tr0 = e == 0 && lane == 0;
      if (tr0) TRB(it, 12);
#ifdef SL_EXPERIMENTS
      if (tr0 && trace && it == 0) {  // placement: the SM this CTA runs on
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trace[31] = smid;
      }
#endif
      tc::mbar_wait(&tfull_bar[mt], it & 1);
      tc::fence_after_sync();
      if (tr0) TRB(it, 8);
      if constexpr (C > 1) {
        // reduce-scatter of the K-split partials: send each peer the columns of
        // the units it finalizes (coalesced: a warp writes 32 consecutive rows)
#pragma unroll 1
        for (int pi = 1; pi < C; ++pi) {
          const int p = (r + pi) % C;
          if (use > 0) {  // one cluster-scope acquire per warp, then warp-ordered
            if (lane == 0) mbar_wait_cluster(&free_bar[fb][p], (use - 1) & 1);
            __syncwarp();
          }
          float v[UT];
          tmem_ld_cols<UT>(tbase + p * U + lo, v);
          const int slot_at_p = (r - p + C) % C - 1;  // my slot in p's buffer
          const uint32_t dst = mapa(
              tc::smem_u32(recv + ((rtile * (C - 1) + slot_at_p) * 128 + rl) * U + lo), p);
          const uint32_t rbar = mapa(tc::smem_u32(&recv_full[mt]), p);
          static_assert(UT % 4 == 0, "DSMEM partial sends move 4 or 8 values per store");
          // st.async: each store completes its bytes on p's receive barrier, so
          // no release fence (which would wait for this thread's pending global
          // stores) sits on the exchange path
          if constexpr (X3) {  // fp32 partials: the reduction stays fp32-exact
#pragma unroll
            for (int u = 0; u < UT; u += 4)
              st_async_v4(dst + u * 4,
                          make_uint4(__float_as_uint(v[u]), __float_as_uint(v[u + 1]), __float_as_uint(v[u + 2]),
                                     __float_as_uint(v[u + 3])),
                          rbar);
          } else {
            Bf16Vec<UT> w;
            w.pack(v);
            if constexpr (UT % 8 == 0) {
#pragma unroll
              for (int u = 0; u < UT; u += 8)
                st_async_v4(dst + u * 2, make_uint4(w.w[u / 2], w.w[u / 2 + 1], w.w[u / 2 + 2], w.w[u / 2 + 3]),
                            rbar);
            } else {
#pragma unroll
              for (int u = 0; u < UT; u += 4)
                st_async_v2(dst + u * 2, make_uint2(w.w[u / 2], w.w[u / 2 + 1]), rbar);
            }
          }
        }
      }
      tmem_ld_cols<UT>(tbase + r * U + lo, dh);
      tc::fence_before_sync();
      tc::mbar_arrive(&tempty_bar[mt]);
      if (tr0) TRB(it, 9);
      if constexpr (C > 1) {
        mbar_wait_cluster(&recv_full[mt], it & 1);
        if (tr0) TRB(it, 10);
        if ((e % (4 * SPLIT)) == 0 && lane == 0)  // phase `use` is complete: arm the next use
          tc::mbar_arrive_expect_tx(&recv_full[mt], kRecvBytes);
#pragma unroll 1
        for (int sl = 0; sl < C - 1; ++sl) {
          const RecvT* src = recv + ((rtile * (C - 1) + sl) * 128 + rl) * U + lo;
          if constexpr (X3) {
#pragma unroll
            for (int u = 0; u < UT; u += 4) {
              const float4 f = *reinterpret_cast<const float4*>(src + u);
              dh[u] += f.x, dh[u + 1] += f.y, dh[u + 2] += f.z, dh[u + 3] += f.w;
            }
          } else if constexpr (UT % 8 == 0) {
#pragma unroll
            for (int u = 0; u < UT; u += 8) {
              float f[8];
              unpack8_bf16(*reinterpret_cast<const uint4*>(src + u), f);
#pragma unroll
              for (int k = 0; k < 8; ++k) dh[u + k] += f[k];
            }
          } else {
#pragma unroll
            for (int u = 0; u < UT; ++u) dh[u] += __bfloat162float(src[u]);
          }
        }
        // the senders learn that their slots are free from ONE arrive per peer
        // after the tile's publish barrier below (every reader is done by then)
      }
      if (tr0) TRB(it, 13);

      // DZ_s: fp32 (x3) or packed bf16 — the ring copy now, the K4 copy after publishing
      typename std::conditional<X3, float[4 * UT], Bf16Vec<UT>[4]>::type dzs;
      if (valid_row) {
        const int hq8 = dz_ring_hq(H);
        if (active) {
          const bool last = (s == len - 1);
          if (last && (a.dh_last || a.dc_last)) {  // the final-state adjoints enter at s = len - 1
#pragma unroll
            for (int u = 0; u < UT; ++u) {
              if (u >= nu) continue;
              if (a.dh_last) dh[u] += a.dh_last[((size_t)gdir * a.B + row) * H + ut0 + u];
              if (a.dc_last) gcar[u] += a.dc_last[((size_t)gdir * a.B + row) * H + ut0 + u];
            }
          }
          if constexpr (X3) {  // the reference's adjoint, fp32 (tape.cpp:1157-1170)
            float tcs[UT];  // tanh(c_s), two units per paired instruction (two-MUFU tanh, abs. error ~1e-7)
#pragma unroll
            for (int u = 0; u < UT; u += 2) {
              const float2 c2 = make_float2(gv[1][u] * cp[u] + gv[0][u] * gv[2][u],
                                            gv[1][u + 1] * cp[u + 1] + gv[0][u + 1] * gv[2][u + 1]);
              const float2 t2 = fm::tanh2(c2);
              tcs[u] = t2.x, tcs[u + 1] = t2.y;
            }
#pragma unroll
            for (int u = 0; u < UT; ++u) {
              const float gh = dh[u] + dyv[u], gc = gcar[u];
              const float gi = gv[0][u], gf = gv[1][u], gg = gv[2][u], go = gv[3][u];
              const float tcv = tcs[u];
              const float d_o = gh * tcv;
              const float dcn = gc + gh * go * (1.f - tcv * tcv);
              gcar[u] = dcn * gf;
              dzs[u] = dcn * gg * gi * (1.f - gi);
              dzs[UT + u] = dcn * cp[u] * gf * (1.f - gf);
              dzs[2 * UT + u] = dcn * gi * (1.f - gg * gg);
              dzs[3 * UT + u] = d_o * go * (1.f - go);
            }
          } else {
            float dz[4 * UT];
            const float2 one = f2s(1.f), mone = f2s(-1.f);
#pragma unroll
            for (int u = 0; u < UT; u += 2) {  // two units per paired-fp32 instruction
              const float2 gh = add2(f2(dh[u], dh[u + 1]), f2(dyv[u], dyv[u + 1]));
              const float2 gc = f2(gcar[u], gcar[u + 1]);
              const float2 gi = bf16x2_f2(gv[0].w[u / 2]), gf = bf16x2_f2(gv[1].w[u / 2]);
              const float2 gg = bf16x2_f2(gv[2].w[u / 2]), go = bf16x2_f2(gv[3].w[u / 2]);
              const float2 cpu = bf16x2_f2(cp.w[u / 2]);
              const float2 tcv = tanh2(fma2(gf, cpu, mul2(gi, gg)));
              const float2 d_o = mul2(gh, tcv);                                      // tape.cpp:1161
              const float2 dcn = fma2(mul2(gh, go), fma2(mul2(mone, tcv), tcv, one), gc);  // tape.cpp:1162
              const float2 cg = mul2(dcn, gf);                                       // tape.cpp:1166
              gcar[u] = cg.x, gcar[u + 1] = cg.y;
              const float2 zi = mul2(mul2(dcn, gg), mul2(gi, fma2(mone, gi, one)));    // tape.cpp:1167
              const float2 zf = mul2(mul2(dcn, cpu), mul2(gf, fma2(mone, gf, one)));   // tape.cpp:1168
              const float2 zg = mul2(mul2(dcn, gi), fma2(mul2(mone, gg), gg, one));    // tape.cpp:1169
              const float2 zo = mul2(mul2(d_o, go), fma2(mone, go, one));              // tape.cpp:1170
              dz[u] = zi.x, dz[u + 1] = zi.y;
              dz[UT + u] = zf.x, dz[UT + u + 1] = zf.y;
              dz[2 * UT + u] = zg.x, dz[2 * UT + u + 1] = zg.y;
              dz[3 * UT + u] = zo.x, dz[3 * UT + u + 1] = zo.y;
            }
#pragma unroll
            for (int g = 0; g < 4; ++g) dzs[g].pack(dz + g * UT);
          }
        } else {
          if constexpr (X3) {
#pragma unroll
            for (int u = 0; u < 4 * UT; ++u) dzs[u] = 0.f;
          } else {
#pragma unroll
            for (int g = 0; g < 4; ++g) dzs[g].zero();
          }
        }
        if (tr0) TRB(it, 14);
        constexpr int CW = UT < 8 ? UT : 8;  // the ring's 8-unit chunks are Bp * 16 B apart
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int c = 0; c < UT; c += CW) {
            const size_t off = dz_ring_off((it + 1) & 1, row, g * hq8 + ut0 + c, dz_ring_bp(a.B), a.Kz);
            const int n = max(0, min(CW, nu - c));
            if constexpr (X3) {
              store_bf16<CW>(zr + off, dzs + g * UT + c, n);
              float l[CW];  // DZ_lo = DZ - bf16(DZ)
#pragma unroll
              for (int u = 0; u < CW; ++u)
                l[u] = dzs[g * UT + c + u] - __bfloat162float(__float2bfloat16_rn(dzs[g * UT + c + u]));
              store_bf16<CW>(a.dzring_lo[d] + off, l, n);
            } else {
              Bf16Vec<CW> part;
#pragma unroll
              for (int w = 0; w < CW / 2; ++w) part.w[w] = dzs[g].w[c / 2 + w];
              part.store(zr + off, n);
            }
          }
      }
      if (tr0) TRB(it, 11);
      named_sync(1 + mt, kEpiTile);
      if ((e % (4 * SPLIT)) == 0 && lane == 0) {
        tc::fence_proxy_async_global();
        {  // every DZ box my columns fall in (ascending, each once), after ONE release fence
          const int ua = u0, ub = min(u0 + U, H);
          int prev = -1;
          fence_acq_rel_gpu();
#pragma unroll 1
          for (int g = 0; g < 4 && ua < ub; ++g)
            for (int gb = (g * hq8c + ua) / bw; gb <= (g * hq8c + ub - 1) / bw; ++gb)
              if (gb != prev) {
                red_relaxed_gpu(ctr + mt * kBoxCtrs + gb, 1u);
                prev = gb;
              }
          TRB(it, 6 + mt);
        }
        if constexpr (C > 1)  // every sender's slot in my receive buffer is free again
          for (int pi = 1; pi < C; ++pi)
            mbar_arrive_remote_relaxed(mapa(tc::smem_u32(&free_bar[MODE == kX3C ? 0 : mt][r]), (r + pi) % C),
                                       kEpiTile);
      }
#ifdef SL_EXPERIMENTS
      const bool skip_k4 = (a.debug_flags & 8) != 0;  // timing experiment: no K4 operand copy
#else
      constexpr bool skip_k4 = false;
#endif
      if (valid_row && !skip_k4) {  // the K4 operand copy is off the cross-CTA critical path
        if constexpr (X3) {  // the split image the K4 GEMMs read: hi and lo
          __nv_bfloat16* zh = a.dzimg + pos * a.dzcat_ld + (size_t)gdir * a.dz_dir_off + ut0;
          __nv_bfloat16* zl = zh + a.dzimg_rows * a.dzcat_ld;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float l[UT];
#pragma unroll
            for (int u = 0; u < UT; ++u) l[u] = dzs[g * UT + u] - __bfloat162float(__float2bfloat16_rn(dzs[g * UT + u]));
            store_bf16<UT>(zh + g * H, dzs + g * UT, nu);
            store_bf16<UT>(zl + g * H, l, nu);
          }
        } else {
          __nv_bfloat16* zc = a.dzcat + pos * a.dzcat_ld + (size_t)d * a.dz_dir_off + ut0;
#pragma unroll
          for (int g = 0; g < 4; ++g) dzs[g].store(zc + g * H, nu);
        }
      }
    }
    if (valid_row) {  // DZ rows of positions beyond the longest sequence
      float zero[UT];
#pragma unroll
      for (int u = 0; u < UT; ++u) zero[u] = 0.f;
      for (int s = Tmax; s < T; ++s) {
        if constexpr (X3) {
          __nv_bfloat16* zh = a.dzimg + ((size_t)row * T + s) * a.dzcat_ld + (size_t)gdir * a.dz_dir_off + ut0;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            store_bf16<UT>(zh + g * H, zero, nu);
            store_bf16<UT>(zh + a.dzimg_rows * a.dzcat_ld + g * H, zero, nu);
          }
        } else {
          __nv_bfloat16* zc =
              a.dzcat + ((size_t)row * T + s) * a.dzcat_ld + (size_t)d * a.dz_dir_off + ut0;
#pragma unroll
          for (int g = 0; g < 4; ++g) store_bf16<UT>(zc + g * H, zero, nu);
        }
      }
    }
  }
  __syncthreads();
  if constexpr (C > 1) cluster_sync();  // no CTA leaves while a peer may still touch its smem
  if (warp == 1) tc::tmem_dealloc<kTmemCols>(tmem);
}

// RB[(cl*C + r)*NB + n][kk] = R[cl*C*U + n][r*Kc + kk]  (bf16; zero outside the layer)
// BOTH: also the rounding remainder R - bf16(R) (x3), written P * NB rows further on —
// R read once for both parts.
// One CTA per packed row; threads along kk (coalesced on both sides), 32-bit math.
template <bool BOTH>
__global__ void pack_rb_kernel(const float* __restrict__ R, int H, int C, int U, int NB, int P,
                               int Kc, __nv_bfloat16* __restrict__ RB, bool interleave = false) {
  const int rowi = blockIdx.x;
  const int cta = rowi / NB, n = rowi % NB;
  const int cl = cta / C, r = cta % C;
  const int unit = cl * C * U + n;
  const bool live = n < C * U && unit < H;
  // interleave (the streamed R of kX3C): the rows in the core-matrix layout
  // [Kc / 8][P * NB rows][8], so a TMA box of NB rows x 8 K is one contiguous 128 B-row run
  // (16 B rows of a row-major slice would cost one TMA request each)
  const size_t part = (size_t)P * NB * Kc;  // the lo part follows the hi part
  auto at = [&](int kk) -> __nv_bfloat16* {
    return interleave ? RB + ((size_t)(kk / 8) * P * NB + rowi) * 8 + kk % 8 : RB + (size_t)rowi * Kc + kk;
  };
  auto lo_of = [](float v) { return __float2bfloat16_rn(v - __bfloat162float(__float2bfloat16_rn(v))); };
  const int hq8 = dz_ring_hq(H);
  if (hq8 != H) {  // gate blocks padded to a multiple of 8 columns in the DZ ring
    for (int kk = threadIdx.x; kk < Kc; kk += blockDim.x) {
      const int col = r * Kc + kk, g = col / hq8, u = col % hq8;
      const float v = (live && g < 4 && u < H) ? __ldg(R + (size_t)unit * 4 * H + (size_t)g * H + u) : 0.f;
      *at(kk) = __float2bfloat16_rn(v);
      if (BOTH) at(kk)[part] = lo_of(v);
    }
    return;
  }
  const float* src = R + (size_t)unit * 4 * H + (size_t)r * Kc;
  const int valid = live ? max(0, min(Kc, 4 * H - r * Kc)) : 0;
  // 4 columns per thread: float4 loads when the row start is 16 B aligned, 8 B bf16 stores
  const bool vec = (((uintptr_t)src) & 15) == 0 && (Kc % 4) == 0;
  auto pack4 = [](__nv_bfloat16 b0, __nv_bfloat16 b1, __nv_bfloat16 b2, __nv_bfloat16 b3) {
    __nv_bfloat162 p0, p1;
    p0.x = b0, p0.y = b1, p1.x = b2, p1.y = b3;
    return make_uint2(*reinterpret_cast<const uint32_t*>(&p0), *reinterpret_cast<const uint32_t*>(&p1));
  };
  for (int kk = threadIdx.x * 4; kk < Kc; kk += blockDim.x * 4) {
    float v[4];
    if (vec && kk + 4 <= valid) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(src + kk));
      v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = kk + u < valid ? __ldg(src + kk + u) : 0.f;
    }
    if (kk + 4 <= Kc) {
      *reinterpret_cast<uint2*>(at(kk)) = pack4(__float2bfloat16_rn(v[0]), __float2bfloat16_rn(v[1]),
                                                __float2bfloat16_rn(v[2]), __float2bfloat16_rn(v[3]));
      if (BOTH)
        *reinterpret_cast<uint2*>(at(kk) + part) = pack4(lo_of(v[0]), lo_of(v[1]), lo_of(v[2]), lo_of(v[3]));
    } else {
      for (int u = 0; u < 4 && kk + u < Kc; ++u) {
        *at(kk + u) = __float2bfloat16_rn(v[u]);
        if (BOTH) at(kk + u)[part] = lo_of(v[u]);
      }
    }
  }
}

template <int C, int U, int MT, int MODE>
void launch_bwd(const BwdMaps& mp, const TcRecBwdArgs& a, cudaStream_t stream) {
  auto kern = rec_bwd_tc_kernel<C, U, MT, MODE>;
  const uint32_t smem = bwd_smem_m(MODE, C, U, a.Kz / C, a.stages, a.kb);
  SL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (C > 1)
    SL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  TcRecBwdArgs copy = a;
  constexpr int kSplit = bwd_split(U);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.P * a.nd);
  cfg.blockDim = dim3(64 + 128 * MT * kSplit);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other)
  attrs[0].val.cooperative = 1;
  attrs[1].id = cudaLaunchAttributeClusterDimension;
  attrs[1].val.clusterDim.x = C;
  attrs[1].val.clusterDim.y = 1;
  attrs[1].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  // SL_NO_COOP=1 (profiling only): ncu cannot launch cooperative cluster
  // kernels; the grid (<= #SMs, 1 CTA/SM) is still co-resident in practice.
  static const bool no_coop = getenv("SL_NO_COOP") != nullptr;
  if (no_coop) {
    cfg.attrs = attrs + 1;
    cfg.numAttrs = 1;
  }
  SL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, mp, copy));
  count_launch();
}

// the DZ ring in its interleaved layout, as {8 rows x 8 k (128 contiguous B),
// 8-row groups, K-chunks of 8, slot}: 128 B TMA rows, box = 128 rows x kk K
CUtensorMap dz_ring_map(const __nv_bfloat16* ring, int B, int Kz, int kk) {
  const int Bp = dz_ring_bp(B);
  cuuint64_t zd[4] = {64, (cuuint64_t)Bp / 8, (cuuint64_t)Kz / 8, 2};
  cuuint64_t zs[3] = {128, (cuuint64_t)Bp * 16, (cuuint64_t)Kz / 8 * Bp * 16};
  cuuint32_t zb[4] = {64, 16, (cuuint32_t)kk / 8, 1};
  return tmap(ring, 4, zd, zs, zb, CU_TENSOR_MAP_SWIZZLE_NONE);
}

template <int MODE>
void dispatch_bwd(const TcBwdShape& sh, int MT, const BwdMaps& mp, const TcRecBwdArgs& a, cudaStream_t stream) {
  const int key = sh.C * 1000 + sh.U * 10 + MT;
  switch (key) {
#define SL_BWD_CASE(C_, U_, MT_) \
  case C_ * 1000 + U_ * 10 + MT_: launch_bwd<C_, U_, MT_, MODE>(mp, a, stream); break;
    SL_BWD_CASE(4, 4, 1) SL_BWD_CASE(4, 4, 2) SL_BWD_CASE(4, 8, 1) SL_BWD_CASE(4, 8, 2)
    SL_BWD_CASE(4, 16, 1) SL_BWD_CASE(4, 16, 2) SL_BWD_CASE(2, 4, 1) SL_BWD_CASE(2, 4, 2)
    SL_BWD_CASE(2, 8, 1) SL_BWD_CASE(2, 8, 2) SL_BWD_CASE(2, 16, 1) SL_BWD_CASE(2, 16, 2)
    SL_BWD_CASE(1, 4, 1) SL_BWD_CASE(1, 4, 2) SL_BWD_CASE(1, 8, 1) SL_BWD_CASE(1, 8, 2)
    SL_BWD_CASE(1, 16, 1) SL_BWD_CASE(1, 16, 2)
#undef SL_BWD_CASE
    default: throw Error{SL_ERR_UNSUPPORTED, "rec_bwd_tc: unsupported partition"};
  }
}

int pick_stages(int mode, const TcBwdShape& sh, int kb) {
  const int Kc = sh.Kz / sh.C;
  for (int st = stream_r(mode) ? kStages : 6; st >= 2; --st)
    if (bwd_smem_m(mode, sh.C, sh.U, Kc, st, kb) <= kSmemMax) return st;
  return 0;
}

}  // namespace

TcBwdShape tc_rec_bwd_shape(int H, int nd, int sms) {
  TcBwdShape pair_shape;
  if (tc_rec_bwd_pair_fits(H, nd, sms, 0, &pair_shape)) return pair_shape;
  // Prefer 4-CTA clusters (4x less DZ per CTA); most CTAs that fit a cluster
  // grid (~128 SMs usable by 4-CTA clusters on 148 SMs) and shared memory.
  for (int C : {4, 2, 1}) {
    const int usable = C == 4 ? std::min(sms, 128) : sms;
    for (int U : {4, 8, 16}) {
      const int P = (int)ceil_div(H, (int64_t)C * U) * C;
      const int Kz = (int)round_up(4 * (int64_t)dz_ring_hq(H), 64 * C);
      if ((int64_t)P * nd <= usable && bwd_smem(C, U, Kz / C, 2) <= kSmemMax)
        return TcBwdShape{C, U, P, Kz};
    }
  }
  return TcBwdShape{0, 0, 0, 0};
}

size_t tc_rec_bwd_pack_elems(const TcBwdShape& sh) {
  if (sh.pair) return tc_rec_bwd_pair_pack_elems(sh);
  return (size_t)sh.P * nb_of(sh.C, sh.U) * (sh.Kz / sh.C);
}

void tc_rec_bwd_pack(const float* R, int H, const TcBwdShape& sh, __nv_bfloat16* RB,
                     cudaStream_t stream) {
  if (sh.pair) {
    tc_rec_bwd_pair_pack(R, H, sh, RB, stream);
    return;
  }
  const int NB = nb_of(sh.C, sh.U);
  const int Kc = sh.Kz / sh.C;
  pack_rb_kernel<false><<<(unsigned)(sh.P * NB), 256, 0, stream>>>(R, H, sh.C, sh.U, NB, sh.P, Kc, RB, true);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void rec_bwd_tc(const TcRecBwdArgs& a0, const TcBwdShape& sh, __nv_bfloat16* const* RB,
                cudaStream_t stream) {
  if (sh.pair) {
    rec_bwd_pair(a0, sh, RB, stream);
    return;
  }
  TcRecBwdArgs a = a0;
  a.U = sh.U;
  a.P = sh.P;
  a.Kz = sh.Kz;
  const int NB = nb_of(sh.C, sh.U);
  const int Kc = sh.Kz / sh.C;
  BwdMaps mp{};
  a.kb = (Kc / 64) % 2 == 0 ? 2 : 1;
  for (int k = 0; k < a.nd; ++k) {
    cuuint64_t rd[2] = {(cuuint64_t)Kc, (cuuint64_t)a.P * NB};
    cuuint64_t rs[1] = {(cuuint64_t)Kc * 2};
    cuuint32_t rb[2] = {64, (cuuint32_t)NB};
    mp.R[k] = tmap(RB[k], 2, rd, rs, rb);
    mp.Z[k] = dz_ring_map(a.dzring[k], a.B, a.Kz, stage_k(kBF16, a.kb));
    // R streamed with DZ, from its interleaved pack {8 rows x 8 k, row groups, K chunks}
    cuuint64_t hd[3] = {64, (cuuint64_t)a.P * NB / 8, (cuuint64_t)Kc / 8};
    cuuint64_t hs[2] = {128, (cuuint64_t)a.P * NB * 16};
    cuuint32_t hb[3] = {64, (cuuint32_t)NB / 8, (cuuint32_t)stage_k(kBF16, a.kb) / 8};
    mp.Rhi[k] = tmap(RB[k], 3, hd, hs, hb, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  a.stages = pick_stages(kBF16, sh, a.kb);
  SL_REQUIRE(a.stages >= 2, SL_ERR_UNSUPPORTED, "rec_bwd_tc: R slice does not fit in shared memory");
  SL_REQUIRE(a.Kz / (a.kb * 64) <= kBoxCtrs && 4 * kBoxCtrs <= kBarPerChunk, SL_ERR_UNSUPPORTED,
             "rec_bwd_tc: too many DZ boxes for the step counters");
  unsigned* bar0 = a.bar;
  for (int b0 = 0; b0 < a.B; b0 += 256) {
    a.b0 = b0;
    a.bar = bar0 + kBarPerChunk * (b0 / 256);
    dispatch_bwd<kBF16>(sh, (a.B - b0) > 128 ? 2 : 1, mp, a, stream);
  }
}

TcBwdShape tc_rec_bwd_x3_shape(int H, int sms, int nd) {
  if (nd == 2) {  // kX3C: both directions per launch, R streamed with DZ (4-CTA clusters)
    const int C = 4, U = 16;
    const int P = (int)ceil_div(H, (int64_t)C * U) * C;
    const int Kz = (int)round_up(4 * (int64_t)dz_ring_hq(H), 64 * C);
    TcBwdShape sh{C, U, P, Kz};
    sh.pair = 2;
    if ((int64_t)2 * P <= std::min(sms, 128) && Kz / stage_k(kX3C, 1) <= kBoxCtrs && pick_stages(kX3C, sh, 1) >= 2)
      return sh;
  }
  for (int C : {4, 2, 1}) {  // kX3: one direction per launch
    const int usable = C == 4 ? std::min(sms, 128) : sms;
    for (int U : {8, 4, 16}) {
      const int P = (int)ceil_div(H, (int64_t)C * U) * C;
      const int Kz = (int)round_up(4 * (int64_t)dz_ring_hq(H), 64 * C);
      if (P <= usable && Kz / 64 <= kBoxCtrs) {  // kb = 1
        TcBwdShape sh{C, U, P, Kz};
        sh.pair = 1;
        if (pick_stages(kX3, sh, 1) >= 2) return sh;
      }
    }
  }
  return TcBwdShape{0, 0, 0, 0};
}

size_t tc_rec_bwd_x3_pack_elems(const TcBwdShape& sh) {
  return (size_t)2 * sh.P * nb_of(sh.C, sh.U) * (sh.Kz / sh.C);
}

void tc_rec_bwd_x3_pack(const float* R, int H, const TcBwdShape& sh, __nv_bfloat16* RB, cudaStream_t stream) {
  const int NB = nb_of(sh.C, sh.U);
  const int Kc = sh.Kz / sh.C;
  pack_rb_kernel<true><<<(unsigned)(sh.P * NB), 256, 0, stream>>>(R, H, sh.C, sh.U, NB, sh.P, Kc, RB,
                                                                   sh.pair == 2);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

// sh.pair == 2 (kX3C): a.nd == 2, both directions; sh.pair == 1 (kX3): a.nd == 1
void rec_bwd_x3(const TcRecBwdArgs& a0, const TcBwdShape& sh, const __nv_bfloat16* const* RB, cudaStream_t stream) {
  TcRecBwdArgs a = a0;
  const int mode = sh.pair == 2 ? kX3C : kX3;
  SL_REQUIRE(mode == kX3C ? a.nd == 2 : a.nd == 1, SL_ERR_INVALID_ARGUMENT, "rec_bwd_x3: direction count");
  a.U = sh.U;
  a.P = sh.P;
  a.Kz = sh.Kz;
  const int NB = nb_of(sh.C, sh.U);
  const int Kc = sh.Kz / sh.C;
  a.kb = 1;
  BwdMaps mp{};
  for (int k = 0; k < a.nd; ++k) {
    cuuint64_t rd[2] = {(cuuint64_t)Kc, (cuuint64_t)2 * a.P * NB};
    cuuint64_t rs[1] = {(cuuint64_t)Kc * 2};
    cuuint32_t rb[2] = {64, (cuuint32_t)NB};
    mp.R[k] = tmap(RB[k], 2, rd, rs, rb);
    mp.Z[k] = dz_ring_map(a.dzring[k], a.B, a.Kz, stage_k(mode, 1));
    mp.Zlo[k] = dz_ring_map(a.dzring_lo[k], a.B, a.Kz, stage_k(mode, 1));
    if (mode == kX3C) {  // interleaved R_lo {8 rows x 8 k, row groups, K chunks}: lands as [kk / 8][NB rows][8]
      cuuint64_t ld[3] = {64, (cuuint64_t)a.P * NB / 8, (cuuint64_t)Kc / 8};
      cuuint64_t ls[2] = {128, (cuuint64_t)a.P * NB * 16};
      cuuint32_t lb[3] = {64, (cuuint32_t)NB / 8, (cuuint32_t)stage_k(kX3C, 1) / 8};
      mp.Rlo[k] = tmap(RB[k] + (size_t)a.P * NB * Kc, 3, ld, ls, lb, CU_TENSOR_MAP_SWIZZLE_NONE);
      mp.Rhi[k] = tmap(RB[k], 3, ld, ls, lb, CU_TENSOR_MAP_SWIZZLE_NONE);  // R_hi streamed the same way
    }
  }
  a.stages = pick_stages(mode, sh, a.kb);
  SL_REQUIRE(a.stages >= 2, SL_ERR_UNSUPPORTED, "rec_bwd_x3: R slice does not fit in shared memory");
  SL_REQUIRE(a.Kz / stage_k(mode, 1) <= kBoxCtrs && 4 * kBoxCtrs <= kBarPerChunk, SL_ERR_UNSUPPORTED,
             "rec_bwd_x3: too many DZ boxes for the step counters");
  unsigned* bar0 = a.bar;
  for (int b0 = 0; b0 < a.B; b0 += 256) {
    a.b0 = b0;
    a.bar = bar0 + kBarPerChunk * (b0 / 256);
    if (mode == kX3C) dispatch_bwd<kX3C>(sh, (a.B - b0) > 128 ? 2 : 1, mp, a, stream);
    else dispatch_bwd<kX3>(sh, (a.B - b0) > 128 ? 2 : 1, mp, a, stream);
  }
}

}  // namespace sl
