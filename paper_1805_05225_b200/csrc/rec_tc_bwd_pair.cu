// K3, CTA-pair form — persistent tensor-core BPTT on the CTA-pair datapath.
//
// Per step the BPTT needs dh_s = DZ_{s+1} [B x 4H] . R^T [4H x H]: a K = 4H
// contraction that no single SM can hold R for, so K is split over the pairs of
// an 8-CTA cluster and the partial products are reduce-scattered through DSMEM.
// Compared with the single-CTA form (rec_tc_bwd.cu: 4-CTA clusters, N = 64,
// both 128-row batch tiles through every CTA), the pair form issues
// M = 256 (the two batch tiles, one per CTA of the pair) x N = 128 (the
// cluster's 128 hidden units, each CTA holding the R rows of 64) MMAs — full
// tensor rate — and each CTA streams only its own tile's rows of DZ: half the
// MMA instructions and half the stream bytes per SM for the same work.
//
// Cluster (8 CTAs) = 128 hidden units of one direction; rank = 2 k + h: pair k
// (K slice k of the 4H DZ columns), CTA h of the pair (batch tile h, B rows
// [64 h, 64 h + 64) of the pair's 128).  Per step:
//   warp 0 (both)   waits for the step counter of its tile, TMA-streams its
//                   tile's K-slice of DZ_{s+1} from the interleaved L2 ring,
//                   completing on the pair leader's stage barriers;
//   warp 1 (leader) issues the M=256 x N=128 x K=16 MMAs: partial dh of all 128
//                   units over K-slice k, for both tiles;
//   warps 2..9      2 threads per batch row x 16 units: load the partial
//                   columns of all 4 pairs' units (one TMEM round trip), send
//                   each other pair's 32 units to the same-tile CTA of that pair
//                   (st.async, completing on its receive barrier), sum the 3
//                   partials received for the own 32 units, run the cell adjoint
//                   (tape.cpp:1157-1170) and write DZ_s to the ring and to the
//                   K4 operand.
// Semantics as rec_tc_bwd.cu.

#ifndef SL_EXPERIMENTS
// Experiments builds only (-DSL_EXPERIMENTS): measured slower than the 4-CTA
// cluster form on B200, and the encoder's 16 clusters of 8 CTAs do not fit.
#include "rec_tc.h"
namespace sl {
bool tc_rec_bwd_pair_fits(int, int, int, int, TcBwdShape*) { return false; }
size_t tc_rec_bwd_pair_pack_elems(const TcBwdShape&) { return 0; }
void tc_rec_bwd_pair_pack(const float*, int, const TcBwdShape&, __nv_bfloat16*, cudaStream_t) {
  throw Error{SL_ERR_UNSUPPORTED, "rec_bwd_pair: experiments build only"};
}
void rec_bwd_pair(const TcRecBwdArgs&, const TcBwdShape&, __nv_bfloat16* const*, cudaStream_t) {
  throw Error{SL_ERR_UNSUPPORTED, "rec_bwd_pair: experiments build only"};
}
}  // namespace sl
#else
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "profile.h"
#include "rec_tc.h"
#include "rec_tc_common.cuh"

namespace sl {
namespace {
using namespace rtc;

constexpr int kPU = 128;          // hidden units per cluster = MMA N of every pair
constexpr int kKS = 4;            // pairs per cluster = K split
constexpr int kCl = 2 * kKS;      // CTAs per cluster
constexpr int kFU = kPU / kKS;    // units each CTA finalizes (32)
constexpr int kUT = 16;           // units per epilogue thread
constexpr int kEpi = 128 * (kFU / kUT);  // epilogue threads (256)
constexpr int kThreads = 64 + kEpi;
constexpr int kMaxStages = 6;
constexpr uint32_t kTile = 128 * 64 * 2;  // 128 rows x 64 K bf16
constexpr uint32_t kSmemMax = 227 * 1024;
constexpr uint32_t kRecvBytes = (uint32_t)(kKS - 1) * 128 * kFU * 2;  // partials received per step

// 16 consecutive TMEM columns of this thread's lane, no wait (batch, then tmem_wait_ld)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

uint32_t bp_smem(int Kc, int stages, int kb) {
  return (uint32_t)(kPU / 2) * Kc * 2 + stages * kTile * kb + kRecvBytes + 1024;
}

__global__ void __launch_bounds__(kThreads, 1)
    rec_bwd_pair_kernel(const __grid_constant__ CUtensorMap tmR0, const __grid_constant__ CUtensorMap tmR1,
                        const __grid_constant__ CUtensorMap tmZ0, const __grid_constant__ CUtensorMap tmZ1,
                        TcRecBwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t r_bar, tfull_bar, tempty_bar, recv_full, free_bar[kKS];
  __shared__ uint32_t tmem_sh;
  __shared__ int tmax_sh;

  const int per_dir = a.P;                  // CTAs per direction
  const int d = blockIdx.x / per_dir;
  const int cl = (blockIdx.x % per_dir) / kCl;
  const int rank = (int)cluster_rank();
  const int k = rank / 2, h = rank % 2;      // pair (K slice), CTA in pair (tile / B half)
  const bool leader = h == 0;
  const int Kc = a.Kz / kKS;
  const int nkc = Kc / 64;
  const CUtensorMap* tmR = d == 0 ? &tmR0 : &tmR1;
  const CUtensorMap* tmZ = d == 0 ? &tmZ0 : &tmZ1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t base = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - tc::smem_u32(smem_raw));
  const uint32_t r_bytes = (uint32_t)(kPU / 2) * Kc * 2;
  uint8_t* sR = smem;
  uint8_t* sA = smem + r_bytes;
  const uint32_t stage_bytes = kTile * a.kb;
  // [3 slots][128 rows][32 units] bf16: the other pairs' partials for my units
  __nv_bfloat16* recv = reinterpret_cast<__nv_bfloat16*>(sA + a.stages * stage_bytes);

  if (threadIdx.x == 0) {
    tmax_sh = 0;
    tc::prefetch_tmap(tmR);
    tc::prefetch_tmap(tmZ);
    for (int s = 0; s < a.stages; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    tc::mbar_init(&r_bar, 1);
    tc::mbar_init(&tfull_bar, 1);
    tc::mbar_init(&tempty_bar, 2 * kEpi);  // both CTAs of the pair (leader's copy used)
    tc::mbar_init(&recv_full, 1);          // armed once per step; the peers' st.async complete it
    for (int p = 0; p < kKS; ++p) tc::mbar_init(&free_bar[p], kEpi);
    tc::fence_barrier_init();
    tc::mbar_arrive_expect_tx(&recv_full, kRecvBytes);
  }
  if (warp == 1) tmem_alloc_pair<kPU>(&tmem_sh);
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();
  tc::fence_after_sync();
  {
    int m = 0;
    for (int i = threadIdx.x; i < a.B; i += blockDim.x) m = max(m, (int)a.lens[i]);
    atomicMax(&tmax_sh, m);
  }
  __syncthreads();
  const int Tmax = tmax_sh;
  const uint32_t tmem = tmem_sh;
  unsigned* ctr = a.bar + d * 2 + h;  // step counter of (direction, my batch tile)
  const unsigned pubs = (unsigned)(per_dir / 2);  // CTAs publishing into one tile's counter
  unsigned long long* trace =
      (a.trace && (a.trace_cta < 0 || (int)blockIdx.x == a.trace_cta))
          ? a.trace + (a.trace_cta < 0 ? (size_t)blockIdx.x * a.T * 16 : 0) : nullptr;
  const int ngrp = nkc / a.kb;
  const int kc_off = (cl * kKS + k) % ngrp;

  if (warp == 0) {
    if (lane == 0) {  // -------------------------------------------- producer (both CTAs)
      const uint32_t r_bar_l = mapa(tc::smem_u32(&r_bar), (uint32_t)(rank & ~1));
      if (leader) tc::mbar_arrive_expect_tx(&r_bar, 2 * r_bytes);
      const int rrow = ((cl * kKS + k) * 2 + h) * (kPU / 2);
      for (int kc = 0; kc < nkc; ++kc)
        tma_load_2d_pair(sR + (size_t)kc * (kPU / 2) * 128, tmR, r_bar_l, kc * 64, rrow);
      int st = 0;
      uint32_t ph = 0;
      const int pf_u = cl * kPU + k * kFU;  // my 32 units = two 16-unit chunks of the saves
      const int pf_row = a.b0 + h * 128;
      const int pf_rows = max(0, min(a.B - pf_row, 128));
      const bool pf = a.gates[d] != nullptr && pf_u < a.H && pf_rows > 0;
      for (int s = 0; s < Tmax; ++s) {  // s = iteration (processing step Tmax-1-s)
        if (pf) {  // this iteration's saved activations into L2 ahead of the epilogue's loads
          const int ps = Tmax - 1 - s;
#pragma unroll
          for (int c = 0; c < kFU; c += 16) {
            if (pf_u + c >= a.H) break;
#pragma unroll
            for (int g = 0; g < 4; ++g)
              prefetch_l2(a.gates[d] + gate_save_off(ps, g, pf_row, a.B, a.H, pf_u + c), pf_rows * 32);
            prefetch_l2(a.cprev[d] + cprev_save_off(ps, pf_row, a.B, a.H, pf_u + c), pf_rows * 32);
          }
        }
        if (s > 0) {
          const unsigned target = pubs * (unsigned)s;
          while (ld_acquire(ctr) < target) {
          }
          tc::fence_proxy_async_global();
        }
        if (trace) trace[s * 16 + 0] = gtimer();
        for (int kq = 0; kq < ngrp; ++kq) {
          const int kg = (kq + kc_off) % ngrp;
          tc::mbar_wait(&empty_bar[st], ph ^ 1);
          if (leader) tc::mbar_arrive_expect_tx(&full_bar[st], 2 * stage_bytes);
          tma_load_4d_pair(sA + st * stage_bytes, tmZ, mapa(tc::smem_u32(&full_bar[st]), (uint32_t)(rank & ~1)),
                           0, (a.b0 + h * 128) / 8, (k * nkc + kg * a.kb) * 8, s & 1);
          if (++st == a.stages) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ------------------------------------ MMA issuer (pair leader)
      constexpr uint32_t idesc = tc::make_idesc(256, kPU, 1, false, false);
      const uint16_t pair_mask = (uint16_t)(0x3u << (rank & ~1));  // this pair's two cluster ranks
      tc::mbar_wait(&r_bar, 0);
      int st = 0;
      uint32_t ph = 0;
      for (int s = 0; s < Tmax; ++s) {
        tc::mbar_wait(&tempty_bar, (s & 1) ^ 1);
        tc::fence_after_sync();
        for (int kq = 0; kq < ngrp; ++kq) {
          const int kg = (kq + kc_off) % ngrp;
          tc::mbar_wait(&full_bar[st], ph);
          tc::fence_after_sync();
          if (kq == 0 && trace) trace[s * 16 + 1] = gtimer();
          if (kq == ngrp - 1 && trace) trace[s * 16 + 2] = gtimer();
          for (int j = 0; j < a.kb; ++j) {
            const int kc = kg * a.kb + j;
            const uint32_t sa = base + r_bytes + st * stage_bytes + j * kTile;  // interleaved DZ chunks
            const uint32_t sb = base + (uint32_t)kc * (kPU / 2) * 128;         // SW128 R rows
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_f16_pair(tmem, tc::make_sdesc_noswz(sa + kk * 2 * 2048, 2048, 128),
                           tc::make_sdesc(sb + kk * 32, 0, 1024), idesc, (kq | j | kk) != 0);
          }
          mma_commit_pair(&empty_bar[st], pair_mask);
          if (++st == a.stages) {
            st = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair(&tfull_bar, pair_mask);
      }
    }
  } else {  // ------------------------------------------------------ epilogue (both CTAs)
    const int e = warp - 2;
    const int q = warp & 3;
    const int hf = e / 4;             // which 16 of my 32 units
    const int rl = q * 32 + lane;     // row within my tile
    const int row = a.b0 + h * 128 + rl;
    const bool valid_row = row < a.B;
    const int len = valid_row ? a.lens[row] : 0;
    const int dir = a.dirsign[d];
    const int H = a.H, T = a.T;
    const int ut0 = cl * kPU + k * kFU + hf * kUT;  // first global unit of this thread
    const int nu = max(0, min(kUT, H - ut0));
    __nv_bfloat16* zr = a.dzring[d];
    const __nv_bfloat16* gates = a.gates[d];
    const __nv_bfloat16* cprev = a.cprev[d];
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + hf * kUT;
    const uint32_t tempty_l = mapa(tc::smem_u32(&tempty_bar), (uint32_t)(rank & ~1));
    const int hq8 = dz_ring_hq(H), Bp = dz_ring_bp(a.B);
    float gcar[kUT];
#pragma unroll
    for (int u = 0; u < kUT; ++u) gcar[u] = 0.f;

    for (int it = 0; it < Tmax; ++it) {
      const int s = Tmax - 1 - it;  // processing step
      const bool active = valid_row && s < len;
      const int t = active ? src_time(s, len, dir) : s;
      const size_t pos = (size_t)row * T + t;
      float dyv[kUT];
      if (active)  // prefetch the step's upstream gradient (the saved activations come later:
                   // registers are short while all partial columns are in flight)
        load_f32<kUT>(a.dy + pos * a.dy_ld + (size_t)d * H + ut0, dyv, nu, (H % 4) == 0 && (a.dy_ld % 4) == 0);
      const bool tr0 = trace && e == 0 && lane == 0;
      if (tr0) trace[it * 16 + 12] = gtimer();
      if (lane == 0) tc::mbar_wait_sleep(&tfull_bar, it & 1);
      __syncwarp();
      tc::fence_after_sync();
      if (tr0) trace[it * 16 + 8] = gtimer();
      // the partial dh of all 4 pairs' 16-unit slices in one TMEM round trip
      // the partial dh: my own 16 units, then each other pair's slice (packed and
      // sent right away — one 16-column slice live at a time keeps registers free)
      uint32_t own[kUT];
      tmem_ld16_nowait(tbase + k * kFU, own);
      tc::tmem_wait_ld();
#pragma unroll 1
      for (int pi = 1; pi < kKS; ++pi) {
        const int p = (k + pi) % kKS;
        uint32_t pr[kUT];
        tmem_ld16_nowait(tbase + p * kFU, pr);
        tc::tmem_wait_ld();
        if (pi == kKS - 1) {  // every column read: the accumulator may be overwritten
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote_relaxed(tempty_l, 32);
        }
        Bf16Vec<kUT> w;
#pragma unroll
        for (int i = 0; i < kUT; i += 2) {
          const __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(pr[i]), __uint_as_float(pr[i + 1]));
          w.w[i / 2] = *reinterpret_cast<const uint32_t*>(&b);
        }
        if (it > 0) {
          if (lane == 0) mbar_wait_cluster(&free_bar[p], (it - 1) & 1);
          __syncwarp();
        }
        const int slot_at_p = (k - p + kKS) % kKS - 1;  // my slot in p's receive buffer
        const uint32_t dst_rank = (uint32_t)(2 * p + h);
        const uint32_t dst = mapa(tc::smem_u32(recv + ((size_t)slot_at_p * 128 + rl) * kFU + hf * kUT), dst_rank);
        const uint32_t rbar = mapa(tc::smem_u32(&recv_full), dst_rank);
        st_async_v4(dst, make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]), rbar);
        st_async_v4(dst + 16, make_uint4(w.w[4], w.w[5], w.w[6], w.w[7]), rbar);
      }
      if (tr0) trace[it * 16 + 9] = gtimer();
      // the step's saved gates / c_{s-1} (L2-prefetched by the producer), loaded
      // while the peers' partials arrive
      Bf16Vec<kUT> gv[4], cp;
      if (active) {
#pragma unroll
        for (int g = 0; g < 4; ++g) gv[g].load(gates + gate_save_off(s, g, row, a.B, H, ut0), nu, true);
        cp.load(cprev + cprev_save_off(s, row, a.B, H, ut0), nu, true);
      }
      float dh[kUT];
#pragma unroll
      for (int i = 0; i < kUT; ++i) dh[i] = __uint_as_float(own[i]);
      mbar_wait_cluster(&recv_full, it & 1);
      if (e == 0 && lane == 0) tc::mbar_arrive_expect_tx(&recv_full, kRecvBytes);  // arm the next step
      if (tr0) trace[it * 16 + 10] = gtimer();
#pragma unroll
      for (int sl = 0; sl < kKS - 1; ++sl) {
        Bf16Vec<kUT> pv;
        pv.load_shared(recv + ((size_t)sl * 128 + rl) * kFU + hf * kUT);
#pragma unroll
        for (int i = 0; i < kUT; ++i) dh[i] += pv[i];
      }
      if (tr0) trace[it * 16 + 13] = gtimer();

      Bf16Vec<kUT> dzp[4];
      if (valid_row) {
        if (active) {
          const bool last = (s == len - 1);
          if (last && (a.dh_last || a.dc_last)) {
#pragma unroll
            for (int u = 0; u < kUT; ++u) {
              if (u >= nu) continue;
              if (a.dh_last) dh[u] += a.dh_last[((size_t)d * a.B + row) * H + ut0 + u];
              if (a.dc_last) gcar[u] += a.dc_last[((size_t)d * a.B + row) * H + ut0 + u];
            }
          }
          const float2 one = f2s(1.f), mone = f2s(-1.f);
          auto pk = [](float2 v) {  // two DZ values -> one packed bf16 word
            const __nv_bfloat162 b = __floats2bfloat162_rn(v.x, v.y);
            return *reinterpret_cast<const uint32_t*>(&b);
          };
#pragma unroll
          for (int u = 0; u < kUT; u += 2) {
            const float2 gh = add2(f2(dh[u], dh[u + 1]), f2(dyv[u], dyv[u + 1]));
            const float2 gc = f2(gcar[u], gcar[u + 1]);
            const float2 gi = bf16x2_f2(gv[0].w[u / 2]), gf = bf16x2_f2(gv[1].w[u / 2]);
            const float2 gg = bf16x2_f2(gv[2].w[u / 2]), go = bf16x2_f2(gv[3].w[u / 2]);
            const float2 cpu = bf16x2_f2(cp.w[u / 2]);
            const float2 tcv = tanh2(fma2(gf, cpu, mul2(gi, gg)));
            const float2 d_o = mul2(gh, tcv);                                           // tape.cpp:1161
            const float2 dcn = fma2(mul2(gh, go), fma2(mul2(mone, tcv), tcv, one), gc);  // tape.cpp:1162
            const float2 cg = mul2(dcn, gf);                                            // tape.cpp:1166
            gcar[u] = cg.x, gcar[u + 1] = cg.y;
            dzp[0].w[u / 2] = pk(mul2(mul2(dcn, gg), mul2(gi, fma2(mone, gi, one))));     // tape.cpp:1167
            dzp[1].w[u / 2] = pk(mul2(mul2(dcn, cpu), mul2(gf, fma2(mone, gf, one))));    // tape.cpp:1168
            dzp[2].w[u / 2] = pk(mul2(mul2(dcn, gi), fma2(mul2(mone, gg), gg, one)));     // tape.cpp:1169
            dzp[3].w[u / 2] = pk(mul2(mul2(d_o, go), fma2(mone, go, one)));               // tape.cpp:1170
          }
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g) dzp[g].zero();
        }
        if (tr0) trace[it * 16 + 14] = gtimer();
        // DZ_s into the interleaved ring: two 8-unit chunks per gate
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int c = 0; c < kUT; c += 8) {
            Bf16Vec<8> part;
#pragma unroll
            for (int w = 0; w < 4; ++w) part.w[w] = dzp[g].w[c / 2 + w];
            part.store(zr + dz_ring_off((it + 1) & 1, row, g * hq8 + ut0 + c, Bp, a.Kz), max(0, min(8, nu - c)));
          }
      }
      if (tr0) trace[it * 16 + 11] = gtimer();
      named_sync(1, kEpi);
      if (e == 0 && lane == 0) {
        tc::fence_proxy_async_global();
        red_release_gpu(ctr, 1u);
        for (int pi = 1; pi < kKS; ++pi)  // every sender's slot in my receive buffer is free again
          mbar_arrive_remote_relaxed(mapa(tc::smem_u32(&free_bar[k]), (uint32_t)(2 * ((k + pi) % kKS) + h)), kEpi);
        if (trace) trace[it * 16 + 6] = gtimer();
      }
      if (valid_row) {  // the K4 operand copy, off the cross-CTA critical path
        __nv_bfloat16* zc = a.dzcat + pos * a.dzcat_ld + (size_t)d * a.dz_dir_off + ut0;
#pragma unroll
        for (int g = 0; g < 4; ++g) dzp[g].store(zc + g * H, nu);
      }
    }
    if (valid_row) {  // DZ rows of positions beyond the longest sequence
      float zero[kUT];
#pragma unroll
      for (int u = 0; u < kUT; ++u) zero[u] = 0.f;
      for (int s = Tmax; s < T; ++s) {
        __nv_bfloat16* zc = a.dzcat + ((size_t)row * T + s) * a.dzcat_ld + (size_t)d * a.dz_dir_off + ut0;
#pragma unroll
        for (int g = 0; g < 4; ++g) store_bf16<kUT>(zc + g * H, zero, nu);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  cluster_sync();  // no CTA leaves while a peer may still touch its smem / TMEM
  if (warp == 1) tmem_dealloc_pair<kPU>(tmem);
}

// RB rows ((cl * 4 + k) * 2 + h) * 64 + n = unit cl * 128 + 64 h + n over the
// DZ-ring columns [k * Kc, (k + 1) * Kc) (gate stride dz_ring_hq(H)), bf16.
__global__ void pack_rb_pair_kernel(const float* __restrict__ R, int H, int Kc, int rows,
                                    __nv_bfloat16* __restrict__ RB) {
  const int rowi = blockIdx.x;
  if (rowi >= rows) return;
  const int n = rowi % 64, hh = (rowi / 64) % 2, kk_slice = (rowi / 128) % kKS, cl = rowi / (128 * kKS);
  const int unit = cl * kPU + 64 * hh + n;
  const int hq8 = dz_ring_hq(H);
  __nv_bfloat16* dst = RB + (size_t)rowi * Kc;
  for (int kk = threadIdx.x; kk < Kc; kk += blockDim.x) {
    const int col = kk_slice * Kc + kk, g = col / hq8, u = col % hq8;
    const float v = (unit < H && g < 4 && u < H) ? __ldg(R + (size_t)unit * 4 * H + (size_t)g * H + u) : 0.f;
    dst[kk] = __float2bfloat16_rn(v);
  }
}

}  // namespace

// Pair form: clusters of 8 covering 128 units; P = CTAs per direction.
// Opt-in (SL_BWD_PAIR=1): measured slower than the single-CTA form on B200 —
// the decoder-shaped layer (H = 1000, one direction) takes 1.68 ms vs 1.38 ms:
// the pair form halves the MMA issue and stream bytes per SM but loses the
// overlap of two independent batch-tile recurrences per CTA.  And the encoder's
// 2 x 8 clusters of 8 CTAs do not fit (at most 15 co-resident on 148 SMs).
bool tc_rec_bwd_pair_fits(int H, int nd, int sms, int B, TcBwdShape* out) {
  const char* env = getenv("SL_BWD_PAIR");
  if (!(env && env[0] == '1')) return false;
  const int ncl = (H + kPU - 1) / kPU;
  const int P = ncl * kCl;
  const int Kz = (int)round_up(4 * (int64_t)dz_ring_hq(H), 64 * kKS);
  if ((int64_t)P * nd > sms || bp_smem(Kz / kKS, 2, 2) > kSmemMax || (Kz / kKS) % 128 != 0) return false;
  (void)B;
  // every cluster of 8 must be co-resident (cooperative grid)
  static int max_clusters = -1;
  if (max_clusters < 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(P * nd);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = bp_smem(Kz / kKS, 2, 2);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = kCl;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaFuncSetAttribute(rec_bwd_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)cfg.dynamicSmemBytes) != cudaSuccess ||
        cudaOccupancyMaxActiveClusters(&n, rec_bwd_pair_kernel, &cfg) != cudaSuccess)
      n = 0;
    cudaGetLastError();  // a failed query must not leave an error behind for later checks
    max_clusters = n;
  }
  if (getenv("SL_DEBUG_SHAPES"))
    fprintf(stderr, "[seqloom] bwd pair: H=%d nd=%d P=%d Kz=%d smem=%u max_active_clusters=%d need=%d\n", H, nd,
            P, Kz, bp_smem(Kz / kKS, 2, 2), max_clusters, P * nd / kCl);
  if ((int64_t)max_clusters * kCl < (int64_t)P * nd) return false;
  if (out) *out = TcBwdShape{kCl, kFU, P, Kz};
  if (out) out->pair = 1;
  return true;
}

size_t tc_rec_bwd_pair_pack_elems(const TcBwdShape& sh) { return (size_t)sh.P * 64 * (sh.Kz / kKS); }

void tc_rec_bwd_pair_pack(const float* R, int H, const TcBwdShape& sh, __nv_bfloat16* RB, cudaStream_t stream) {
  const int rows = sh.P * 64;
  pack_rb_pair_kernel<<<rows, 256, 0, stream>>>(R, H, sh.Kz / kKS, rows, RB);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void rec_bwd_pair(const TcRecBwdArgs& a0, const TcBwdShape& sh, __nv_bfloat16* const* RB, cudaStream_t stream) {
  TcRecBwdArgs a = a0;
  a.U = kFU;
  a.P = sh.P;
  a.Kz = sh.Kz;
  const int Kc = sh.Kz / kKS;
  a.kb = (Kc / 64) % 2 == 0 ? 2 : 1;
  CUtensorMap tr[2], tz[2];
  for (int d = 0; d < a.nd; ++d) {
    cuuint64_t rd[2] = {(cuuint64_t)Kc, (cuuint64_t)sh.P * 64};
    cuuint64_t rs[1] = {(cuuint64_t)Kc * 2};
    cuuint32_t rb[2] = {64, 64};
    tr[d] = tmap(RB[d], 2, rd, rs, rb);
    const int Bp = dz_ring_bp(a.B);
    cuuint64_t zd[4] = {64, (cuuint64_t)Bp / 8, (cuuint64_t)a.Kz / 8, 2};
    cuuint64_t zs[3] = {128, (cuuint64_t)Bp * 16, (cuuint64_t)a.Kz / 8 * Bp * 16};
    cuuint32_t zb[4] = {64, 16, (cuuint32_t)a.kb * 8, 1};
    tz[d] = tmap(a.dzring[d], 4, zd, zs, zb, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  a.stages = 0;
  for (int st = kMaxStages; st >= 2 && !a.stages; --st)
    if (bp_smem(Kc, st, a.kb) <= kSmemMax) a.stages = st;
  SL_REQUIRE(a.stages >= 2, SL_ERR_UNSUPPORTED, "rec_bwd_pair: R slice does not fit in shared memory");
  const uint32_t smem = bp_smem(Kc, a.stages, a.kb);
  SL_CUDA_TRY(cudaFuncSetAttribute(rec_bwd_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CUtensorMap r0 = tr[0], r1 = tr[a.nd > 1 ? 1 : 0], z0 = tz[0], z1 = tz[a.nd > 1 ? 1 : 0];
  unsigned* bar0 = a.bar;
  for (int b0 = 0; b0 < a.B; b0 += 256) {
    a.b0 = b0;
    a.bar = bar0 + kBarPerChunk * (b0 / 256);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sh.P * a.nd);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = kCl;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeCooperative;
    attrs[1].val.cooperative = 1;
    cfg.attrs = attrs;
    static const bool no_coop = getenv("SL_NO_COOP") != nullptr;
    cfg.numAttrs = no_coop ? 1 : 2;
    SL_CUDA_TRY(cudaLaunchKernelEx(&cfg, rec_bwd_pair_kernel, r0, r1, z0, z1, a));
    count_launch();
  }
}

}  // namespace sl

#endif  // SL_EXPERIMENTS
