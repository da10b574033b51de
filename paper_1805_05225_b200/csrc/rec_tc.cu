// K2 — persistent tensor-core forward recurrence (SL_PREC_BF16 path).
//
// One launch runs all T steps of both directions.  The hidden units of a
// direction are split over clusters of C CTAs; a cluster owns UC = C*U units
// (its N = 4*UC gate columns) and K-splits the recurrent product over its C
// CTAs: CTA r keeps R[K-slice r, the cluster's gate columns] (bf16, K-major)
// RESIDENT in shared memory for the whole sequence.  Per step s:
//   warp 0      waits on the step counter of the (direction, batch tile) —
//               every CTA published its slice of h_{s-1} — then TMA-streams
//               ITS K-slice of h_{s-1} [128-row tile x 64] from the L2 ring;
//   warp 1      tcgen05.mma M = 128 batch rows x N = 4*UC (128 for C=2,U=16:
//               the measured full-rate MMA width) x K = 16 into TMEM: the
//               partial Z_rec over the CTA's K-slice;
//   warps 2..   two threads per batch row: tcgen05.ld the partial columns of
//               the peers' units and push them to the peers through DSMEM
//               (st.shared::cluster.v4, one remote mbarrier arrive per warp),
//               add the peers' partials for the own units, add x W + b (K1),
//               apply sigmoid / tanh (SFU), update the fp32 cell state held in
//               registers, and write h_s (bf16 ring), y and the saved
//               activations; then release-increment the tile's step counter.
// No relaunch and no grid-wide sync per step.  The two 128-row batch tiles are
// independent recurrences with their own counters, so one tile's epilogue
// overlaps the other's loads and MMAs.  Reference semantics: layers.cpp:27-33,
// tape.cpp:1103-1135 (step), tape.cpp:797 (mask), tape.cpp:846 (reversal).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "profile.h"
#include "rec_tc.h"
#include "rec_tc_common.cuh"

namespace sl {
namespace {
using namespace rtc;

constexpr int kStages = 6;                      // max h-tile ring depth
constexpr uint32_t kHTileBytes = 128 * 64 * 2;  // 128 rows x 64 K bf16 = 16 KB
constexpr uint32_t kSmemMax = 227 * 1024;

// R slice + h ring stages + per batch tile the (C-1) peers' partials [128 rows][4U] bf16
uint32_t fwd_smem(int C, int U, int Kc, int stages) {
  const uint32_t recv = C > 1 ? (uint32_t)2 * (C - 1) * 128 * 4 * U * 2 : 0;
  return (uint32_t)4 * C * U * Kc * 2 + stages * kHTileBytes * 2 + recv + 1024;
}

template <int C, int U, int MT, int SPLIT = (U >= 8 ? 2 : 1), int UT = U / SPLIT>
__global__ void __launch_bounds__(64 + 128 * MT * SPLIT, 1)
    rec_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmR0,
                      const __grid_constant__ CUtensorMap tmR1,
                      const __grid_constant__ CUtensorMap tmH0,
                      const __grid_constant__ CUtensorMap tmH1, TcRecFwdArgs a) {
  constexpr int UC = C * U;   // units per cluster
  constexpr int N = 4 * UC;   // MMA N: the cluster's gate columns, ordered (gate, unit)
  constexpr int kEpiTile = 128 * SPLIT;
  constexpr uint32_t kTmemCols = (MT * N <= 32) ? 32 : (MT * N <= 64) ? 64 : (MT * N <= 128) ? 128
                                 : (MT * N <= 256) ? 256 : 512;
  constexpr int RS = 4 * U;   // recv row stride (bf16): 4 gates x U units
  constexpr uint32_t kRecvBytes = (uint32_t)(C - 1) * 128 * RS * 2;  // per tile and step
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t r_bar, tfull_bar[MT], tempty_bar[MT];
  __shared__ __align__(8) uint64_t recv_full[MT], free_bar[MT][C];
  __shared__ uint32_t tmem_sh;
  __shared__ int tmax_sh;

  const int d = blockIdx.x / a.P;
  const int cta = blockIdx.x % a.P;
  const int r = C > 1 ? (int)cluster_rank() : 0;
  const int cl = cta / C;
  const int u0 = cl * UC + r * U;  // first unit this CTA finalizes
  const int Kc = a.Kp / C;
  const CUtensorMap* tmR = d == 0 ? &tmR0 : &tmR1;
  const CUtensorMap* tmH = d == 0 ? &tmH0 : &tmH1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t base = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - tc::smem_u32(smem_raw));
  const uint32_t r_bytes = (uint32_t)N * Kc * 2;
  uint8_t* sR = smem;
  uint8_t* sH = smem + r_bytes;
  const uint32_t stage_bytes = kHTileBytes * a.kb;  // a.kb 64-wide K chunks per TMA box
  // [MT][C-1][128][RS] bf16: one buffer per batch tile so the tiles stay independent
  __nv_bfloat16* recv = reinterpret_cast<__nv_bfloat16*>(sH + a.stages * stage_bytes);
  const int nkc = Kc / 64;

  if (threadIdx.x == 0) {
    tmax_sh = 0;
    tc::prefetch_tmap(tmR);
    tc::prefetch_tmap(tmH);
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
      tc::mbar_init(&recv_full[m], 1);  // armed once per step; the peers' st.async complete it
      for (int p = 0; p < C; ++p) tc::mbar_init(&free_bar[m][p], kEpiTile);
    }
    tc::fence_barrier_init();
    if (C > 1)
      for (int m = 0; m < MT; ++m) tc::mbar_arrive_expect_tx(&recv_full[m], kRecvBytes);
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(&tmem_sh);
  tc::fence_before_sync();
  __syncthreads();
  if constexpr (C > 1) cluster_sync();
  tc::fence_after_sync();
  {  // longest sequence (steps beyond it only need zero outputs)
    int m = 0;
    for (int i = threadIdx.x; i < a.B; i += blockDim.x) m = max(m, (int)a.lens[i]);
    atomicMax(&tmax_sh, m);
  }
  __syncthreads();
  const int Tmax = tmax_sh;
  const uint32_t tmem = tmem_sh;
  // one step counter per (direction, batch tile)
  unsigned* ctr = a.bar + d * 2;
  const int ngrp = nkc / a.kb;  // TMA boxes per tile
  const int kc_off = cta % ngrp;

  if (warp == 0) {
    if (lane == 0) {  // -------------------------------------------- producer
      tc::mbar_arrive_expect_tx(&r_bar, r_bytes);
      for (int kc = 0; kc < nkc; ++kc)
        tc::tma_load_2d(sR + (size_t)kc * N * 128, tmR, &r_bar, kc * 64, cta * N);
      int st = 0;
      uint32_t ph = 0;
      const int nst = a.stages;
      for (int s = 0; s < Tmax; ++s) {
        const int slot = s & 1;  // ring slot holding h_{s-1}
        for (int mt = 0; mt < MT; ++mt) {
          if (s > 0) {
            const unsigned target = (unsigned)a.P * (unsigned)s;
            while (ld_acquire(ctr + mt) < target) {
            }
            tc::fence_proxy_async_global();
          }
          SL_TRACE(mt == 0 ? 0 : 3);
          for (int kq = 0; kq < ngrp; ++kq) {
            const int kg = (kq + kc_off) % ngrp;
            tc::mbar_wait(&empty_bar[st], ph ^ 1);
            tc::mbar_arrive_expect_tx(&full_bar[st], stage_bytes);
            tma_load_4d(sH + st * stage_bytes, tmH, &full_bar[st], 0, a.b0 + mt * 128,
                        r * (Kc / 64) + kg * a.kb, slot);
            if (++st == nst) {
              st = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // -------------------------------------------- MMA issuer
      constexpr uint32_t idesc = tc::make_idesc(128, N, 1, false, false);
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
            if (kq == 0) SL_TRACE(mt == 0 ? 1 : 4);
            if (kq == ngrp - 1) SL_TRACE(mt == 0 ? 2 : 5);
            for (int j = 0; j < a.kb; ++j) {
            const int kc = kg * a.kb + j;
            const uint32_t sa = base + r_bytes + st * stage_bytes + j * kHTileBytes;
            const uint32_t sb = base + (uint32_t)kc * N * 128;
#ifdef SL_EXPERIMENTS
            if (!(a.debug_flags & 1))
#endif
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc::mma_f16(tmem + mt * N, tc::make_sdesc(sa + k * 32, 0, 1024),
                            tc::make_sdesc(sb + k * 32, 0, 1024), idesc, (kq | j | k) != 0);
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
    // SPLIT threads per batch row, UT units each; warps e = 0.. in groups of 4
    // cover the four TMEM lane quarters (a warp may only touch quarter warp % 4).
    const int e = warp - 2;
    const int mt = e / (4 * SPLIT);
    const int half = (e / 4) % SPLIT;
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    const int row = a.b0 + mt * 128 + rl;
    const bool valid_row = row < a.B;
    const int len = valid_row ? a.lens[row] : 0;
    const int dir = a.dirsign[d];
    const int H = a.H, T = a.T;
    const int lo = half * UT;   // first local unit of this thread (within the CTA's U)
    const int ut0 = u0 + lo;    // first global unit
    const int nu = max(0, min(UT, H - ut0));
    const __nv_bfloat16* xw = a.xw[d];
    __nv_bfloat16* hb = a.hbuf[d];
    const bool save = a.gates[d] != nullptr;
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + mt * N;
    float cst[UT], hst[UT];
#pragma unroll
    for (int u = 0; u < UT; ++u) cst[u] = hst[u] = 0.f;

    for (int s = 0; s < Tmax; ++s) {
      const int use = s;  // this tile's exchange buffer is used once per step
      const bool active = valid_row && s < len;
      const int t = active ? src_time(s, len, dir) : s;
      const size_t pos = (size_t)row * T + t;
      Bf16Vec<UT> xv[4];
      if (active) {  // prefetch (before the MMA wait): hoisted input projection x W + b of this step (K1 output)
        const __nv_bfloat16* xr = xw + pos * a.xw_ld + ut0;
        const bool vec = (H % 8) == 0 && (a.xw_ld % 8) == 0;
#pragma unroll
        for (int g = 0; g < 4; ++g) xv[g].load(xr + g * H, nu, vec);
      }
      float z[4 * UT];
      const bool tr0 = a.trace && blockIdx.x == a.trace_cta && e == 0 && lane == 0;
      if (tr0) a.trace[s * 16 + 12] = gtimer();
      tc::mbar_wait(&tfull_bar[mt], s & 1);
      tc::fence_after_sync();
      if (tr0) a.trace[s * 16 + 8] = gtimer();
      if constexpr (C > 1) {  // push the peers' columns of my partial Z
#pragma unroll 1
        for (int pi = 1; pi < C; ++pi) {
          const int p = (r + pi) % C;
          if (use > 0) mbar_wait_cluster(&free_bar[mt][p], (use - 1) & 1);
          const int slot_at_p = (r - p + C) % C - 1;  // my slot in p's buffer
          const uint32_t dst =
              mapa(tc::smem_u32(recv + (((size_t)mt * (C - 1) + slot_at_p) * 128 + rl) * RS + lo), p);
          const uint32_t rbar = mapa(tc::smem_u32(&recv_full[mt]), p);
          static_assert(UT % 4 == 0, "partial sends move 4 or 8 bf16 per store");
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float v[UT];
            tmem_ld_cols<UT>(tbase + g * UC + p * U + lo, v);
            Bf16Vec<UT> w;
            w.pack(v);
            const uint32_t dg = dst + g * U * 2;
            if constexpr (UT % 8 == 0) {
#pragma unroll
              for (int u = 0; u < UT; u += 8)
                st_async_v4(dg + u * 2, make_uint4(w.w[u / 2], w.w[u / 2 + 1], w.w[u / 2 + 2], w.w[u / 2 + 3]),
                            rbar);
            } else {
#pragma unroll
              for (int u = 0; u < UT; u += 4) st_async_v2(dg + u * 2, make_uint2(w.w[u / 2], w.w[u / 2 + 1]), rbar);
            }
          }
        }
      }
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float v[UT];
        tmem_ld_cols<UT>(tbase + g * UC + r * U + lo, v);
#pragma unroll
        for (int u = 0; u < UT; ++u) z[g * UT + u] = v[u];
      }
      if (tr0) a.trace[s * 16 + 9] = gtimer();
      tc::fence_before_sync();
      tc::mbar_arrive(&tempty_bar[mt]);
      if constexpr (C > 1) {
        mbar_wait_cluster(&recv_full[mt], use & 1);
        if ((e % (4 * SPLIT)) == 0 && lane == 0)  // step `use` is complete: arm the next one
          tc::mbar_arrive_expect_tx(&recv_full[mt], kRecvBytes);
        if (tr0) a.trace[s * 16 + 10] = gtimer();
#pragma unroll 1
        for (int pi = 0; pi < C - 1; ++pi) {
          const __nv_bfloat16* src = recv + (((size_t)mt * (C - 1) + pi) * 128 + rl) * RS + lo;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            Bf16Vec<UT> v;
            v.load_shared(src + g * U);
#pragma unroll
            for (int u = 0; u < UT; ++u) z[g * UT + u] += v[u];
          }
        }
        __syncwarp();
        if (lane == 0)  // every sender's slot in my buffer is free again
          for (int pi = 1; pi < C; ++pi)
            mbar_arrive_remote_relaxed(mapa(tc::smem_u32(&free_bar[mt][r]), (r + pi) % C), 32);
      }

#ifdef SL_EXPERIMENTS
      if (valid_row && !(a.debug_flags & 2)) {
#else
      if (valid_row) {
#endif
        if (active) {
#pragma unroll
          for (int u = 0; u < UT; ++u) {
            const float gi = tc::sigmoid_approx(z[u] + xv[0][u]);
            const float gf = tc::sigmoid_approx(z[UT + u] + xv[1][u]);
            const float gg = tc::tanh_approx(z[2 * UT + u] + xv[2][u]);
            const float go = tc::sigmoid_approx(z[3 * UT + u] + xv[3][u]);
            z[u] = gi;
            z[UT + u] = gf;
            z[2 * UT + u] = gg;
            z[3 * UT + u] = go;
            const float cn = fmaf(gf, cst[u], gi * gg);
            cst[u] = cn;
            hst[u] = go * tc::tanh_approx(cn);
          }
        }
        // only h_s is on the cross-CTA critical path: write it, publish, and
        // store everything else (saves, y) afterwards
        store_bf16<UT>(hb + ((size_t)((s + 1) & 1) * a.B + row) * a.Kp + ut0, hst, nu);
      }
      if (tr0) a.trace[s * 16 + 11] = gtimer();
      named_sync(1 + mt, kEpiTile);  // the tile's epilogue threads only
      if ((e % (4 * SPLIT)) == 0 && lane == 0) {
        tc::fence_proxy_async_global();
        red_release_gpu(ctr + mt, 1u);
        SL_TRACE(6 + mt);
      }
#ifdef SL_EXPERIMENTS
      if (valid_row && !(a.debug_flags & 2)) {
#else
      if (valid_row) {
#endif
        if (active) {
          if (save) {
#pragma unroll
            for (int g = 0; g < 4; ++g)
              store_bf16<UT>(a.gates[d] + gate_save_off(s, g, row, a.B, H, ut0), z + g * UT, nu);
          }
          if (a.y) store_f32<UT>(a.y + pos * a.y_ld + (size_t)d * H + ut0, hst, nu);
          if (a.ybf) store_bf16<UT>(a.ybf + pos * a.ybf_ld + (size_t)d * H + ut0, hst, nu);
          if (save) {  // saved (c, h)_{prev}: zeros at step 0, (c_s, h_s) at step s + 1's position
            if (s == 0) {
              float zero[UT];
#pragma unroll
              for (int u = 0; u < UT; ++u) zero[u] = 0.f;
              store_bf16<UT>(a.cprev[d] + cprev_save_off(0, row, a.B, H, ut0), zero, nu);
              store_bf16<UT>(a.hprev[d] + pos * a.hprev_ld + ut0, zero, nu);
            }
            if (s + 1 < len) {
              const size_t pn = (size_t)row * T + src_time(s + 1, len, dir);
              store_bf16<UT>(a.cprev[d] + cprev_save_off(s + 1, row, a.B, H, ut0), cst, nu);
              store_bf16<UT>(a.hprev[d] + pn * a.hprev_ld + ut0, hst, nu);
            }
          }
        } else {  // padded position t == s: zero output (tape.cpp:797), frozen state
          float zero[UT];
#pragma unroll
          for (int u = 0; u < UT; ++u) zero[u] = 0.f;
          if (a.y) store_f32<UT>(a.y + pos * a.y_ld + (size_t)d * H + ut0, zero, nu);
          if (a.ybf) store_bf16<UT>(a.ybf + pos * a.ybf_ld + (size_t)d * H + ut0, zero, nu);
          if (save) store_bf16<UT>(a.hprev[d] + pos * a.hprev_ld + ut0, zero, nu);
        }
      }
    }
    // positions beyond the longest sequence, final states
    if (valid_row) {
      float zero[UT];
#pragma unroll
      for (int u = 0; u < UT; ++u) zero[u] = 0.f;
      for (int s = Tmax; s < T; ++s) {
        const size_t pos = (size_t)row * T + s;
        if (a.y) store_f32<UT>(a.y + pos * a.y_ld + (size_t)d * H + ut0, zero, nu);
        if (a.ybf) store_bf16<UT>(a.ybf + pos * a.ybf_ld + (size_t)d * H + ut0, zero, nu);
        if (save) store_bf16<UT>(a.hprev[d] + pos * a.hprev_ld + ut0, zero, nu);
      }
#pragma unroll
      for (int u = 0; u < UT; ++u) {
        if (u >= nu) continue;
        if (a.h_last) a.h_last[((size_t)d * a.B + row) * H + ut0 + u] = hst[u];
        if (a.c_last) a.c_last[((size_t)d * a.B + row) * H + ut0 + u] = cst[u];
      }
    }
  }
  __syncthreads();
  if constexpr (C > 1) cluster_sync();  // no CTA leaves while a peer may still touch its smem
  if (warp == 1) tc::tmem_dealloc<kTmemCols>(tmem);
}

// RT[(cl*C + r)*N + g*UC + j][kk] = R[r*Kc + kk][g*H + cl*UC + j]  (bf16, zero outside)
// Generic (K-split) form: a 32x32 shared-memory transpose over (packed row, k).
__global__ void pack_rt_kernel(const float* __restrict__ R, int H, int C, int U, int P, int Kc,
                               __nv_bfloat16* __restrict__ RT) {
  __shared__ float tile[32][33];
  const int UC = C * U, N = 4 * UC;
  const int Kp = Kc * C;
  const int row0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8 threads
  for (int i = ty; i < 32; i += 8) {
    const int k = k0 + i, rowi = row0 + tx;
    float v = 0.f;
    if (rowi < P * N && k < H) {
      const int cta = rowi / N, j = rowi % N;
      const int cl = cta / C, r = cta % C;
      const int g = j / UC, unit = cl * UC + j % UC;
      if (unit < H && k / Kc == r) v = R[(size_t)k * 4 * H + (size_t)g * H + unit];
    }
    tile[i][tx] = v;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int rowi = row0 + i, k = k0 + tx;
    if (rowi >= P * N || k >= Kp) continue;
    const int r = (rowi / N) % C;
    if (k / Kc != r) continue;
    RT[(size_t)rowi * Kc + (k - r * Kc)] = __float2bfloat16_rn(tile[tx][i]);
  }
}

// No K split (C = 1): the rows (cta, g, j) of one (cta, gate) are UC consecutive
// columns of R, so each block transposes a [64 k x UC columns] tile: float4
// loads along the columns, 16 B bf16 stores along k.  grid = (P * 4, Kp / 64).
template <int UC>
__global__ void __launch_bounds__(256) pack_rt_c1_kernel(const float* __restrict__ R, int H, int Kp,
                                                         __nv_bfloat16* __restrict__ RT) {
  __shared__ float tile[64][UC + 1];
  const int cg = blockIdx.x;            // (cta, gate)
  const int cta = cg / 4, g = cg % 4;
  const int k0 = blockIdx.y * 64;
  const int c0 = g * H + cta * UC;      // first R column of the tile
  const int units_here = min(UC, H - cta * UC);
  const bool vec = (H % 4) == 0 && units_here == UC;
  constexpr int CV = UC / 4;            // float4 per tile row
  for (int e = threadIdx.x; e < 64 * CV; e += 256) {
    const int i = e / CV, cq = (e % CV) * 4;
    const int k = k0 + i;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (k < H) {
      const float* src = R + (size_t)k * 4 * H + c0 + cq;
      if (vec) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(src));
        v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (cq + u < units_here) v[u] = __ldg(src + u);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) tile[i][cq + u] = v[u];
  }
  __syncthreads();
  // 8 k per thread-store: UC rows x 8 chunks of 8 bf16
  for (int e = threadIdx.x; e < UC * 8; e += 256) {
    const int j = e / 8, kq = (e % 8) * 8;
    float f[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) f[u] = tile[kq + u][j];
    *reinterpret_cast<uint4*>(RT + ((size_t)cta * 4 * UC + g * UC + j) * Kp + k0 + kq) = pack8_bf16(f);
  }
}

template <int C, int U, int MT>
void launch_fwd(const CUtensorMap* tr, const CUtensorMap* th, const TcRecFwdArgs& a,
                cudaStream_t stream) {
  auto kern = rec_fwd_tc_kernel<C, U, MT>;
  const uint32_t smem = fwd_smem(C, U, a.Kp / C, a.kb == 2 ? a.stages : (a.stages + 1) / 2);
  SL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  TcRecFwdArgs copy = a;
  CUtensorMap r0 = tr[0], r1 = tr[a.nd > 1 ? 1 : 0], h0 = th[0], h1 = th[a.nd > 1 ? 1 : 0];
  constexpr int kSplit = U >= 8 ? 2 : 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.P * a.nd);
  cfg.blockDim = dim3(64 + 128 * MT * kSplit);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  // cooperative: every CTA co-resident (they wait on each other's step
  // counters) — the launch fails loudly instead of deadlocking otherwise
  attrs[0].id = cudaLaunchAttributeCooperative;
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
  SL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, r0, r1, h0, h1, copy));
  count_launch();
}

}  // namespace

TcFwdShape tc_rec_fwd_shape(int H, int nd, int sms) {
  // the CTA-pair kernel (M = 256 x N = 128 MMAs, 32 units per pair) where it fits;
  // otherwise the single-CTA form.  (2-CTA K-split clusters, N = 4*C*U = 128, trade
  // the h stream for a DSMEM partial exchange: measured slower, experiments builds only.)
#ifdef SL_EXPERIMENTS
  const char* env = getenv("SL_FWD_CLUSTER");
  const bool cluster = env && env[0] == '1';
#else
  constexpr bool cluster = false;
#endif
  if (!cluster && tc_rec_fwd_pair_fits(H, nd, sms)) {
    const int pu = tc_rec_fwd_pair_units(H, nd, sms);
    TcFwdShape sh{1, pu, (int)ceil_div(H, pu), (int)round_up(H, 64)};
    sh.pair = 1;
    return sh;
  }
  for (int C : {2, 1})
    for (int U : {16, 8, 4}) {
      const int P = (int)ceil_div(H, (int64_t)C * U) * C;
      const int Kp = (int)round_up(H, 64 * C);
      if ((C == 1 || cluster) && 4 * C * U <= 128 && (int64_t)P * nd <= sms &&
          fwd_smem(C, U, Kp / C, 2) <= kSmemMax && ((int64_t)ceil_div(H, (int64_t)C * U / 2) * C * nd > sms || U == 4))
        return TcFwdShape{C, U, P, Kp};
    }
  return TcFwdShape{0, 0, 0, 0};
}

size_t tc_rec_hbuf_elems(int B, const TcFwdShape& sh) { return (size_t)2 * dz_ring_bp(B) * sh.Kp; }

size_t tc_rec_pack_elems(const TcFwdShape& sh) {
  return (size_t)sh.P * 4 * sh.C * sh.U * (sh.Kp / sh.C);
}

void tc_rec_pack(const float* R, int H, const TcFwdShape& sh, __nv_bfloat16* RT,
                 cudaStream_t stream) {
  const int Kc = sh.Kp / sh.C;
  if (sh.C == 1 && (sh.U == 16 || sh.U == 32) && sh.Kp % 64 == 0) {
    const dim3 grid((unsigned)sh.P * 4, (unsigned)(sh.Kp / 64));
    if (sh.U == 32) pack_rt_c1_kernel<32><<<grid, 256, 0, stream>>>(R, H, sh.Kp, RT);
    else pack_rt_c1_kernel<16><<<grid, 256, 0, stream>>>(R, H, sh.Kp, RT);
  } else {
    const dim3 grid((unsigned)ceil_div((int64_t)sh.P * 4 * sh.C * sh.U, 32), (unsigned)ceil_div(sh.Kp, 32));
    pack_rt_kernel<<<grid, 256, 0, stream>>>(R, H, sh.C, sh.U, sh.P, Kc, RT);
  }
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void rec_fwd_tc(const TcRecFwdArgs& a0, const TcFwdShape& sh, __nv_bfloat16* const* RT,
                cudaStream_t stream) {
  if (sh.pair) {
    rec_fwd_pair(a0, sh, RT, stream);
    return;
  }
  TcRecFwdArgs a = a0;
  a.U = sh.U;
  a.P = sh.P;
  a.Kp = sh.Kp;
  const int N = 4 * sh.C * sh.U;
  const int Kc = sh.Kp / sh.C;
  CUtensorMap tr[2], th[2];
  for (int k = 0; k < a.nd; ++k) {
    cuuint64_t rd[2] = {(cuuint64_t)Kc, (cuuint64_t)a.P * N};
    cuuint64_t rs[1] = {(cuuint64_t)Kc * 2};
    cuuint32_t rb[2] = {64, (cuuint32_t)N};
    tr[k] = tmap(RT[k], 2, rd, rs, rb);
    // {k_in 64, rows, k_chunk, slot}: one TMA box = kb consecutive 64-wide chunks
    a.kb = (Kc / 64) % 2 == 0 ? 2 : 1;
    cuuint64_t hd[4] = {64, (cuuint64_t)a.B, (cuuint64_t)a.Kp / 64, 2};
    cuuint64_t hs[3] = {(cuuint64_t)a.Kp * 2, 128, (cuuint64_t)a.Kp * 2 * a.B};
    cuuint32_t hbx[4] = {64, 128, (cuuint32_t)a.kb, 1};
    th[k] = tmap(a.hbuf[k], 4, hd, hs, hbx);
  }
  a.stages = 0;  // stages of a.kb chunks (fwd_smem counts two chunks per stage)
  for (int st = kStages; st >= 2 && !a.stages; --st)
    if (fwd_smem(sh.C, sh.U, Kc, a.kb == 2 ? st : (st + 1) / 2) <= kSmemMax) a.stages = st;
  SL_REQUIRE(a.stages >= 2, SL_ERR_UNSUPPORTED, "rec_fwd_tc: R slice does not fit in shared memory");
  unsigned* bar0 = a.bar;
  for (int b0 = 0; b0 < a.B; b0 += 256) {  // batch chunks of up to two 128-row tiles
    a.b0 = b0;
    a.bar = bar0 + kBarPerChunk * (b0 / 256);  // fresh zeroed counters per chunk
    const int MT = (a.B - b0) > 128 ? 2 : 1;
    switch (sh.C * 1000 + sh.U * 10 + MT) {
#define SL_FWD_CASE(C_, U_, MT_) \
  case C_ * 1000 + U_ * 10 + MT_: launch_fwd<C_, U_, MT_>(tr, th, a, stream); break;
      SL_FWD_CASE(2, 4, 1) SL_FWD_CASE(2, 4, 2) SL_FWD_CASE(2, 8, 1) SL_FWD_CASE(2, 8, 2)
      SL_FWD_CASE(2, 16, 1) SL_FWD_CASE(2, 16, 2) SL_FWD_CASE(1, 4, 1) SL_FWD_CASE(1, 4, 2)
      SL_FWD_CASE(1, 8, 1) SL_FWD_CASE(1, 8, 2) SL_FWD_CASE(1, 16, 1) SL_FWD_CASE(1, 16, 2)
#undef SL_FWD_CASE
      default: throw Error{SL_ERR_UNSUPPORTED, "rec_fwd_tc: unsupported partition"};
    }
  }
}

}  // namespace sl
