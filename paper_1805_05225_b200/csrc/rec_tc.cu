// K2 — persistent tensor-core forward recurrence (SL_PREC_BF16 path).
//
// One launch runs all T steps of both directions.  CTA c of direction d owns
// hidden units [c*U, c*U+U) and keeps its slice of R — the 4U gate columns of
// those units, all K = H rows, bf16 — RESIDENT in shared memory for the whole
// sequence (loaded once by TMA).  Per step s:
//   warp 0      waits on the direction's step counter (every CTA published
//               h_{s-1}), then TMA-streams h_{s-1} [128-row batch tile x 64]
//               bf16 chunks from the L2-resident ring buffer into a smem ring;
//   warp 1      issues tcgen05.mma (M = 128 batch rows, N = 4U gate columns,
//               K = 16) into TMEM: Z_rec = h_{s-1} . R[:, cols];
//   warps 2..   (4 per batch tile, one thread per batch row) tcgen05.ld the
//               accumulator, add the hoisted input projection x W + b (K1),
//               apply sigmoid / tanh, update the fp32 cell state held in
//               registers, and write h_s (bf16, ring buffer), y, and the
//               saved activations; then publish the step with one
//               release-increment of the direction counter.
// No kernel relaunch per step, no grid-wide cooperative sync: the only
// cross-CTA dependency is "all slices of h_{s-1} are written" (reference
// semantics: layers.cpp:27-33, tape.cpp:1103-1135; masking tape.cpp:797;
// per-sequence reversal tape.cpp:846).
#include <cudaTypedefs.h>

#include "profile.h"
#include "rec_tc.h"
#include "rec_tc_common.cuh"

namespace sl {
namespace {
using namespace rtc;

constexpr int kStages = 6;  // max h-tile ring depth
// h_s is written to kHCopies replicas of the ring and CTA c reads replica
// c % kHCopies: ~P/kHCopies CTAs (not all P) request each L2 line per step.
constexpr int kHCopies = 4;
constexpr uint32_t kHTileBytes = 128 * 64 * 2;  // 128 rows x 64 K bf16 = 16 KB
constexpr uint32_t kSmemMax = 227 * 1024;

uint32_t fwd_smem(int N, int Kp, int stages) {
  return (uint32_t)N * Kp * 2 + stages * kHTileBytes + 1024;
}

// U units per CTA (N = 4U), MT 128-row batch tiles.
template <int U, int MT, int SPLIT = (U >= 8 ? 2 : 1), int UT = U / SPLIT>
__global__ void __launch_bounds__(64 + 128 * MT * SPLIT, 1)
    rec_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmR0,
                      const __grid_constant__ CUtensorMap tmR1,
                      const __grid_constant__ CUtensorMap tmH0,
                      const __grid_constant__ CUtensorMap tmH1, TcRecFwdArgs a) {
  constexpr int N = 4 * U;
  constexpr int kEpi = 128 * MT * SPLIT;
  constexpr uint32_t kTmemCols = (MT * N <= 32) ? 32 : (MT * N <= 64) ? 64 : (MT * N <= 128) ? 128
                                 : (MT * N <= 256) ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t r_bar, tfull_bar[MT], tempty_bar[MT];
  __shared__ uint32_t tmem_sh;
  __shared__ int tmax_sh;

  const int d = blockIdx.x / a.P;
  const int cta = blockIdx.x % a.P;
  const int u0 = cta * U;
  const CUtensorMap* tmR = d == 0 ? &tmR0 : &tmR1;
  const CUtensorMap* tmH = d == 0 ? &tmH0 : &tmH1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t base = (tc::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - tc::smem_u32(smem_raw));
  const uint32_t r_bytes = (uint32_t)N * a.Kp * 2;
  uint8_t* sR = smem;
  uint8_t* sH = smem + r_bytes;
  const int nkc = a.Kp / 64;

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
      tc::mbar_init(&tempty_bar[m], kEpi / MT);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(&tmem_sh);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  {  // longest sequence (steps beyond it only need zero outputs)
    int m = 0;
    for (int i = threadIdx.x; i < a.B; i += blockDim.x) m = max(m, (int)a.lens[i]);
    atomicMax(&tmax_sh, m);
  }
  __syncthreads();
  const int Tmax = tmax_sh;
  const uint32_t tmem = tmem_sh;
  // One step counter per (direction, batch tile): the two 128-row tiles are
  // independent recurrences, so tile 0 of step s+1 streams and multiplies
  // while tile 1 of step s is still in its epilogue.
  unsigned* ctr = a.bar + d * 2;
  // Stagger the K-chunk order per CTA so the ~P CTAs of a direction do not
  // all pull the same 16 KB h tile from the same L2 lines at the same time.
  const int kc_off = cta % nkc;

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
          for (int kq = 0; kq < nkc; ++kq) {
            const int kc = (kq + kc_off) % nkc;
            tc::mbar_wait(&empty_bar[st], ph ^ 1);
            tc::mbar_arrive_expect_tx(&full_bar[st], kHTileBytes);
            tma_load_3d(sH + st * kHTileBytes, tmH, &full_bar[st], kc * 64, a.b0 + mt * 128,
                        (cta % kHCopies) * 2 + slot);
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
          for (int kq = 0; kq < nkc; ++kq) {
            const int kc = (kq + kc_off) % nkc;
            tc::mbar_wait(&full_bar[st], ph);
            tc::fence_after_sync();
            if (kq == 0) SL_TRACE(mt == 0 ? 1 : 4);
            if (kq == nkc - 1) SL_TRACE(mt == 0 ? 2 : 5);
            const uint32_t sa = base + r_bytes + st * kHTileBytes;
            const uint32_t sb = base + (uint32_t)kc * N * 128;
            if (!(a.debug_flags & 1))
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc::mma_f16(tmem + mt * N, tc::make_sdesc(sa + k * 32, 0, 1024),
                          tc::make_sdesc(sb + k * 32, 0, 1024), idesc, (kq | k) != 0);
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
    const int row = a.b0 + mt * 128 + q * 32 + lane;
    const bool valid_row = row < a.B;
    const int len = valid_row ? a.lens[row] : 0;
    const int dir = a.dirsign[d];
    const int H = a.H, T = a.T;
    const int lo = half * UT;          // first local unit of this thread
    const int ut0 = u0 + lo;           // first global unit
    const int nu = max(0, min(UT, H - ut0));
    const float* xw = a.xw[d];
    __nv_bfloat16* hb = a.hbuf[d];
    const bool save = a.gates[d] != nullptr;
    float cst[UT], hst[UT];
#pragma unroll
    for (int u = 0; u < UT; ++u) cst[u] = hst[u] = 0.f;

    for (int s = 0; s < Tmax; ++s) {
      const bool active = valid_row && s < len;
      const int t = active ? src_time(s, len, dir) : s;
      const size_t pos = (size_t)row * T + t;
      float xv[4 * UT];
      if (active) {
        const float* xr = xw + pos * a.xw_ld + ut0;
        if (nu == UT && (UT % 4) == 0 && ((uintptr_t)xr & 15) == 0 && (H % 4) == 0) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int u = 0; u < UT; u += 4) {
              const float4 v4 = __ldg(reinterpret_cast<const float4*>(xr + g * H + u));
              xv[g * UT + u] = v4.x;
              xv[g * UT + u + 1] = v4.y;
              xv[g * UT + u + 2] = v4.z;
              xv[g * UT + u + 3] = v4.w;
            }
        } else {
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int u = 0; u < UT; ++u) xv[g * UT + u] = (u < nu) ? __ldg(xr + g * H + u) : 0.f;
        }
      }
      float z[4 * UT];
      tc::mbar_wait(&tfull_bar[mt], s & 1);
      tc::fence_after_sync();
      {
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + mt * N + lo;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float v[UT];
          tmem_ld_cols<UT>(tbase + g * U, v);
#pragma unroll
          for (int u = 0; u < UT; ++u) z[g * UT + u] = v[u];
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&tempty_bar[mt]);

      if (valid_row && !(a.debug_flags & 2)) {
        __nv_bfloat16* hn = hb + ((size_t)((s + 1) & 1) * a.B + row) * a.Kp + ut0;
        if (active) {
          if (save) {  // c_{s-1}, h_{s-1} before the update
            store_f32<UT>(a.cprev[d] + pos * H + ut0, cst, nu);
            store_bf16<UT>(a.hprev[d] + pos * a.hprev_ld + ut0, hst, nu);
          }
#pragma unroll
          for (int u = 0; u < UT; ++u) {
            const float gi = tc::sigmoid_approx(z[u] + xv[u]);
            const float gf = tc::sigmoid_approx(z[UT + u] + xv[UT + u]);
            const float gg = tc::tanh_approx(z[2 * UT + u] + xv[2 * UT + u]);
            const float go = tc::sigmoid_approx(z[3 * UT + u] + xv[3 * UT + u]);
            z[u] = gi;
            z[UT + u] = gf;
            z[2 * UT + u] = gg;
            z[3 * UT + u] = go;
            const float cn = fmaf(gf, cst[u], gi * gg);
            cst[u] = cn;
            hst[u] = go * tc::tanh_approx(cn);
          }
          if (save) {
            float* gsave = a.gates[d] + pos * 4 * H + ut0;
#pragma unroll
            for (int g = 0; g < 4; ++g) store_f32<UT>(gsave + g * H, z + g * UT, nu);
          }
          if (a.y) store_f32<UT>(a.y + pos * a.y_ld + (size_t)d * H + ut0, hst, nu);
          if (a.ybf) store_bf16<UT>(a.ybf + pos * a.ybf_ld + (size_t)d * H + ut0, hst, nu);
        } else {  // padded position t == s: zero output (tape.cpp:797), frozen state
          float zero[UT];
#pragma unroll
          for (int u = 0; u < UT; ++u) zero[u] = 0.f;
          if (a.y) store_f32<UT>(a.y + pos * a.y_ld + (size_t)d * H + ut0, zero, nu);
          if (a.ybf) store_bf16<UT>(a.ybf + pos * a.ybf_ld + (size_t)d * H + ut0, zero, nu);
          if (save) store_bf16<UT>(a.hprev[d] + pos * a.hprev_ld + ut0, zero, nu);
        }
#pragma unroll
        for (int cp = 0; cp < kHCopies; ++cp) store_bf16<UT>(hn + (size_t)cp * 2 * a.B * a.Kp, hst, nu);
      }
      named_sync(1 + mt, kEpi / MT);  // the tile's epilogue threads only
      if ((e % (4 * SPLIT)) == 0 && lane == 0) {
        tc::fence_proxy_async_global();
        red_release_gpu(ctr + mt, 1u);
        SL_TRACE(6 + mt);
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
      for (int u = 0; u < nu; ++u) {
        if (a.h_last) a.h_last[((size_t)d * a.B + row) * H + ut0 + u] = hst[u];
        if (a.c_last) a.c_last[((size_t)d * a.B + row) * H + ut0 + u] = cst[u];
      }
    }
  }
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<kTmemCols>(tmem);
}

// RT[c*N + g*U + u][k] = R[k][g*H + c*U + u] (bf16), zero outside [H) x [H).
__global__ void pack_rt_kernel(const float* __restrict__ R, int H, int U, int P, int Kp,
                               __nv_bfloat16* __restrict__ RT) {
  const int N = 4 * U;
  const int64_t n = (int64_t)P * N * Kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e % Kp);
    const int r = (int)(e / Kp);
    const int c = r / N, j = r % N, g = j / U, u = j % U;
    const int unit = c * U + u;
    float v = 0.f;
    if (unit < H && k < H) v = R[(int64_t)k * 4 * H + (int64_t)g * H + unit];
    RT[e] = __float2bfloat16_rn(v);
  }
}

template <int U, int MT>
void launch_fwd(const CUtensorMap* tr, const CUtensorMap* th, const TcRecFwdArgs& a,
                cudaStream_t stream) {
  auto kern = rec_fwd_tc_kernel<U, MT>;
  const uint32_t smem = fwd_smem(4 * U, a.Kp, a.stages);
  SL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  TcRecFwdArgs copy = a;
  CUtensorMap r0 = tr[0], r1 = tr[a.nd > 1 ? 1 : 0], h0 = th[0], h1 = th[a.nd > 1 ? 1 : 0];
  void* params[] = {&r0, &r1, &h0, &h1, &copy};
  // Cooperative launch: guarantees every CTA is co-resident (they spin on each
  // other's step counters), and fails loudly instead of deadlocking if not.
  constexpr int kSplit = U >= 8 ? 2 : 1;
  SL_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(a.P * a.nd), dim3(64 + 128 * MT * kSplit),
                                          params, smem, stream));
  count_launch();
}

}  // namespace

int tc_rec_units(int H, int nd, int sms) {
  const int Kp = (int)round_up(H, 64);
  for (int U : {4, 8, 16})
    if ((int64_t)ceil_div(H, U) * nd <= sms && fwd_smem(4 * U, Kp, 2) <= kSmemMax) return U;
  return 0;
}

size_t tc_rec_hbuf_elems(int B, int H) { return (size_t)kHCopies * 2 * B * round_up(H, 64); }

size_t tc_rec_pack_elems(int H, int U) {
  const int P = (int)ceil_div(H, U);
  return (size_t)P * 4 * U * round_up(H, 64);
}

void tc_rec_pack(const float* R, int H, int U, __nv_bfloat16* RT, cudaStream_t stream) {
  const int P = (int)ceil_div(H, U);
  const int Kp = (int)round_up(H, 64);
  const int64_t n = (int64_t)P * 4 * U * Kp;
  pack_rt_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 148 * 16), 256, 0, stream>>>(
      R, H, U, P, Kp, RT);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void rec_fwd_tc(const TcRecFwdArgs& a0, __nv_bfloat16* const* RT, cudaStream_t stream) {
  TcRecFwdArgs a = a0;
  const int N = 4 * a.U;
  CUtensorMap tr[2], th[2];
  for (int k = 0; k < a.nd; ++k) {
    cuuint64_t rd[2] = {(cuuint64_t)a.Kp, (cuuint64_t)a.P * N};
    cuuint64_t rs[1] = {(cuuint64_t)a.Kp * 2};
    cuuint32_t rb[2] = {64, (cuuint32_t)N};
    tr[k] = tmap(RT[k], 2, rd, rs, rb);
    cuuint64_t hd[3] = {(cuuint64_t)a.Kp, (cuuint64_t)a.B, (cuuint64_t)2 * kHCopies};
    cuuint64_t hs[2] = {(cuuint64_t)a.Kp * 2, (cuuint64_t)a.Kp * 2 * a.B};
    cuuint32_t hbx[3] = {64, 128, 1};
    th[k] = tmap(a.hbuf[k], 3, hd, hs, hbx);
  }
  a.stages = 0;
  for (int st = kStages; st >= 2 && !a.stages; --st)
    if (fwd_smem(N, a.Kp, st) <= kSmemMax) a.stages = st;
  SL_REQUIRE(a.stages >= 2, SL_ERR_UNSUPPORTED, "rec_fwd_tc: R slice does not fit in shared memory");
  unsigned* bar0 = a.bar;
  for (int b0 = 0; b0 < a.B; b0 += 256) {  // batch chunks of up to two 128-row tiles
    a.b0 = b0;
    a.bar = bar0 + 4 * (b0 / 256);  // fresh zeroed counters per chunk (2 dirs x 2 tiles)
    const int MT = (a.B - b0) > 128 ? 2 : 1;
    switch (a.U * 10 + MT) {
      case 41: launch_fwd<4, 1>(tr, th, a, stream); break;
      case 42: launch_fwd<4, 2>(tr, th, a, stream); break;
      case 81: launch_fwd<8, 1>(tr, th, a, stream); break;
      case 82: launch_fwd<8, 2>(tr, th, a, stream); break;
      case 161: launch_fwd<16, 1>(tr, th, a, stream); break;
      case 162: launch_fwd<16, 2>(tr, th, a, stream); break;
      default: throw Error{SL_ERR_UNSUPPORTED, "rec_fwd_tc: unsupported units per CTA"};
    }
  }
}

}  // namespace sl
