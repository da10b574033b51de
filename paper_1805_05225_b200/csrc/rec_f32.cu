// FP32 persistent recurrence kernels (SL_PREC_FP32 path).
//
// One cooperative launch runs ALL T steps of BOTH directions: CTAs
// [d*P, (d+1)*P) own direction d, and CTA c of a direction owns hidden units
// [c*U, c*U+U) — all four gate columns of each unit, so the gate math, the
// cell update and the output of a unit never leave the CTA.  Per step the
// CTA computes Z[:, its 4U cols] = h_{s-1} . R[:, cols] on FP32 FMA units,
// adds the hoisted input projection (x W + b, computed once for all T by the
// K1 GEMM), applies the gates and writes h_s; then a per-direction flag
// barrier (no kernel relaunch) publishes h_s to every CTA of the direction.
//
// Reference semantics (layers.cpp:8-37, tape.cpp:1074-1222, tape.cpp:785-877):
// zero initial state, gate order (i,f,g,o), direction -1 reverses each
// sequence's valid prefix (src_time), padded outputs exactly 0.  Rows whose
// sequence has ended are frozen instead of stepping on padding: their outputs
// are masked by the reference anyway and their gradients are exactly zero,
// so every valid output and gradient is unchanged (SURVEY §7 hard part 6).
#include "profile.h"
#include "recurrence.h"

namespace sl {
namespace {

constexpr int NT = 256;  // threads per CTA; one batch row per thread per row-block
constexpr int KT = 32;   // K tile

__device__ int block_max_len(const int32_t* lens, int B) {
  __shared__ int smax;
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  int m = 0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) m = max(m, (int)lens[i]);
  atomicMax(&smax, m);
  __syncthreads();
  int r = smax;
  __syncthreads();
  return r;
}

template <int U>
__global__ void __launch_bounds__(NT) rec_fwd_f32_kernel(RecFwdArgs a) {
  constexpr int G = 4 * U;
  __shared__ float sh_h[NT][KT + 1];
  __shared__ __align__(16) float sh_R[KT][G];
  const int d = blockIdx.x / a.ctas_per_dir;
  const int cb = blockIdx.x % a.ctas_per_dir;
  const int u0 = cb * U;
  const int B = a.B, T = a.T, H = a.H, G4 = 4 * H;
  const int dir = a.dirsign[d];
  const float* __restrict__ R = a.R[d];
  const float* __restrict__ xw = a.xw[d];
  float* hb = a.hbuf[d];
  float* cb_state = a.cbuf[d];
  const bool save = a.gates[d] != nullptr;
  const int Tmax = block_max_len(a.lens, B);

  for (int s = 0; s < Tmax; ++s) {
    const float* hp = hb + (size_t)(s & 1) * B * H;
    float* hn = hb + (size_t)((s + 1) & 1) * B * H;
    for (int rb = 0; rb < B; rb += NT) {
      const int row = rb + threadIdx.x;
      float acc[G];
#pragma unroll
      for (int j = 0; j < G; ++j) acc[j] = 0.f;
      for (int k0 = 0; k0 < H; k0 += KT) {
        for (int e = threadIdx.x; e < NT * KT; e += NT) {
          int r = e / KT, k = e % KT;
          int gr = rb + r, gk = k0 + k;
          sh_h[r][k] = (gr < B && gk < H) ? hp[(size_t)gr * H + gk] : 0.f;
        }
        for (int e = threadIdx.x; e < KT * G; e += NT) {
          int k = e / G, j = e % G;
          int gk = k0 + k, gate = j / U, uu = u0 + j % U;
          sh_R[k][j] = (gk < H && uu < H) ? R[(size_t)gk * G4 + gate * H + uu] : 0.f;
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < KT; ++k) {
          const float hv = sh_h[threadIdx.x][k];
#pragma unroll
          for (int j = 0; j < G; j += 4) {
            float4 r4 = *reinterpret_cast<const float4*>(&sh_R[k][j]);
            acc[j] = fmaf(hv, r4.x, acc[j]);
            acc[j + 1] = fmaf(hv, r4.y, acc[j + 1]);
            acc[j + 2] = fmaf(hv, r4.z, acc[j + 2]);
            acc[j + 3] = fmaf(hv, r4.w, acc[j + 3]);
          }
        }
        __syncthreads();
      }
      if (row < B) {
        const int len = a.lens[row];
        if (s < len) {
          const int t = src_time(s, len, dir);
          const size_t pos = (size_t)row * T + t;
          const float* xr = xw + pos * a.xw_ld;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int uu = u0 + u;
            if (uu >= H) break;
            // Reference order: Z = x W (+) h R (+) b; here xw already holds x W + b.
            const float zi = xr[uu] + acc[u];
            const float zf = xr[H + uu] + acc[U + u];
            const float zg = xr[2 * H + uu] + acc[2 * U + u];
            const float zo = xr[3 * H + uu] + acc[3 * U + u];
            const float gi = sigmoidf_(zi), gf = sigmoidf_(zf), gg = tanhf(zg), go = sigmoidf_(zo);
            const float cp = cb_state[(size_t)row * H + uu];
            const float cn = gf * cp + gi * gg;
            const float hv = go * tanhf(cn);
            const float hprev_v = hp[(size_t)row * H + uu];
            cb_state[(size_t)row * H + uu] = cn;
            hn[(size_t)row * H + uu] = hv;
            a.y[pos * a.y_ld + (size_t)d * H + uu] = hv;
            if (save) {
              float* gr = a.gates[d] + pos * G4;
              gr[uu] = gi;
              gr[H + uu] = gf;
              gr[2 * H + uu] = gg;
              gr[3 * H + uu] = go;
              a.cprev[d][pos * H + uu] = cp;
              a.hprev[d][pos * H + uu] = hprev_v;
            }
          }
        } else {
          const size_t pos = (size_t)row * T + s;  // padded position (t == s)
          for (int u = 0; u < U; ++u) {
            const int uu = u0 + u;
            if (uu >= H) break;
            hn[(size_t)row * H + uu] = hp[(size_t)row * H + uu];  // freeze
            a.y[pos * a.y_ld + (size_t)d * H + uu] = 0.f;          // tape.cpp:797
            if (save) a.hprev[d][pos * H + uu] = 0.f;
          }
        }
      }
    }
    group_barrier(a.bar + d, (unsigned)a.ctas_per_dir * (unsigned)(s + 1));
  }
  // Positions beyond the longest sequence and final states.
  const float* hfin = hb + (size_t)(Tmax & 1) * B * H;
  for (int row = threadIdx.x; row < B; row += NT) {
    for (int u = 0; u < U; ++u) {
      const int uu = u0 + u;
      if (uu >= H) break;
      for (int s = Tmax; s < T; ++s) {
        const size_t pos = (size_t)row * T + s;
        a.y[pos * a.y_ld + (size_t)d * H + uu] = 0.f;
        if (save) a.hprev[d][pos * H + uu] = 0.f;
      }
      if (a.h_last) a.h_last[((size_t)d * B + row) * H + uu] = hfin[(size_t)row * H + uu];
      if (a.c_last) a.c_last[((size_t)d * B + row) * H + uu] = cb_state[(size_t)row * H + uu];
    }
  }
}

template <int U>
__global__ void __launch_bounds__(NT) rec_bwd_f32_kernel(RecBwdArgs a) {
  constexpr int G = 4 * U;
  __shared__ float sh_dz[NT][KT + 1];
  __shared__ float sh_R[U][KT + 1];
  __shared__ float sh_db[G];
  const int d = blockIdx.x / a.ctas_per_dir;
  const int cb = blockIdx.x % a.ctas_per_dir;
  const int u0 = cb * U;
  const int B = a.B, T = a.T, H = a.H, G4 = 4 * H;
  const int dir = a.dirsign[d];
  const float* __restrict__ R = a.R[d];
  float* zb = a.dzbuf[d];
  float* gcb = a.gcbuf[d];
  const int Tmax = block_max_len(a.lens, B);
  for (int j = threadIdx.x; j < G; j += NT) sh_db[j] = 0.f;
  float dbp[G];
#pragma unroll
  for (int j = 0; j < G; ++j) dbp[j] = 0.f;

  for (int s = Tmax - 1; s >= 0; --s) {
    const float* zn = zb + (size_t)((s + 1) & 1) * B * G4;  // DZ_{s+1} (zero at the start)
    float* zc = zb + (size_t)(s & 1) * B * G4;
    for (int rb = 0; rb < B; rb += NT) {
      const int row = rb + threadIdx.x;
      float acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = 0.f;
      // dh_rec[row, u] = sum_j DZ_{s+1}[row, j] * R[u, j]   (tape.cpp:1182-1189)
      for (int j0 = 0; j0 < G4; j0 += KT) {
        for (int e = threadIdx.x; e < NT * KT; e += NT) {
          int r = e / KT, j = e % KT;
          int gr = rb + r;
          sh_dz[r][j] = (gr < B && j0 + j < G4) ? zn[(size_t)gr * G4 + j0 + j] : 0.f;
        }
        for (int e = threadIdx.x; e < U * KT; e += NT) {
          int u = e / KT, j = e % KT;
          int uu = u0 + u;
          sh_R[u][j] = (uu < H && j0 + j < G4) ? R[(size_t)uu * G4 + j0 + j] : 0.f;
        }
        __syncthreads();
#pragma unroll 4
        for (int j = 0; j < KT; ++j) {
          const float z = sh_dz[threadIdx.x][j];
#pragma unroll
          for (int u = 0; u < U; ++u) acc[u] = fmaf(z, sh_R[u][j], acc[u]);
        }
        __syncthreads();
      }
      if (row < B) {
        const int len = a.lens[row];
        if (s < len) {
          const int t = src_time(s, len, dir);
          const size_t pos = (size_t)row * T + t;
          const float* gr = a.gates[d] + pos * G4;
          const bool last = (s == len - 1);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int uu = u0 + u;
            if (uu >= H) break;
            float gh = acc[u] + a.dy[pos * a.dy_ld + (size_t)d * H + uu];
            float gc = gcb[(size_t)row * H + uu];
            if (last && a.dh_last) gh += a.dh_last[((size_t)d * B + row) * H + uu];
            if (last && a.dc_last) gc += a.dc_last[((size_t)d * B + row) * H + uu];
            const float gi = gr[uu], gf = gr[H + uu], gg = gr[2 * H + uu], go = gr[3 * H + uu];
            const float cp = a.cprev[d][pos * H + uu];
            const float tc = tanhf(gf * cp + gi * gg);
            // tape.cpp:1161-1170
            const float d_o = gh * tc;
            const float dc = gc + gh * go * (1.f - tc * tc);
            gcb[(size_t)row * H + uu] = dc * gf;
            const float zi = dc * gg * gi * (1.f - gi);
            const float zf = dc * cp * gf * (1.f - gf);
            const float zg = dc * gi * (1.f - gg * gg);
            const float zo = d_o * go * (1.f - go);
            float* zr = zc + (size_t)row * G4;
            zr[uu] = zi;
            zr[H + uu] = zf;
            zr[2 * H + uu] = zg;
            zr[3 * H + uu] = zo;
            float* dzo = a.dz[d] + pos * G4;
            dzo[uu] = zi;
            dzo[H + uu] = zf;
            dzo[2 * H + uu] = zg;
            dzo[3 * H + uu] = zo;
            dbp[u] += zi;
            dbp[U + u] += zf;
            dbp[2 * U + u] += zg;
            dbp[3 * U + u] += zo;
          }
        } else {
          const size_t pos = (size_t)row * T + s;
          float* zr = zc + (size_t)row * G4;
          float* dzo = a.dz[d] + pos * G4;
          for (int u = 0; u < U; ++u) {
            const int uu = u0 + u;
            if (uu >= H) break;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              zr[g * H + uu] = 0.f;
              dzo[g * H + uu] = 0.f;
            }
          }
        }
      }
    }
    group_barrier(a.bar + d, (unsigned)a.ctas_per_dir * (unsigned)(Tmax - s));
  }
  for (int row = threadIdx.x; row < B; row += NT) {
    for (int s = Tmax; s < T; ++s) {
      float* dzo = a.dz[d] + ((size_t)row * T + s) * G4;
      for (int u = 0; u < U; ++u) {
        const int uu = u0 + u;
        if (uu >= H) break;
        for (int g = 0; g < 4; ++g) dzo[g * H + uu] = 0.f;
      }
    }
  }
  if (a.db[d]) {
#pragma unroll
    for (int j = 0; j < G; ++j) atomicAdd(&sh_db[j], dbp[j]);
    __syncthreads();
    for (int j = threadIdx.x; j < G; j += NT) {
      const int uu = u0 + j % U;
      if (uu >= H) continue;
      float* dst = a.db[d] + (j / U) * H + uu;
      *dst = a.accumulate ? *dst + sh_db[j] : sh_db[j];
    }
  }
}

template <typename Args, typename K>
void launch_coop(K kernel, const Args& a, int grid, cudaStream_t stream) {
  Args copy = a;
  void* params[] = {&copy};
  SL_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kernel, dim3(grid), dim3(NT), params, 0,
                                          stream));
  count_launch();
}

}  // namespace

void rec_partition(int H, int nd, int* U, int* ctas_per_dir) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int u = 4;
  while (u < 16 && (int64_t)ceil_div(H, u) * nd > sms) u *= 2;
  SL_REQUIRE((int64_t)ceil_div(H, u) * nd <= sms, SL_ERR_UNSUPPORTED,
             "persistent recurrence: hidden size " + std::to_string(H) + " x " +
                 std::to_string(nd) + " directions exceeds one resident CTA per SM");
  *U = u;
  *ctas_per_dir = (int)ceil_div(H, u);
}

void rec_fwd_f32(const RecFwdArgs& a, cudaStream_t stream) {
  const int grid = a.ctas_per_dir * a.nd;
  switch (a.U) {
    case 4: launch_coop(rec_fwd_f32_kernel<4>, a, grid, stream); break;
    case 8: launch_coop(rec_fwd_f32_kernel<8>, a, grid, stream); break;
    case 16: launch_coop(rec_fwd_f32_kernel<16>, a, grid, stream); break;
    default: throw Error{SL_ERR_UNSUPPORTED, "rec_fwd_f32: bad units per CTA"};
  }
}

void rec_bwd_f32(const RecBwdArgs& a, cudaStream_t stream) {
  const int grid = a.ctas_per_dir * a.nd;
  switch (a.U) {
    case 4: launch_coop(rec_bwd_f32_kernel<4>, a, grid, stream); break;
    case 8: launch_coop(rec_bwd_f32_kernel<8>, a, grid, stream); break;
    case 16: launch_coop(rec_bwd_f32_kernel<16>, a, grid, stream); break;
    default: throw Error{SL_ERR_UNSUPPORTED, "rec_bwd_f32: bad units per CTA"};
  }
}

}  // namespace sl
