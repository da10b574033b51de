// Decoder cell step (K5): Tape::lstm_step forward/backward (tape.cpp:1074-1219)
// for the Listing-1 decoder `s` cell that the graph executor calls once per
// target step (compiler.cpp:640-650).  Z = x W + h0 R + b is two fp32-class
// tensor-core GEMMs (split-bf16 x3) into a stream-ordered scratch; the gate
// math / its adjoint are one fused elementwise kernel each (expf / tanhf, fp32).
#include <algorithm>

#include "cell.h"
#include "gemm.h"
#include "profile.h"

namespace sl {
namespace {

__global__ void cell_gates_kernel(int B, int H, const float* __restrict__ z,
                                  const float* __restrict__ c0, float* __restrict__ h,
                                  float* __restrict__ c, float* __restrict__ saved) {
  const int64_t n = (int64_t)B * H;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / H), j = (int)(e % H);
    const float* zr = z + (int64_t)r * 4 * H;
    const float gi = sigmoidf_(zr[j]), gf = sigmoidf_(zr[H + j]);
    const float gg = tanhf(zr[2 * H + j]), go = sigmoidf_(zr[3 * H + j]);
    const float cn = gf * c0[e] + gi * gg;
    const float tc = tanhf(cn);
    c[e] = cn;
    h[e] = go * tc;
    if (saved) {
      float* sv = saved + (int64_t)r * 5 * H;
      sv[j] = gi;
      sv[H + j] = gf;
      sv[2 * H + j] = gg;
      sv[3 * H + j] = go;
      sv[4 * H + j] = tc;
    }
  }
}

__global__ void cell_dz_kernel(int B, int H, const float* __restrict__ saved,
                               const float* __restrict__ c0, const float* __restrict__ gh,
                               const float* __restrict__ gc, float* __restrict__ dz,
                               float* __restrict__ dc0, int accumulate) {
  const int64_t n = (int64_t)B * H;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / H), j = (int)(e % H);
    const float* sv = saved + (int64_t)r * 5 * H;
    const float ghv = gh ? gh[e] : 0.f, gcv = gc ? gc[e] : 0.f;
    const float gi = sv[j], gf = sv[H + j], gg = sv[2 * H + j], go = sv[3 * H + j];
    const float tc = sv[4 * H + j];
    const float d_o = ghv * tc;
    const float dcn = gcv + ghv * go * (1.f - tc * tc);
    if (dc0) dc0[e] = accumulate ? dc0[e] + dcn * gf : dcn * gf;
    float* zr = dz + (int64_t)r * 4 * H;
    zr[j] = dcn * gg * gi * (1.f - gi);
    zr[H + j] = dcn * c0[e] * gf * (1.f - gf);
    zr[2 * H + j] = dcn * gi * (1.f - gg * gg);
    zr[3 * H + j] = d_o * go * (1.f - go);
  }
}

// db (+)= column sums of dz [B, N]
__global__ void colsum_kernel(int B, int N, const float* __restrict__ dz, float* __restrict__ db,
                              int accumulate) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  float s = 0.f;
  for (int r = 0; r < B; ++r) s += dz[(int64_t)r * N + j];
  db[j] = accumulate ? db[j] + s : s;
}

int grid_for(int64_t n) { return (int)std::min<int64_t>(ceil_div(n, 256), 148 * 8); }

// stream-ordered scratch of one call: [z or dz : B x 4H fp32 | split-bf16 GEMM operands]
size_t cell_ws(int B, int D, int H) {
  const size_t g = std::max({gemm_f32x3_workspace_bytes(false, false, B, 4 * H, D, false),
                             gemm_f32x3_workspace_bytes(false, false, B, 4 * H, H, false),
                             gemm_f32x3_workspace_bytes(false, true, B, D, 4 * H, false),
                             gemm_f32x3_workspace_bytes(false, true, B, H, 4 * H, false),
                             gemm_f32x3_workspace_bytes(true, false, D, 4 * H, B, true),
                             gemm_f32x3_workspace_bytes(true, false, H, 4 * H, B, false)});
  return (size_t)round_up((int64_t)B * 4 * H * 4, 256) + g;
}

}  // namespace

// Both GEMMs of the step on the tensor cores at fp32 class (gemm_f32x3.cu: split-bf16,
// fp32 accumulation): Z = x W + b, Z += h0 R (tape.cpp:1103-1109).
void cell_fwd(int B, int D, int H, const float* x, const float* h0, const float* c0,
              const float* W, const float* R, const float* b, float* h, float* c, float* saved,
              cudaStream_t stream) {
  char* ws = nullptr;
  SL_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ws), cell_ws(B, D, H), stream));
  float* z = reinterpret_cast<float*>(ws);
  void* g = ws + round_up((int64_t)B * 4 * H * 4, 256);
  gemm_f32x3(false, false, B, 4 * H, D, x, D, W, 4 * H, 0.f, z, 4 * H, b, nullptr, 0, g, stream);
  gemm_f32x3(false, false, B, 4 * H, H, h0, H, R, 4 * H, 1.f, z, 4 * H, nullptr, nullptr, 0, g, stream);
  cell_gates_kernel<<<grid_for((int64_t)B * H), 256, 0, stream>>>(B, H, z, c0, h, c, saved);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
  SL_CUDA_TRY(cudaFreeAsync(ws, stream));
}

void cell_bwd(int B, int D, int H, const float* x, const float* h0, const float* c0,
              const float* W, const float* R, const float* saved, const float* gh,
              const float* gc, float* dx, float* dh0, float* dc0, float* dW, float* dR,
              float* db, int accumulate, cudaStream_t stream) {
  char* ws = nullptr;
  const float beta = accumulate ? 1.f : 0.f;
  SL_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ws), cell_ws(B, D, H), stream));
  float* dz = reinterpret_cast<float*>(ws);
  void* g = ws + round_up((int64_t)B * 4 * H * 4, 256);
  cell_dz_kernel<<<grid_for((int64_t)B * H), 256, 0, stream>>>(B, H, saved, c0, gh, gc, dz, dc0,
                                                               accumulate);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
  if (dx) gemm_f32x3(false, true, B, D, 4 * H, dz, 4 * H, W, 4 * H, beta, dx, D, nullptr, nullptr, 0, g, stream);
  if (dh0) gemm_f32x3(false, true, B, H, 4 * H, dz, 4 * H, R, 4 * H, beta, dh0, H, nullptr, nullptr, 0, g, stream);
  if (dW) {  // [dW; db] = [x | 1]^T dz in one GEMM
    gemm_f32x3(true, false, D, 4 * H, B, x, D, dz, 4 * H, beta, dW, 4 * H, nullptr, db, 4 * H, g, stream);
  } else if (db) {
    colsum_kernel<<<(unsigned)ceil_div(4 * H, 256), 256, 0, stream>>>(B, 4 * H, dz, db, accumulate);
    SL_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
  if (dR) gemm_f32x3(true, false, H, 4 * H, B, h0, H, dz, 4 * H, beta, dR, 4 * H, nullptr, nullptr, 0, g, stream);
  SL_CUDA_TRY(cudaFreeAsync(ws, stream));
}

}  // namespace sl
