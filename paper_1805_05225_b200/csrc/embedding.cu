// Embedding lookup: the reference's Linear layer applied to ids
// — gather_rows(table = {layer}/W, ids) (compiler.cpp:584-589, tape.cpp:448-492)
// — and its adjoint, a scatter-add of the output gradient rows into the table
// gradient.
//
// Forward: one warp per id row copies D floats (16 B vectors when aligned) to
// a row of stride ld (so the rows can land inside a wider buffer, e.g. the
// decoder's [target embedding ‖ context] input); a bf16 variant writes the
// rows straight into the padded layer-0 LSTM input (with the ones column at D
// that the fused bias gradient uses, SL_LAYER_X_BF16), so the first layer's
// conversion pass disappears.
//
// Backward, deterministic and in the reference's summation order: the
// reference builds a zero table gradient and adds the output-gradient rows in
// row order r = 0, 1, ... (tape.cpp:478-486), then accumulates that into the
// parameter's gradient.  Here the (id, r) pairs are radix-sorted by id (the
// sort is stable, so r stays ascending inside each id), and one warp per
// distinct id sums its rows in that order, lanes over the D columns, and
// writes old + sum (accumulate) or sum.  Rows of the table that no id touches
// are zeroed up front unless accumulating.
#include <cub/device/device_radix_sort.cuh>

#include "embedding.h"
#include "profile.h"

namespace sl {
namespace {

// ids < 0 with SL_EMB_NEGATIVE_ZERO: a zero row, no error (the decoder's
// "previous target" at t = 0, the reference's initial_output = 0, models.cpp:96).
// Any other id outside [0, V) is the reference's IndexError: the row is filled
// with NaN so the step's loss and gradients are non-finite and a fused optimizer
// step skips the update (the reference raises before touching any parameter).
enum IdClass { kIdOk = 0, kIdZero = 1, kIdBad = 2 };
__device__ __forceinline__ int id_class(int id, int V, int flags, int64_t r, int lane, int* bad_row) {
  if (id >= 0 && id < V) return kIdOk;
  if (id < 0 && (flags & SL_EMB_NEGATIVE_ZERO)) return kIdZero;
  if (lane == 0) atomicMin(bad_row, (int)min(r, (int64_t)INT32_MAX));  // IndexError (tape.cpp:464-467)
  return kIdBad;
}

__global__ void gather_kernel(int64_t n, const int32_t* __restrict__ ids, int V, int D,
                              const float* __restrict__ table, float* __restrict__ out, int64_t ld, int flags,
                              int* bad_row) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= n) return;
  const int id = ids[r];
  float* dst = out + r * ld;
  const int cls = id_class(id, V, flags, r, lane, bad_row);
  if (cls != kIdOk) {
    const float fill = cls == kIdBad ? __int_as_float(0x7fc00000) : 0.f;
    for (int j = lane; j < D; j += 32) dst[j] = fill;
    return;
  }
  const float* src = table + (int64_t)id * D;
  if ((D % 4) == 0 && (ld % 4) == 0 &&
      ((reinterpret_cast<uintptr_t>(table) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    for (int j = lane * 4; j < D; j += 128)
      *reinterpret_cast<float4*>(dst + j) = __ldg(reinterpret_cast<const float4*>(src + j));
  } else {
    for (int j = lane; j < D; j += 32) dst[j] = __ldg(src + j);
  }
}

// bf16 rows: [0, D) the embedding; with SL_EMB_ONES_COLUMN also D = 1.0 and (D, ld) = 0
// (the padded layer-0 LSTM input, SL_LAYER_X_BF16)
__global__ void gather_bf16_kernel(int64_t n, const int32_t* __restrict__ ids, int V, int D,
                                   const float* __restrict__ table, __nv_bfloat16* __restrict__ out, int64_t ld,
                                   int flags, int* bad_row) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= n) return;
  const int id = ids[r];
  const int cls = id_class(id, V, flags, r, lane, bad_row);
  const bool ok = cls == kIdOk;
  const float fill = cls == kIdBad ? __int_as_float(0x7fc00000) : 0.f;  // NaN poisons a bad id's row
  const float* src = table + (int64_t)(ok ? id : 0) * D;
  __nv_bfloat16* dst = out + r * ld;
  const bool ones = flags & SL_EMB_ONES_COLUMN;
  const int64_t end = ones ? ld : D;
  if ((ld % 2) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0) {
    for (int64_t j = 2 * lane; j < end; j += 64) {
      float a = j < D ? fill : 0.f, b = j + 1 < D ? fill : 0.f;
      if (ok && j < D) a = __ldg(src + j);
      if (ok && j + 1 < D) b = __ldg(src + j + 1);
      if (ones && j == D) a = 1.f;
      if (ones && j + 1 == D) b = 1.f;
      if (j + 1 < end) *reinterpret_cast<__nv_bfloat162*>(dst + j) = __floats2bfloat162_rn(a, b);
      else dst[j] = __float2bfloat16_rn(a);
    }
  } else {
    for (int64_t j = lane; j < end; j += 32)
      dst[j] = __float2bfloat16_rn(ok && j < D ? __ldg(src + j) : j < D ? fill : (ones && j == D ? 1.f : 0.f));
  }
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

__global__ void iota_kernel(int64_t n, int32_t* v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// one warp per distinct id of the sorted keys: d_table[id] (+)= sum of its rows, ascending r
__global__ void scatter_sorted_kernel(int64_t n, const int32_t* __restrict__ keys, const int32_t* __restrict__ rows,
                                      int V, int D, const float* __restrict__ d_out, int64_t ld,
                                      float* __restrict__ d_table, int accumulate) {
  const int64_t i = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (i >= n) return;
  const int id = keys[i];
  if ((i > 0 && keys[i - 1] == id) || id < 0 || id >= V) return;  // not the start of a segment
  int64_t e = i + 1;
  while (e < n && keys[e] == id) ++e;
  float* dst = d_table + (int64_t)id * D;
  for (int j = lane; j < D; j += 32) {
    float s = 0.f;  // the reference's zero-initialised per-call table gradient
    for (int64_t k = i; k < e; ++k) s += d_out[(int64_t)rows[k] * ld + j];
    dst[j] = accumulate ? dst[j] + s : s;
  }
}

struct EmbWs {
  int32_t *keys_in, *keys_out, *rows_in, *rows_out;
  void* tmp;
  size_t tmp_bytes;
};

size_t sort_tmp_bytes(int64_t n, int /*V*/) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return bytes;
}

EmbWs carve(int64_t n, int V, void* ws) {
  EmbWs w;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += round_up((int64_t)bytes, 256);
    return q;
  };
  w.keys_out = reinterpret_cast<int32_t*>(take(n * 4));
  w.rows_in = reinterpret_cast<int32_t*>(take(n * 4));
  w.rows_out = reinterpret_cast<int32_t*>(take(n * 4));
  w.tmp_bytes = sort_tmp_bytes(n, V);
  w.tmp = take(w.tmp_bytes);
  w.keys_in = nullptr;
  return w;
}

}  // namespace

size_t embedding_workspace_bytes(int64_t n, int V) {
  return 3 * (size_t)round_up(n * 4, 256) + (size_t)round_up((int64_t)sort_tmp_bytes(n, V), 256) + 256;
}

void embedding_fwd(int64_t n, const int32_t* ids, int V, int D, const float* table, float* out, int64_t ld,
                   int flags, int* bad_row, cudaStream_t st) {
  set_int_kernel<<<1, 1, 0, st>>>(bad_row, INT32_MAX);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
  if (n <= 0) return;
  Phase ph(st, "k9_embedding_fwd", 0.0, 8.0 * n * D);
  gather_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, ids, V, D, table, out, ld, flags, bad_row);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void embedding_fwd_bf16(int64_t n, const int32_t* ids, int V, int D, const float* table, __nv_bfloat16* out,
                        int64_t ld, int flags, int* bad_row, cudaStream_t st) {
  set_int_kernel<<<1, 1, 0, st>>>(bad_row, INT32_MAX);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
  if (n <= 0) return;
  Phase ph(st, "k9_embedding_fwd", 0.0, 6.0 * n * D);
  gather_bf16_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, ids, V, D, table, out, ld, flags, bad_row);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch();
}

void embedding_bwd(int64_t n, const int32_t* ids, int V, int D, const float* d_out, int64_t ld, float* d_table,
                   bool accumulate, void* ws, cudaStream_t st) {
  Phase ph(st, "k9_embedding_bwd", 0.0, 8.0 * n * D + (accumulate ? 0.0 : 4.0 * V * D));
  if (!accumulate) SL_CUDA_TRY(cudaMemsetAsync(d_table, 0, sizeof(float) * (size_t)V * D, st));
  if (n <= 0) return;
  EmbWs w = carve(n, V, ws);
  iota_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1184), 256, 0, st>>>(n, w.rows_in);
  SL_CUDA_TRY(cudaGetLastError());
  size_t tb = w.tmp_bytes;
  // all 32 key bits: ids outside [0, V) form their own segments, which the
  // scatter skips (negative ids are the zero rows of SL_EMB_NEGATIVE_ZERO;
  // out-of-range ones were reported by the forward, as the reference throws
  // before recording a backward)
  SL_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.tmp, tb, ids, w.keys_out, w.rows_in, w.rows_out, (int)n, 0,
                                              32, st));
  scatter_sorted_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, st>>>(n, w.keys_out, w.rows_out, V, D, d_out, ld,
                                                                  d_table, accumulate ? 1 : 0);
  SL_CUDA_TRY(cudaGetLastError());
  count_launch(3);
}

}  // namespace sl
