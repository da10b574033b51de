// Embedding lookup and its scatter-add adjoint (embedding.cu).
#pragma once
#include "common.cuh"
#include "seqloom_cuda.h"

namespace sl {

size_t embedding_workspace_bytes(int64_t n, int V);
void embedding_fwd(int64_t n, const int32_t* ids, int V, int D, const float* table, float* out, int64_t ld,
                   int flags, int* bad_row, cudaStream_t st);
void embedding_fwd_bf16(int64_t n, const int32_t* ids, int V, int D, const float* table, __nv_bfloat16* out,
                        int64_t ld, int flags, int* bad_row, cudaStream_t st);
void embedding_bwd(int64_t n, const int32_t* ids, int V, int D, const float* d_out, int64_t ld, float* d_table,
                   bool accumulate, void* ws, cudaStream_t st);

}  // namespace sl
