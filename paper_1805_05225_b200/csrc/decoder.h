// The Listing-1 attention decoder over the whole target sequence (decoder.cu).
#pragma once
#include "common.cuh"

namespace sl {

struct DecDims {
  int B, Ts, T, Emb, E, H, K, Rd, Vt;
};

struct DecParams {  // fp32, reference layouts (compiler.cpp:470-500)
  const float *ctx_W, *ctx_b;     // enc_ctx   [E, K], [K]
  const float *s_W, *s_R, *s_b;   // s (lstm)  [Emb+E, 4H], [H, 4H], [4H]
  const float *fb_W, *fb_b;       // weight_feedback [1, K], [K]
  const float *str_W, *str_b;     // s_tr      [H, K], [K]
  const float *e_W, *e_b;         // e         [K, 1], [1]
  const float *ro_W, *ro_b;       // readout   [H+Emb+E, Rd], [Rd]
  const float* trg_W;             // trg       [Vt, Emb]
};

struct DecGrads {
  float *ctx_W, *ctx_b, *s_W, *s_R, *s_b, *fb_W, *fb_b, *str_W, *str_b, *e_W, *e_b, *ro_W, *ro_b, *trg_W;
};

void decoder_check(const DecDims& d);
size_t decoder_workspace_bytes(const DecDims& d);
void decoder_fwd(const DecDims& d, const DecParams& p, const __nv_bfloat16* enc, int64_t ld_enc,
                 const int32_t* src_lens, const int32_t* prev_ids, float* readout, int32_t* bad_row, void* ws,
                 cudaStream_t st);
void decoder_bwd(const DecDims& d, const DecParams& p, const DecGrads& g, const __nv_bfloat16* enc,
                 int64_t ld_enc, const int32_t* src_lens, const int32_t* prev_ids, const float* readout,
                 const float* d_readout, float* d_enc, void* ws, cudaStream_t st);

// SL_PREC_FP32 (decoder_f32.cu): fp32 encoder output [B, Ts, E] (contiguous),
// every product on the split-bf16 tcgen05 GEMM, fp32 state and attention
void decoder_f32_check(const DecDims& d);
size_t decoder_f32_workspace_bytes(const DecDims& d);
void decoder_f32_fwd(const DecDims& d, const DecParams& p, const float* enc, const int32_t* src_lens,
                     const int32_t* prev_ids, float* readout, int32_t* bad_row, void* ws, cudaStream_t st);
void decoder_f32_bwd(const DecDims& d, const DecParams& p, const DecGrads& g, const float* enc,
                     const int32_t* src_lens, const int32_t* prev_ids, const float* readout, const float* d_readout,
                     float* d_enc, void* ws, cudaStream_t st);

}  // namespace sl
