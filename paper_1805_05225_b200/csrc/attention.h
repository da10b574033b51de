// The decoder's MLP attention step (attention.cu).
#pragma once
#include "common.cuh"
#include "gemm.h"

namespace sl {

struct AttnArgs {
  int B, Ts, K, E, H;
  const int32_t* lens;     // source lengths [B]
  const float* enc_ctx;    // [B, Ts, K]
  const float* enc;        // [B, Ts, E]
  const float* accum;      // [B, Ts]
  const float* W_fb;       // [1, K]
  const float* b_fb;       // [K]
  const float* v;          // [K, 1]
  const float* b_v;        // [1] (device)
  float* s_tr;             // workspace [B, K]
  // forward outputs
  float* att;              // [B, E]
  float* a;                // [B, Ts]
  float* accum_out;        // [B, Ts]
  // backward
  const float* a_saved;    // [B, Ts] from the forward
  const float* d_att;      // [B, E]
  const float* d_accum_out;  // [B, Ts] or null
  float* d_s_tr;           // workspace [B, K]
  float* d_enc_ctx;        // [B, Ts, K]
  float* d_enc;            // [B, Ts, E]
  float* d_accum;          // [B, Ts]
  int d_accum_fresh;       // d_accum written, not accumulated, even when `accumulate` is set
  float* d_W_fb;           // [K]
  float* d_b_fb;           // [K]
  float* d_v;              // [K]
  float* d_b_v;            // [1]
  int accumulate;
  // optional (the decoder's loop): W_s split once per call into its hi/lo image
  // (gemm.h x3_split_img), read by both s_tr = s W_s (W_s3_fwd) and d s = d s_tr W_s^T
  // (W_s3_bwd: the same image); s_tr written to / read from a caller buffer [B, K]
  // instead of recomputed in the backward
  const __nv_bfloat16* W_s3_fwd;
  const __nv_bfloat16* W_s3_bwd;
  float* s_tr_out;
  const float* s_tr_in;
  // optional (the decoder's loop): defer every accumulation over the steps — the
  // backward then writes only d s (via d s_tr, to d_s_tr_out when set), d accum and
  // the softmax adjoint de [B, Ts] (to de_out); d enc, d enc_ctx, d W_fb, d b_fb,
  // d v and d b_v are left to the caller (decoder_f32.cu sums them after the loop)
  int defer;
  float* d_s_tr_out;
  float* de_out;
  // optional (the decoder's loop): further row-strided destinations of att [B, E]
  // (the readout input and the next step's [att | s] row), written by the context kernel
  float* att_copy[2];
  int64_t att_copy_ld[2];
  // optional (the decoder's loop, with W_s3_bwd): the backward's d s = d s_tr W_s^T handed
  // to the caller as split-K partials through ds_parts_out instead of accumulated into d_s
  X3Parts* ds_parts_out;
  // optional (the decoder's loop): att also written as split image rows (hi at att_img,
  // row stride att_img_ld, lo att_img_lo further on)
  __nv_bfloat16* att_img;
  int64_t att_img_ld, att_img_lo;
  // optional (the decoder's loop): s as its split image rows (the s_tr projection's A
  // operand: no per-step split)
  const __nv_bfloat16* s_img;
  int64_t s_img_ld, s_img_lo;
  // (internal) deferred backward: the tanh pass's per-chunk d s_tr partials
  float* ds_part;
};

size_t attention_workspace_bytes(int B, int K, int H, int Ts);
void attention_fwd(AttnArgs p, const float* s, const float* W_s, const float* b_s, void* ws, cudaStream_t st);
void attention_bwd(AttnArgs p, const float* s, const float* W_s, const float* b_s, float* d_s, float* d_W_s,
                   float* d_b_s, void* ws, cudaStream_t st);

}  // namespace sl
