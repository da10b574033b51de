/* seqloom_cuda.h — C ABI of the B200-native fused LSTM layer.
 *
 * This is the drop-in boundary for the reference's LSTM hot path:
 *   seqloom::lstm_sequence(Tape&, W, R, b, xs, direction)   reference layers.hpp:17 / layers.cpp:8-37
 *   Tape::lstm_step(W, R, b, x, h_prev, c_prev)              reference tape.hpp:123-129 / tape.cpp:1074-1222
 * plus the fused bidirectional variant eval_layer builds for the Listing-1
 * encoder (reference compiler.cpp:600-608: two lstm_sequence calls whose
 * outputs feed concat_feature, tape.cpp:709-783).
 *
 * Conventions (all match the reference's layouts so no caller-side reshuffle
 * is needed, reference tensor.hpp:21 canonical order, row-major):
 *   x   [B, T, D]          fp32 (bf16 padded with SL_LAYER_X_BF16), batch-major, padded
 *                          positions t >= len[b] ignored
 *   y   [B, T, ndir*H]     fp32 (bf16 padded with SL_LAYER_Y_BF16); direction d writes
 *                          columns [d*H, (d+1)*H) — the
 *                          concat_feature([fw, bw]) layout; padded positions are 0
 *   W   [D, 4H]  R [H, 4H]  b [4H]   fp32, gate blocks (i | f | g | o)
 *   seq_lens [B]           int32 in (0, T] (reference tensor.cpp:121-138)
 *   h_last/c_last [ndir, B, H]  state after step len[b]-1 in processing order
 * All data pointers are DEVICE pointers owned by the caller; pointer arrays
 * (W[d], ...) are host arrays of device pointers, one per direction.
 * Every call is asynchronous on `stream`.  No exception crosses the ABI: each
 * entry point returns SL_OK or an error code, with a message retrievable by
 * sl_last_error() (thread-local).  Gradient outputs follow the tape's
 * GradBuffer::accumulate contract (reference tape.cpp:76-89) when
 * `accumulate` != 0 (+=), else they are overwritten.
 */
#ifndef SEQLOOM_CUDA_H_
#define SEQLOOM_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sl_stream_t; /* == cudaStream_t */

enum sl_status {
  SL_OK = 0,
  SL_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument (layers.cpp:14-16) */
  SL_ERR_SHAPE = 2,            /* reference: seqloom::ShapeError (tape.cpp:1092-1094) */
  SL_ERR_CUDA = 3,             /* CUDA runtime / launch failure */
  SL_ERR_WORKSPACE = 4,        /* reserve / workspace too small */
  SL_ERR_UNSUPPORTED = 5       /* e.g. not running on an sm_100 device */
};

enum sl_precision {
  SL_PREC_FP32 = 0, /* fp32 semantics: rel. parity 1e-4 vs the fp32 reference */
  SL_PREC_BF16 = 1  /* bf16 tensor-core operands, fp32 accumulate / cell state; rel. 2e-2 */
};

/* sl_lstm_layer.flags (SL_PREC_BF16 only): bf16 activations between stacked
 * layers, so a layer's output feeds the next layer's input GEMM with no fp32
 * round trip and no conversion pass.  The bf16 tensors are row-padded to
 * sl_lstm_bf16_pitch(features) columns with 1.0 in column `features` (the
 * layer's own bias/db column) and FINITE (e.g. zero-initialised) padding. */
enum sl_layer_flags {
  SL_LAYER_X_BF16 = 1, /* x is bf16 [B, T, sl_lstm_bf16_pitch(D)], 1.0 at column D; kept
                          unchanged by the caller until the matching bwd */
  SL_LAYER_Y_BF16 = 2, /* y is written as bf16 [B, T, sl_lstm_bf16_pitch(ndir*H)] with 1.0 at
                          column ndir*H: directly the next layer's SL_LAYER_X_BF16 input */
  /* SL_PREC_FP32 only: the activations between stacked layers as their split-bf16
   * ("x3") image — two planes [2][B*T][sl_lstm_bf16_pitch(features)] of bf16, hi =
   * bf16(v) then lo = bf16(v - hi), 1.0 at column `features` of the hi plane, zero
   * padding — the operand the fp32-class input GEMM reads, so no split pass runs */
  SL_LAYER_X_X3 = 16, /* x is that image of [B, T, D]; kept unchanged until the matching bwd */
  SL_LAYER_Y_X3 = 32  /* y is written as that image of [B, T, ndir*H] (zero-initialised by the
                         caller): directly the next layer's SL_LAYER_X_X3 input */
};
/* Row pitch (elements) of the padded bf16 activation layout: round_up(features + 1, 64). */
int64_t sl_lstm_bf16_pitch(int32_t features);

/* One LSTM layer, one or two directions over the same input. */
typedef struct sl_lstm_layer {
  int32_t batch;     /* B  */
  int32_t time;      /* T  (max length; seq_lens[b] <= T) */
  int32_t input_dim; /* D  */
  int32_t hidden;    /* H  */
  int32_t num_dirs;  /* 1, or 2 = bidirectional: dir 0 forward, dir 1 backward, run concurrently */
  int32_t direction; /* num_dirs == 1: +1 or -1 (reference layers.cpp:14) */
  int32_t precision; /* enum sl_precision */
  int32_t flags;     /* enum sl_layer_flags (0 = fp32 x / y) */
} sl_lstm_layer;

/* Library version (major*10000 + minor*100 + patch). */
int sl_version(void);
/* Last error message of the calling thread ("" when none). */
const char* sl_last_error(void);

/* Which kernels a descriptor runs on (0 = invalid descriptor, see sl_last_error):
 *   SL_PATH_BF16_TC     SL_PREC_BF16: bf16 tcgen05 GEMMs and persistent recurrences
 *   SL_PATH_FP32_X3_TC  SL_PREC_FP32 on the tensor cores: split-bf16 ("x3") tcgen05
 *                       GEMMs and recurrences, A B = A_hi B_hi + A_lo B_hi + A_hi B_lo
 *                       with fp32 accumulation (relative error ~1e-5), fp32 state
 *   SL_PATH_FP32_SIMT   SL_PREC_FP32 for hidden sizes the x3 recurrences do not
 *                       cover: fp32 CUDA-core GEMMs and recurrences */
enum sl_path { SL_PATH_BF16_TC = 1, SL_PATH_FP32_X3_TC = 2, SL_PATH_FP32_SIMT = 3 };
int sl_lstm_layer_path(const sl_lstm_layer* layer);

/* Validate a descriptor: SL_OK, or the error (and message) fwd/bwd would raise. */
int sl_lstm_layer_check(const sl_lstm_layer* layer);

/* Bytes of the caller-owned buffer that carries saved activations from
 * sl_lstm_layer_fwd to sl_lstm_layer_bwd (cuDNN "reserve space" semantics;
 * pass NULL / 0 to fwd for inference: nothing is saved). */
size_t sl_lstm_reserve_size(const sl_lstm_layer* layer);
/* Bytes of per-call scratch needed by fwd and by bwd. */
size_t sl_lstm_workspace_size(const sl_lstm_layer* layer);

/* Forward of lstm_sequence over all directions (layers.cpp:8-37).
 * h_last / c_last may be NULL. */
int sl_lstm_layer_fwd(const sl_lstm_layer* layer, const float* x, const int32_t* seq_lens,
                      const float* const* W, const float* const* R, const float* const* b,
                      float* y, float* h_last, float* c_last, void* reserve,
                      size_t reserve_bytes, void* workspace, size_t workspace_bytes,
                      sl_stream_t stream);

/* Backward (BPTT) of lstm_sequence: the adjoint of every tape record the
 * reference's forward emits (tape.cpp:1142-1219 per step, plus the
 * slice/stack/mask/reverse adjoints).  dy is [B, T, ndir*H]; dh_last and
 * dc_last ([ndir, B, H]) may be NULL.  dx, dW[d], dR[d], db[d] may be NULL
 * (not needed).  `reserve` must come from the matching fwd call. */
int sl_lstm_layer_bwd(const sl_lstm_layer* layer, const float* x, const int32_t* seq_lens,
                      const float* const* W, const float* const* R, const float* dy,
                      const float* dh_last, const float* dc_last, float* dx, float* const* dW,
                      float* const* dR, float* const* db, int accumulate, const void* reserve,
                      size_t reserve_bytes, void* workspace, size_t workspace_bytes,
                      sl_stream_t stream);

/* Single step, Tape::lstm_step (tape.cpp:1074-1141): x [B, D], h0/c0 [B, H]
 * -> h, c [B, H].  `saved` [B, 5H] fp32 (i, f, g, o, tanh c) may be NULL
 * when no backward follows. */
int sl_lstm_cell_fwd(int32_t batch, int32_t input_dim, int32_t hidden, int32_t precision,
                     const float* x, const float* h0, const float* c0, const float* W,
                     const float* R, const float* b, float* h, float* c, float* saved,
                     sl_stream_t stream);

/* Backward closure of lstm_step (tape.cpp:1142-1219).  gh / gc may be NULL
 * (zero); any output may be NULL. */
int sl_lstm_cell_bwd(int32_t batch, int32_t input_dim, int32_t hidden, int32_t precision,
                     const float* x, const float* h0, const float* c0, const float* W,
                     const float* R, const float* saved, const float* gh, const float* gc,
                     float* dx, float* dh0, float* dc0, float* dW, float* dR, float* db,
                     int accumulate, sl_stream_t stream);

/* ---- optimizer (the training step around the hot path) --------
 * One fused step over a flat fp32 parameter buffer of n elements:
 *   g' = grad_scale * g;  clip: g' *= min(1, clip_norm / ||g'||_2)  (clip_norm <= 0: off)
 *   m = b1 m + (1-b1) g';  v = b2 v + (1-b2) g'^2;
 *   p -= lr * (m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps)
 * (reference SPEC.md:429-437 adam_step, global-norm clip 5.0 before Adam
 * SPEC.md:484).  step >= 1 is the step number; step == 0 uses the counter kept
 * in `scratch` (+1 per successful step) so a captured CUDA graph replays real
 * Adam steps.  `scratch` must be zero-filled once before its first use.  A
 * non-finite gradient leaves p, m, v
 * untouched and sets *nonfinite_out (device int32, may be NULL); *grad_norm_out
 * (device float, may be NULL) receives ||grad_scale * g||_2 before clipping.
 * `scratch` is a device buffer of sl_adam_scratch_size() bytes.  All buffers
 * 16 B aligned, device-resident, asynchronous on `stream`. */
size_t sl_adam_scratch_size(void);
int sl_adam_step(int64_t n, float* params, const float* grads, float* m, float* v, int32_t step,
                 float lr, float beta1, float beta2, float eps, float grad_scale, float clip_norm,
                 void* scratch, float* grad_norm_out, int32_t* nonfinite_out, sl_stream_t stream);

/* ---- decoder MLP attention step --------------------------------
 * One step of the Listing-1 decoder's attention subnet (reference
 * models.cpp:107-154, compiler.cpp:616-639), fp32:
 *   s_tr = s W_s + b_s;  e = tanh(enc_ctx + accum W_fb + b_fb + s_tr) v + b_v;
 *   a = softmax over the valid source positions (tape.cpp:926-985);
 *   accum_out = accum + a;  att = sum_j a_j enc_j (tape.cpp:987-1072).
 * Shapes: enc_ctx [B, Ts, K], enc [B, Ts, E], s [B, H], accum / a / accum_out
 * [B, Ts], W_s [H, K], b_s [K], W_fb [1, K], b_fb [K], v [K, 1], b_v [1] (a
 * device scalar), att [B, E]; src_lens [B].  The backward takes the forward's
 * `a`, the upstream d_att and d_accum_out (may be NULL), and writes (or, with
 * accumulate, adds) every input gradient; any gradient output may be NULL
 * except d_enc_ctx, d_enc, d_accum, d_W_fb, d_b_fb, d_v, d_b_v. */
typedef struct sl_attention {
  int32_t batch;     /* B  */
  int32_t src_time;  /* Ts */
  int32_t key_dim;   /* K  */
  int32_t enc_dim;   /* E  */
  int32_t state_dim; /* H  */
} sl_attention;
size_t sl_attention_workspace_size(const sl_attention* att);
int sl_attention_step_fwd(const sl_attention* att, const int32_t* src_lens, const float* enc_ctx,
                          const float* enc, const float* s, const float* accum, const float* W_s,
                          const float* b_s, const float* W_fb, const float* b_fb, const float* v,
                          const float* b_v, float* att_out, float* a, float* accum_out, void* workspace,
                          size_t workspace_bytes, sl_stream_t stream);
int sl_attention_step_bwd(const sl_attention* att, const int32_t* src_lens, const float* enc_ctx,
                          const float* enc, const float* s, const float* accum, const float* W_s,
                          const float* b_s, const float* W_fb, const float* b_fb, const float* v,
                          const float* a, const float* d_att, const float* d_accum_out, float* d_enc_ctx,
                          float* d_enc, float* d_s, float* d_accum, float* d_W_s, float* d_b_s, float* d_W_fb,
                          float* d_b_fb, float* d_v, float* d_b_v, int accumulate, void* workspace,
                          size_t workspace_bytes, sl_stream_t stream);

/* ---- the Listing-1 attention decoder over a target sequence ----
 * The reference's `output` subnetwork as its training loop evaluates it with
 * teacher forcing (models.cpp:83-166; compiler.cpp:770-905 runs it step by
 * step), plus the base layer enc_ctx (models.cpp:60), per target step t:
 *   s_t, c_t = lstm_step([trg_{t-1} ‖ att_{t-1}], s_{t-1}, c_{t-1})  (RnnCell `s`)
 *   e = tanh(enc_ctx + accum_{t-1} W_fb + b_fb + s_t W_s + b_s) v + b_v
 *   a_t = softmax over the valid source positions, accum_t = accum_{t-1} + a_t
 *   att_t = sum_j a_t[j] enc_j
 *   readout_t = relu([s_t ‖ trg_{t-1} ‖ att_t] W_ro + b_ro)
 * with trg_{t-1} = trg_W[prev_ids[b, t]] (prev_ids < 0: the zero initial
 * output), att_{-1} = s_{-1} = c_{-1} = accum_{-1} = 0.  The output_prob layer
 * and its loss are sl_output_ce on `readout`.
 * enc is the encoder output in the padded bf16 layout sl_lstm_layer writes with
 * SL_LAYER_Y_BF16 ([B, Ts, enc_ld], enc_ld >= sl_lstm_bf16_pitch(enc_dim), 1.0
 * at column enc_dim); prev_ids [B, T] int32; readout [B, T, readout_dim] fp32.
 * Parameters / gradients are fp32 in the reference layouts (compiler.cpp:
 * 470-500); the backward overwrites every gradient and d_enc [B, Ts, enc_dim].
 * bf16 tensor-core operands, fp32 accumulation and cell state (SL_PREC_BF16
 * tolerance).  The workspace carries the forward's saved activations to the
 * backward (same parameters, inputs and workspace).  Limits: batch <= 256 per
 * call; hidden, enc_dim, key_dim, readout_dim multiples of 8; key_dim <= 1024;
 * an out-of-range prev id sets *bad_row (the reference's IndexError).  Every
 * parameter / gradient pointer must be 16 B aligned. */
typedef struct sl_attn_decoder {
  int32_t batch, src_time, trg_time, embed_dim, enc_dim, hidden, key_dim, readout_dim, trg_vocab;
} sl_attn_decoder;
typedef struct sl_attn_decoder_params {
  const float *enc_ctx_W, *enc_ctx_b;    /* [E, K], [K]            */
  const float *s_W, *s_R, *s_b;          /* [Emb+E, 4H], [H, 4H], [4H] */
  const float *fb_W, *fb_b;              /* weight_feedback [1, K], [K] */
  const float *s_tr_W, *s_tr_b;          /* [H, K], [K]            */
  const float *e_W, *e_b;                /* [K, 1], [1]            */
  const float *readout_W, *readout_b;    /* [H+Emb+E, Rd], [Rd]    */
  const float *trg_W;                    /* [trg_vocab, Emb]       */
} sl_attn_decoder_params;
typedef struct sl_attn_decoder_grads {
  float *enc_ctx_W, *enc_ctx_b, *s_W, *s_R, *s_b, *fb_W, *fb_b, *s_tr_W, *s_tr_b, *e_W, *e_b, *readout_W,
      *readout_b, *trg_W;
} sl_attn_decoder_grads;
size_t sl_attn_decoder_workspace_size(const sl_attn_decoder* dec);
int sl_attn_decoder_fwd(const sl_attn_decoder* dec, const sl_attn_decoder_params* params, const void* enc_bf16,
                        int64_t enc_ld, const int32_t* src_lens, const int32_t* prev_ids, float* readout,
                        int32_t* bad_row, void* workspace, size_t workspace_bytes, sl_stream_t stream);
int sl_attn_decoder_bwd(const sl_attn_decoder* dec, const sl_attn_decoder_params* params,
                        const sl_attn_decoder_grads* grads, const void* enc_bf16, int64_t enc_ld,
                        const int32_t* src_lens, const int32_t* prev_ids, const float* readout,
                        const float* d_readout, float* d_enc, void* workspace, size_t workspace_bytes,
                        sl_stream_t stream);

/* The same decoder at the reference's precision (SL_PREC_FP32 semantics, rel.
 * 1e-4): enc is the fp32 encoder output [B, Ts, enc_dim] (contiguous), every
 * product runs on the split-bf16 tcgen05 GEMM (A B = A_hi B_hi + A_lo B_hi +
 * A_hi B_lo, fp32 accumulation), the cell state, attention and activations
 * are fp32.  Same descriptor, parameters and gradients as above; no batch or
 * width limits beyond src_time <= 4096.  The workspace carries the forward's
 * saved activations to the backward. */
size_t sl_attn_decoder_f32_workspace_size(const sl_attn_decoder* dec);
int sl_attn_decoder_fwd_f32(const sl_attn_decoder* dec, const sl_attn_decoder_params* params, const float* enc,
                            const int32_t* src_lens, const int32_t* prev_ids, float* readout, int32_t* bad_row,
                            void* workspace, size_t workspace_bytes, sl_stream_t stream);
int sl_attn_decoder_bwd_f32(const sl_attn_decoder* dec, const sl_attn_decoder_params* params,
                            const sl_attn_decoder_grads* grads, const float* enc, const int32_t* src_lens,
                            const int32_t* prev_ids, const float* readout, const float* d_readout, float* d_enc,
                            void* workspace, size_t workspace_bytes, sl_stream_t stream);

/* ---- output layer + loss ---------------------------------------
 * The decoder's Softmax layer and its training loss in one call: logits =
 * x W + b (reference compiler.cpp:651-663), log_softmax (tape.cpp:879-924),
 * ce_label_smoothing with `epsilon` averaged over the valid (t < seq_lens[b])
 * positions (tape.cpp:1224-1298), and the gradients of that mean loss:
 *   x [B, T, D] fp32, targets [B, T] int32 in [0, V), W [D, V], b [V];
 *   *loss (device float); dx [B, T, D], dW [D, V], db [V] may be NULL;
 *   *bad_target (device int32) is set when a valid position's id is out of
 *   range (the reference raises IndexError naming the layer); the loss and
 *   that row's dZ are then NaN, so every gradient is non-finite and
 *   sl_adam_step leaves the parameters untouched.
 * bf16 tensor-core GEMMs with fp32 accumulation; the fp32 logits are never
 * written to HBM (bf16 logits + fused online-softmax statistics). */
size_t sl_output_ce_workspace_size(int32_t batch, int32_t time, int32_t input_dim, int32_t vocab);
int sl_output_ce(int32_t batch, int32_t time, int32_t input_dim, int32_t vocab, const float* x,
                 const int32_t* targets, const int32_t* seq_lens, const float* W, const float* b,
                 float epsilon, float* loss, float* dx, float* dW, float* db, int accumulate,
                 void* workspace, size_t workspace_bytes, int32_t* bad_target, sl_stream_t stream);

/* The same at the reference's precision (SL_PREC_FP32 semantics, rel. 1e-4):
 * fp32 logits in the workspace, every GEMM on the split-bf16 tcgen05 path (x3),
 * expf / logf softmax statistics.  db requires dW. */
size_t sl_output_ce_f32_workspace_size(int32_t batch, int32_t time, int32_t input_dim, int32_t vocab);
int sl_output_ce_f32(int32_t batch, int32_t time, int32_t input_dim, int32_t vocab, const float* x,
                     const int32_t* targets, const int32_t* seq_lens, const float* W, const float* b,
                     float epsilon, float* loss, float* dx, float* dW, float* db, int accumulate,
                     void* workspace, size_t workspace_bytes, int32_t* bad_target, sl_stream_t stream);

/* ---- input dropout (the output_prob layer's, models.hpp:18) --------------------
 * The reference's counter-based Tape::dropout (tape.cpp:540-600, applied by
 * eval_layer, compiler.cpp:554-562) on x [B, T, F] keyed by its own Time
 * coordinate: y[b,t,f] = x[b,t,f] / (1 - rate) if
 * u01(mix64(key, mix64(t + 2, b*F + f))) >= rate, else 0 (rng.hpp), bit-identical
 * to the reference.  key = mix64(key0, batch_counter), key0 = mix64(seed,
 * fnv1a("<layer>#<input index>")); batch_counter = *counter (device int32, e.g.
 * the optimizer's step counter, so a captured graph draws a new mask per replay)
 * or counter_value when counter is NULL.  The backward is the same map on dy
 * (the mask is recomputed, never stored).  rate in [0, 1). */
int sl_dropout_fwd(int32_t batch, int32_t time, int32_t features, float rate, uint64_t key0,
                   const int32_t* counter, int64_t counter_value, const float* x, float* y, sl_stream_t stream);
int sl_dropout_bwd(int32_t batch, int32_t time, int32_t features, float rate, uint64_t key0,
                   const int32_t* counter, int64_t counter_value, const float* dy, float* dx, sl_stream_t stream);

/* ---- embedding lookup -------------------------------------------
 * The reference's Linear layer on ids = gather_rows(table, ids) (compiler.cpp:
 * 584-589, tape.cpp:448-492): row r of out (row stride out_ld) = table[ids[r]],
 * table [vocab, dim] fp32.  An id outside [0, vocab) is the reference's
 * IndexError naming the layer: the row is filled with NaN (so the step's loss
 * and gradients become non-finite and sl_adam_step skips the update, as the
 * reference raises before any update) and *bad_row (device int32) receives the
 * first offending row (INT32_MAX when every id is valid) — the host raises
 * after synchronising.  Flags:
 *   SL_EMB_ONES_COLUMN   (bf16 only) also write 1.0 at column dim and zeros up
 *                        to out_ld: the padded layer-0 LSTM input of a layer
 *                        flagged SL_LAYER_X_BF16 (out_ld = sl_lstm_bf16_pitch(dim))
 *   SL_EMB_NEGATIVE_ZERO ids < 0 give zero rows without an error (the decoder's
 *                        previous-target embedding at t = 0: initial_output 0)
 * The backward scatter-adds the d_out rows (stride d_out_ld) into d_table in
 * the reference's order (ascending row per id) — bit-exact, deterministic;
 * without accumulate the untouched rows are zeroed; negative ids add nothing. */
enum sl_embedding_flags { SL_EMB_ONES_COLUMN = 1, SL_EMB_NEGATIVE_ZERO = 2 };
size_t sl_embedding_workspace_size(int64_t n_ids, int32_t vocab);
int sl_embedding_fwd(int64_t n_ids, const int32_t* ids, int32_t vocab, int32_t dim, const float* table,
                     float* out, int64_t out_ld, int flags, int32_t* bad_row, sl_stream_t stream);
int sl_embedding_fwd_bf16(int64_t n_ids, const int32_t* ids, int32_t vocab, int32_t dim, const float* table,
                          void* out_bf16, int64_t out_ld, int flags, int32_t* bad_row, sl_stream_t stream);
int sl_embedding_bwd(int64_t n_ids, const int32_t* ids, int32_t vocab, int32_t dim, const float* d_out,
                     int64_t d_out_ld, float* d_table, int accumulate, void* workspace, size_t workspace_bytes,
                     sl_stream_t stream);

/* ---- measurement hooks (used by bench.py; off by default) -------------------
 * When enabled, every internal kernel phase is bracketed by CUDA events on the
 * stream it is launched on; sl_profile_read folds them into per-phase totals
 * (name, calls, device ms, algorithmic flops / bytes).  Phase names:
 *   k1_xw_gemm, k2_rec_fwd, k3_rec_bwd, k4_dx_gemm, k4_dw_gemm, k4_dr_gemm,
 *   k5_cell_fwd, k5_cell_bwd, k6_grad_norm, k6_adam, k7_logits_gemm, k7_softmax_ce,
 *   k7_dx_gemm, k7_dw_gemm, k8_attention_fwd, k8_attention_bwd, k9_embedding_fwd,
 *   k10_dec_*, k11_dropout,
 *   k9_embedding_bwd */
typedef struct sl_profile_entry {
  char name[32];
  int32_t calls;
  double ms;
  double flops;
  double bytes;
} sl_profile_entry;
int sl_profile_enable(int enable);
int sl_profile_read(sl_profile_entry* out, int max_entries, int reset);
/* Number of this library's kernels launched so far (process-wide). */
unsigned long long sl_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SEQLOOM_CUDA_H_ */
