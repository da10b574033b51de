// Persistent recurrence kernels (K2 forward, K3 BPTT) — argument blocks.
#pragma once
#include "common.cuh"

namespace sl {

// Saved-activation layout shared by the forward and backward kernels, all
// indexed by (b, t) at the ORIGINAL time position t = src_time(s, len[b], dir)
// of processing step s, rows of width given below:
//   gates [B*T, 4H]  activated (i, f, g, o)         (reference saves these, tape.cpp:1129-1133)
//   cprev [B*T, H]   c_{s-1} (reference reads tp.value(c_prev), tape.cpp:1150)
//   hprev [B*T, H]   h_{s-1} (input of the hoisted dR GEMM, replaces tape.cpp:1198-1205)
// tanh(c_s) is recomputed from f*c_{s-1} + i*g instead of being stored.
struct RecFwdArgs {
  int B, T, H, nd, U, ctas_per_dir;
  const int32_t* lens;
  int dirsign[2];
  const float* xw[2];  // [B*T, xw_ld] input projection incl. bias, gate blocks of dir d at col 0
  int64_t xw_ld;
  const float* R[2];   // [H, 4H]
  float* y;            // [B*T, y_ld]; dir d writes cols [d*H, d*H+H)
  int64_t y_ld;
  float* h_last;       // [nd, B, H] or null
  float* c_last;
  float* gates[2];     // saved (null in inference)
  float* cprev[2];
  float* hprev[2];
  float* hbuf[2];      // work [2, B, H], slot 0 zeroed
  float* cbuf[2];      // work [B, H], zeroed
  unsigned* bar;       // [2] zeroed barrier counters
};

struct RecBwdArgs {
  int B, T, H, nd, U, ctas_per_dir;
  const int32_t* lens;
  int dirsign[2];
  const float* R[2];
  const float* gates[2];
  const float* cprev[2];
  const float* dy;  // [B*T, dy_ld]; dir d reads cols [d*H, d*H+H)
  int64_t dy_ld;
  const float* dh_last;  // [nd, B, H] or null
  const float* dc_last;
  float* dz[2];     // out [B*T, 4H] (zero at padded positions)
  float* dzbuf[2];  // work [2, B, 4H], zeroed
  float* gcbuf[2];  // work [B, H], zeroed
  float* db[2];     // [4H] or null
  int accumulate;
  unsigned* bar;
};

void rec_fwd_f32(const RecFwdArgs& a, cudaStream_t stream);
void rec_bwd_f32(const RecBwdArgs& a, cudaStream_t stream);

// Units per CTA for a layer, and CTAs per direction.
void rec_partition(int H, int nd, int* U, int* ctas_per_dir);

}  // namespace sl
