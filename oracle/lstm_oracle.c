/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C (fp64) restatement of the reference's LSTM hot path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker or the timed CPU baseline — never as
 * the product path.  Parity pinned against (a) the reference itself compiled
 * from /root/reference into oracle/_ref/ (tests/test_oracle.py), (b) the
 * reference's own known-answer values (tape_test.cpp:191-213)
 * and (c) the committed golden fixtures under tests/golden/ produced by the
 * reference build (tests/golden/make_golden.py).
 *
 * Layouts are the reference's (tensor.hpp:21 canonical axis order, row-major):
 *   x  [B, T, D]   y [B, T, H]   W [D, 4H]   R [H, 4H]   b [4H]
 * Gate blocks in Z are (i | f | g | o), each H wide (tape.cpp:1095, 1123-1126).
 *
 *   forward step   tape.cpp:1103-1135
 *   backward step  tape.cpp:1152-1215
 *   sequence       layers.cpp:22-36 (zero h0/c0, T steps on padded input too,
 *                  stack_time, apply_time_mask tape.cpp:797, per-sequence
 *                  prefix reversal tape.cpp:846 for direction -1)
 *
 * Extension beyond the reference (which never returns final states,
 * layers.cpp:36): h_last / c_last are the states after processing step
 * len-1 (torch.nn.LSTM semantics), and dh_last / dc_last are
 * injected as upstream gradients at that step.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

static double sigm(double z) { return 1.0 / (1.0 + exp(-z)); }

/* tape.cpp:846 — source time index of step t under per-sequence reversal */
static int src_time(int t, int len, int dir) {
  if (dir > 0) return t;
  return t < len ? len - 1 - t : t;
}

/* One step.  saved (optional) receives [B, 5H] = (i, f, g, o, tanh c). */
void orc_lstm_step_fwd(int B, int D, int H, const double* x, const double* h0,
                       const double* c0, const double* W, const double* R,
                       const double* b, double* h, double* c, double* saved) {
  const int G = 4 * H;
  double* z = (double*)malloc(sizeof(double) * (size_t)G);
  for (int r = 0; r < B; ++r) {
    for (int j = 0; j < G; ++j) {
      double acc = 0.0;
      for (int k = 0; k < D; ++k) acc += x[(size_t)r * D + k] * W[(size_t)k * G + j];
      for (int k = 0; k < H; ++k) acc += h0[(size_t)r * H + k] * R[(size_t)k * G + j];
      z[j] = acc + b[j];
    }
    for (int j = 0; j < H; ++j) {
      double gi = sigm(z[j]), gf = sigm(z[H + j]), gg = tanh(z[2 * H + j]);
      double go = sigm(z[3 * H + j]);
      double cn = gf * c0[(size_t)r * H + j] + gi * gg;
      double tc = tanh(cn);
      c[(size_t)r * H + j] = cn;
      h[(size_t)r * H + j] = go * tc;
      if (saved) {
        double* sv = saved + (size_t)r * 5 * H;
        sv[j] = gi;
        sv[H + j] = gf;
        sv[2 * H + j] = gg;
        sv[3 * H + j] = go;
        sv[4 * H + j] = tc;
      }
    }
  }
  free(z);
}

/* Backward of one step given saved activations (tape.cpp:1152-1215).
 * gh / gc may be NULL (treated as zero).  Outputs are ACCUMULATED (+=) into
 * dx, dh0, dc0, dW, dR, db — the GradBuffer::accumulate contract
 * (tape.cpp:76-89).  Any output pointer may be NULL. */
void orc_lstm_step_bwd(int B, int D, int H, const double* x, const double* h0,
                       const double* c0, const double* W, const double* R,
                       const double* saved, const double* gh, const double* gc,
                       double* dx, double* dh0, double* dc0, double* dW, double* dR,
                       double* db) {
  const int G = 4 * H;
  double* dz = (double*)malloc(sizeof(double) * (size_t)G);
  for (int r = 0; r < B; ++r) {
    const double* sv = saved + (size_t)r * 5 * H;
    for (int j = 0; j < H; ++j) {
      size_t idx = (size_t)r * H + j;
      double ghv = gh ? gh[idx] : 0.0, gcv = gc ? gc[idx] : 0.0;
      double gi = sv[j], gf = sv[H + j], gg = sv[2 * H + j], go = sv[3 * H + j];
      double tc = sv[4 * H + j];
      double d_o = ghv * tc;
      double d_c = gcv + ghv * go * (1.0 - tc * tc);
      if (dc0) dc0[idx] += d_c * gf;
      dz[j] = d_c * gg * gi * (1.0 - gi);
      dz[H + j] = d_c * c0[idx] * gf * (1.0 - gf);
      dz[2 * H + j] = d_c * gi * (1.0 - gg * gg);
      dz[3 * H + j] = d_o * go * (1.0 - go);
    }
    for (int j = 0; j < G; ++j) {
      if (db) db[j] += dz[j];
      if (dW)
        for (int k = 0; k < D; ++k) dW[(size_t)k * G + j] += x[(size_t)r * D + k] * dz[j];
      if (dR)
        for (int k = 0; k < H; ++k) dR[(size_t)k * G + j] += h0[(size_t)r * H + k] * dz[j];
    }
    if (dx)
      for (int k = 0; k < D; ++k) {
        double acc = 0.0;
        for (int j = 0; j < G; ++j) acc += dz[j] * W[(size_t)k * G + j];
        dx[(size_t)r * D + k] += acc;
      }
    if (dh0)
      for (int k = 0; k < H; ++k) {
        double acc = 0.0;
        for (int j = 0; j < G; ++j) acc += dz[j] * R[(size_t)k * G + j];
        dh0[(size_t)r * H + k] += acc;
      }
  }
  free(dz);
}

/* Internal: run the full forward, keeping per-step states/activations in
 * processing order.  hs/cs are [T+1, B, H] (slot 0 = zero initial state),
 * sv is [T, B, 5H], xs is [T, B, D] (the step inputs after reversal). */
static void seq_forward(int B, int T, int D, int H, int dir, const double* x, const int* lens,
                        const double* W, const double* R, const double* b, double* hs,
                        double* cs, double* sv, double* xs) {
  memset(hs, 0, sizeof(double) * (size_t)B * H);
  memset(cs, 0, sizeof(double) * (size_t)B * H);
  for (int s = 0; s < T; ++s) {
    for (int r = 0; r < B; ++r) {
      int t = src_time(s, lens[r], dir);
      memcpy(xs + ((size_t)s * B + r) * D, x + ((size_t)r * T + t) * D, sizeof(double) * (size_t)D);
    }
    orc_lstm_step_fwd(B, D, H, xs + (size_t)s * B * D, hs + (size_t)s * B * H,
                      cs + (size_t)s * B * H, W, R, b, hs + (size_t)(s + 1) * B * H,
                      cs + (size_t)(s + 1) * B * H, sv + (size_t)s * B * 5 * H);
  }
}

/* lstm_sequence forward (layers.cpp:8-37).  h_last/c_last may be NULL. */
void orc_lstm_sequence_fwd(int B, int T, int D, int H, int dir, const double* x,
                           const int* lens, const double* W, const double* R, const double* b,
                           double* y, double* h_last, double* c_last) {
  double* hs = (double*)malloc(sizeof(double) * (size_t)(T + 1) * B * H);
  double* cs = (double*)malloc(sizeof(double) * (size_t)(T + 1) * B * H);
  double* sv = (double*)malloc(sizeof(double) * (size_t)T * B * 5 * H);
  double* xs = (double*)malloc(sizeof(double) * (size_t)T * B * D);
  seq_forward(B, T, D, H, dir, x, lens, W, R, b, hs, cs, sv, xs);
  for (int r = 0; r < B; ++r) {
    for (int s = 0; s < T; ++s) {
      int t = src_time(s, lens[r], dir);
      const double* hsrc = hs + ((size_t)(s + 1) * B + r) * H;
      double* dst = y + ((size_t)r * T + t) * H;
      for (int j = 0; j < H; ++j) dst[j] = s < lens[r] ? hsrc[j] : 0.0; /* tape.cpp:797 */
    }
    int sl = lens[r];
    if (h_last) memcpy(h_last + (size_t)r * H, hs + ((size_t)sl * B + r) * H, sizeof(double) * (size_t)H);
    if (c_last) memcpy(c_last + (size_t)r * H, cs + ((size_t)sl * B + r) * H, sizeof(double) * (size_t)H);
  }
  free(hs);
  free(cs);
  free(sv);
  free(xs);
}

/* lstm_sequence backward: BPTT as the tape replays the per-step closures in
 * reverse (tape.cpp:1363-1381).  dy [B,T,H] (masked positions ignored, the
 * apply_time_mask adjoint tape.cpp:813-814); dh_last/dc_last optional.
 * Outputs are OVERWRITTEN (dx [B,T,D], dW, dR, db); any may be NULL. */
void orc_lstm_sequence_bwd(int B, int T, int D, int H, int dir, const double* x,
                           const int* lens, const double* W, const double* R, const double* b,
                           const double* dy, const double* dh_last, const double* dc_last,
                           double* dx, double* dW, double* dR, double* db) {
  const size_t BH = (size_t)B * H;
  double* hs = (double*)malloc(sizeof(double) * (size_t)(T + 1) * BH);
  double* cs = (double*)malloc(sizeof(double) * (size_t)(T + 1) * BH);
  double* sv = (double*)malloc(sizeof(double) * (size_t)T * BH * 5);
  double* xs = (double*)malloc(sizeof(double) * (size_t)T * B * D);
  double* gh = (double*)calloc(BH, sizeof(double));
  double* gc = (double*)calloc(BH, sizeof(double));
  double* ngh = (double*)calloc(BH, sizeof(double));
  double* ngc = (double*)calloc(BH, sizeof(double));
  double* dxs = (double*)calloc((size_t)B * D, sizeof(double));
  seq_forward(B, T, D, H, dir, x, lens, W, R, b, hs, cs, sv, xs);
  if (dx) memset(dx, 0, sizeof(double) * (size_t)B * T * D);
  if (dW) memset(dW, 0, sizeof(double) * (size_t)D * 4 * H);
  if (dR) memset(dR, 0, sizeof(double) * (size_t)H * 4 * H);
  if (db) memset(db, 0, sizeof(double) * (size_t)4 * H);
  /* gh/gc hold the carried recurrent gradient flowing into step s */
  for (int s = T - 1; s >= 0; --s) {
    for (int r = 0; r < B; ++r) {
      int t = src_time(s, lens[r], dir);
      for (int j = 0; j < H; ++j) {
        size_t idx = (size_t)r * H + j;
        double ext = (s < lens[r] && dy) ? dy[((size_t)r * T + t) * H + j] : 0.0;
        if (s == lens[r] - 1) {
          if (dh_last) ext += dh_last[idx];
          if (dc_last) gc[idx] += dc_last[idx];
        }
        gh[idx] += ext;
      }
    }
    memset(ngh, 0, sizeof(double) * BH);
    memset(ngc, 0, sizeof(double) * BH);
    memset(dxs, 0, sizeof(double) * (size_t)B * D);
    orc_lstm_step_bwd(B, D, H, xs + (size_t)s * B * D, hs + (size_t)s * BH, cs + (size_t)s * BH,
                      W, R, sv + (size_t)s * BH * 5, gh, gc, dxs, ngh, ngc, dW, dR, db);
    if (dx)
      for (int r = 0; r < B; ++r) {
        int t = src_time(s, lens[r], dir);
        double* dst = dx + ((size_t)r * T + t) * D;
        for (int k = 0; k < D; ++k) dst[k] += dxs[(size_t)r * D + k];
      }
    memcpy(gh, ngh, sizeof(double) * BH);
    memcpy(gc, ngc, sizeof(double) * BH);
  }
  free(hs);
  free(cs);
  free(sv);
  free(xs);
  free(gh);
  free(gc);
  free(ngh);
  free(ngc);
  free(dxs);
}
