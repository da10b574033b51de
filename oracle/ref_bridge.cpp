// ORACLE TEST INFRASTRUCTURE — not product code.  Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference leg may load what this builds.
//
// A C-ABI wrapper around the REFERENCE implementation itself, compiled from
// the unmodified reference sources under /root/reference (see oracle/Makefile)
// into oracle/_ref/libseqloom_ref{32,64}.so.  It drives the reference's own
// public API exactly as its callers do:
//   * seqloom::lstm_sequence(Tape&, W, R, b, xs, direction)   (layers.cpp:8-37)
//   * Tape::lstm_step(W, R, b, x, h_prev, c_prev)              (tape.cpp:1074-1222)
//   * a BLSTM stack wired like eval_layer's Rec branch: input =
//     concat_feature([fw, bw]) of the previous layer            (compiler.cpp:600-608)
// and obtains gradients with Tape::backward + param_gradients
// (tape.cpp:1363-1389).  The upstream gradient dy enters through the scalar
// loss L = sum(y * dy) built from reference tape ops, so dL/dy == dy.
//
// All buffers cross the ABI as double; the library's Real is float (…32.so)
// or double (…64.so, -DSEQLOOM_REAL_DOUBLE) exactly as the reference's two
// core builds (core/CMakeLists.txt:21-42).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "seqloom/layers.hpp"
#include "seqloom/param_store.hpp"
#include "seqloom/rng.hpp"
#include "seqloom/tape.hpp"

using namespace seqloom;

namespace {

Tensor make(Shape s, const double* src) {
  Tensor t = Tensor::zeros(std::move(s));
  auto d = t.data();
  for (std::size_t i = 0; i < d.size(); ++i) d[i] = static_cast<Real>(src[i]);
  return t;
}

void put(const Tensor& t, double* dst) {
  if (!dst) return;
  auto d = t.data();
  for (std::size_t i = 0; i < d.size(); ++i) dst[i] = static_cast<double>(d[i]);
}

int fail(const std::exception& e, char* err, int errlen) {
  if (err && errlen > 0) std::snprintf(err, static_cast<std::size_t>(errlen), "%s", e.what());
  return 1;
}

NodeId sum_all(Tape& t, NodeId v) {
  for (Axis a : {Axis::Feature, Axis::Time, Axis::Batch}) {
    if (t.value(v).has_axis(a)) v = t.reduce_sum(v, a);
  }
  return v;
}

}  // namespace

extern "C" {

int ref_real_bytes() { return static_cast<int>(sizeof(Real)); }

// The reference ParamStore's manifest order (param_store.hpp:12, 40-45) for the
// '\n'-separated names in `names`: written back '\n'-separated into out.
int ref_param_manifest_order(const char* names, char* out, int outlen, char* err, int errlen) {
  try {
    ParamStore ps;
    std::string all(names), cur;
    for (char ch : all + "\n") {
      if (ch == '\n') {
        if (!cur.empty()) ps.insert(cur, Tensor::zeros(Shape{{Axis::Feature, 1}}));
        cur.clear();
      } else {
        cur += ch;
      }
    }
    std::string res;
    for (const auto& [name, shape] : ps.manifest()) res += name + "\n";
    if ((int)res.size() + 1 > outlen) throw std::runtime_error("ref_param_manifest_order: out too small");
    std::memcpy(out, res.c_str(), res.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// One LSTM layer over [B, T, D].  dy == nullptr → forward only.
int ref_lstm_sequence(int B, int T, int D, int H, int direction, const double* x,
                      const int* lens, const double* W, const double* R, const double* b,
                      const double* dy, double* y, double* dx, double* dW, double* dR,
                      double* db, char* err, int errlen) {
  try {
    Tape t(dy != nullptr);
    Tensor xt = make({{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, D}}, x);
    std::vector<std::int32_t> lv(lens, lens + B);
    xt.set_seq_lens(lv);
    NodeId xn = dy ? t.param("x", xt) : t.constant(xt);
    NodeId Wn = t.param("W", make({{Axis::Feature, D}, {Axis::Other, 4 * H}}, W));
    NodeId Rn = t.param("R", make({{Axis::Feature, H}, {Axis::Other, 4 * H}}, R));
    NodeId bn = t.param("b", make({{Axis::Feature, 4 * H}}, b));
    NodeId yn = lstm_sequence(t, Wn, Rn, bn, xn, direction);
    put(t.value(yn), y);
    if (!dy) return 0;
    Tensor dyt = make({{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, H}}, dy);
    dyt.set_seq_lens(lv);
    NodeId loss = sum_all(t, t.mul(yn, t.constant(dyt)));
    GradBuffer g = t.backward(loss);
    auto grads = t.param_gradients(g);
    put(grads.at("x"), dx);
    put(grads.at("W"), dW);
    put(grads.at("R"), dR);
    put(grads.at("b"), db);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// One Tape::lstm_step with upstream grads gh, gc (either may be null).
int ref_lstm_step(int B, int D, int H, const double* x, const double* h0, const double* c0,
                  const double* W, const double* R, const double* b, const double* gh,
                  const double* gc, double* h, double* c, double* dx, double* dh0, double* dc0,
                  double* dW, double* dR, double* db, char* err, int errlen) {
  try {
    const bool grad = gh || gc;
    Tape t(grad);
    auto leaf = [&](const char* name, Tensor v) { return grad ? t.param(name, v) : t.constant(v); };
    NodeId xn = leaf("x", make({{Axis::Batch, B}, {Axis::Feature, D}}, x));
    NodeId hn = leaf("h0", make({{Axis::Batch, B}, {Axis::Feature, H}}, h0));
    NodeId cn = leaf("c0", make({{Axis::Batch, B}, {Axis::Feature, H}}, c0));
    NodeId Wn = leaf("W", make({{Axis::Feature, D}, {Axis::Other, 4 * H}}, W));
    NodeId Rn = leaf("R", make({{Axis::Feature, H}, {Axis::Other, 4 * H}}, R));
    NodeId bn = leaf("b", make({{Axis::Feature, 4 * H}}, b));
    auto out = t.lstm_step(Wn, Rn, bn, xn, hn, cn);
    put(t.value(out.h), h);
    put(t.value(out.c), c);
    if (!grad) return 0;
    NodeId loss = kNoNode;
    if (gh) loss = sum_all(t, t.mul(out.h, t.constant(make({{Axis::Batch, B}, {Axis::Feature, H}}, gh))));
    if (gc) {
      NodeId lc = sum_all(t, t.mul(out.c, t.constant(make({{Axis::Batch, B}, {Axis::Feature, H}}, gc))));
      loss = loss == kNoNode ? lc : t.add(loss, lc);
    }
    GradBuffer g = t.backward(loss);
    auto grads = t.param_gradients(g);
    put(grads.at("x"), dx);
    put(grads.at("h0"), dh0);
    put(grads.at("c0"), dc0);
    put(grads.at("W"), dW);
    put(grads.at("R"), dR);
    put(grads.at("b"), db);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// The graph of the reference's own finite-difference test of lstm_step
// (tape_test.cpp:477-492): out = lstm_step(W,R,b,x,h0,c0); out2 = lstm_step(W,R,b,x,out.h,out.c);
// L = sum(out2.h) + sum(out.h); all six inputs are parameters.  Writes L and the gradients.
int ref_lstm_two_steps(int B, int D, int H, const double* x, const double* h0, const double* c0,
                       const double* W, const double* R, const double* b, double* loss, double* dx,
                       double* dh0, double* dc0, double* dW, double* dR, double* db, char* err, int errlen) {
  try {
    Tape t;
    NodeId Wn = t.param("W", make({{Axis::Feature, D}, {Axis::Other, 4 * H}}, W));
    NodeId Rn = t.param("R", make({{Axis::Feature, H}, {Axis::Other, 4 * H}}, R));
    NodeId bn = t.param("b", make({{Axis::Feature, 4 * H}}, b));
    NodeId xn = t.param("x", make({{Axis::Batch, B}, {Axis::Feature, D}}, x));
    NodeId hn = t.param("h0", make({{Axis::Batch, B}, {Axis::Feature, H}}, h0));
    NodeId cn = t.param("c0", make({{Axis::Batch, B}, {Axis::Feature, H}}, c0));
    auto out = t.lstm_step(Wn, Rn, bn, xn, hn, cn);
    auto out2 = t.lstm_step(Wn, Rn, bn, xn, out.h, out.c);
    NodeId l = t.add(sum_all(t, out2.h), sum_all(t, out.h));
    *loss = static_cast<double>(t.value(l).scalar_value());
    GradBuffer g = t.backward(l);
    auto grads = t.param_gradients(g);
    put(grads.at("x"), dx);
    put(grads.at("h0"), dh0);
    put(grads.at("c0"), dc0);
    put(grads.at("W"), dW);
    put(grads.at("R"), dR);
    put(grads.at("b"), db);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// The decoder output layer + loss exactly as the reference builds it:
// ce_label_smoothing(log_softmax(add(matmul(x, W), b)), targets, eps)
// (compiler.cpp:651-663, tape.cpp:879-924, 1224-1298), gradients by
// Tape::backward.  x [B, T, D], targets [B, T] (seq_lens mask), W [D, V].
int ref_output_ce(int B, int T, int D, int V, const double* x, const int* lens, const int* targets,
                  const double* W, const double* b, double eps, double* loss, double* dx, double* dW,
                  double* db, char* err, int errlen) {
  try {
    Tape t(true);
    std::vector<std::int32_t> lv(lens, lens + B);
    Tensor xt = make({{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, D}}, x);
    xt.set_seq_lens(lv);
    NodeId xn = t.param("x", xt);
    NodeId Wn = t.param("W", make({{Axis::Feature, D}, {Axis::Other, V}}, W));
    NodeId bn = t.param("b", make({{Axis::Feature, V}}, b));
    IdTensor ids = IdTensor::from_data({{Axis::Batch, B}, {Axis::Time, T}},
                                       std::vector<std::int32_t>(targets, targets + B * T));
    ids.set_seq_lens(lv);
    NodeId lp = t.log_softmax(t.add(t.matmul(xn, Wn), bn));
    NodeId ln = t.ce_label_smoothing(lp, ids, static_cast<Real>(eps), "output_prob");
    *loss = static_cast<double>(t.value(ln).scalar_value());
    GradBuffer g = t.backward(ln);
    auto grads = t.param_gradients(g);
    put(grads.at("x"), dx);
    put(grads.at("W"), dW);
    put(grads.at("b"), db);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// The reference's embedding lookup, Tape::gather_rows(table, ids, layer)
// (tape.cpp:448-492), over ids [B, T]; with d_out, the table gradient through
// L = sum(out * d_out), so dL/d(out) == d_out.  An out-of-range id is the
// reference's IndexError (message names the layer) → returned as an error.
int ref_gather_rows(int B, int T, int V, int D, const double* table, const int* ids, const double* d_out,
                    double* out, double* d_table, char* err, int errlen) {
  try {
    Tape t(d_out != nullptr);
    NodeId tb = t.param("emb/W", make({{Axis::Feature, V}, {Axis::Other, D}}, table));
    IdTensor it = IdTensor::from_data({{Axis::Batch, B}, {Axis::Time, T}},
                                      std::vector<std::int32_t>(ids, ids + (std::size_t)B * T));
    NodeId on = t.gather_rows(tb, it, "emb");
    put(t.value(on), out);
    if (!d_out) return 0;
    NodeId gy = t.constant(make({{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, D}}, d_out));
    NodeId loss = sum_all(t, t.mul(on, gy));
    GradBuffer g = t.backward(loss);
    put(t.param_gradients(g).at("emb/W"), d_table);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// The reference's input dropout as eval_layer applies it (compiler.cpp:554-562 ->
// Tape::dropout, tape.cpp:540-600) to a [B, T, F] value computed once per batch
// (kStaticStep: elements keyed by their own Time coordinate), with the layer key
// mix64(mix64(seed, fnv1a(qualified + "#" + input_index)), batch_counter); with
// d_out, the gradient through L = sum(out * d_out).
int ref_dropout(int B, int T, int F, const double* x, double rate, unsigned long long seed, const char* qualified,
                int input_index, unsigned long long batch_counter, const double* d_out, double* out, double* dx,
                char* err, int errlen) {
  try {
    Tape t(d_out != nullptr);
    NodeId xn = t.param("x", make({{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, F}}, x));
    DropoutKey key{mix64(mix64(seed, fnv1a(std::string(qualified) + "#" + std::to_string(input_index))),
                         batch_counter)};
    NodeId on = t.dropout(xn, static_cast<Real>(rate), key, kStaticStep, true);
    put(t.value(on), out);
    if (!d_out) return 0;
    NodeId gy = t.constant(make({{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, F}}, d_out));
    NodeId loss = sum_all(t, t.mul(on, gy));
    GradBuffer g = t.backward(loss);
    put(t.param_gradients(g).at("x"), dx);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// One MLP-attention step of the Listing-1 decoder subnet, built from the
// reference's own layer ops exactly as eval_layer wires it (models.cpp:107-154,
// compiler.cpp:616-639): s_tr = s W_s + b_s; weight_feedback = accum W_fb +
// b_fb; e = tanh(enc_ctx + weight_feedback + s_tr) v + b_v; a =
// softmax_over_spatial(e) (tape.cpp:926-985); accum' = accum + a; att =
// generic_attention(a, enc) (tape.cpp:987-1072).  The upstream gradients
// d_att [B, E] and d_accum [B, Ts] enter through L = sum(att d_att) +
// sum(accum' d_accum).  Outputs (optional): att, a, accum' and the gradients.
int ref_attention_step(int B, int Ts, int K, int E, int H, const int* lens, const double* enc_ctx,
                       const double* enc, const double* s, const double* accum, const double* Ws,
                       const double* bs, const double* Wfb, const double* bfb, const double* v, double bv,
                       const double* d_att, const double* d_accum, double* att, double* a, double* accum2,
                       double* g_enc_ctx, double* g_enc, double* g_s, double* g_accum, double* g_Ws,
                       double* g_bs, double* g_Wfb, double* g_bfb, double* g_v, double* g_bv, char* err,
                       int errlen) {
  try {
    const bool grad = d_att != nullptr;
    Tape t(grad);
    std::vector<std::int32_t> lv(lens, lens + B);
    auto leaf = [&](const char* name, Tensor x) { return grad ? t.param(name, x) : t.constant(x); };
    Tensor tc_ = make({{Axis::Batch, B}, {Axis::Time, Ts}, {Axis::Feature, K}}, enc_ctx);
    tc_.set_seq_lens(lv);
    Tensor te = make({{Axis::Batch, B}, {Axis::Time, Ts}, {Axis::Feature, E}}, enc);
    te.set_seq_lens(lv);
    Tensor ta = make({{Axis::Batch, B}, {Axis::Time, Ts}, {Axis::Feature, 1}}, accum);
    ta.set_seq_lens(lv);
    NodeId ctxn = leaf("enc_ctx", tc_), encn = leaf("enc", te), accn = leaf("accum", ta);
    NodeId sn = leaf("s", make({{Axis::Batch, B}, {Axis::Feature, H}}, s));
    NodeId Wsn = leaf("Ws", make({{Axis::Feature, H}, {Axis::Other, K}}, Ws));
    NodeId bsn = leaf("bs", make({{Axis::Feature, K}}, bs));
    NodeId Wfbn = leaf("Wfb", make({{Axis::Feature, 1}, {Axis::Other, K}}, Wfb));
    NodeId bfbn = leaf("bfb", make({{Axis::Feature, K}}, bfb));
    NodeId vn = leaf("v", make({{Axis::Feature, K}, {Axis::Other, 1}}, v));
    NodeId bvn = leaf("bv", make({{Axis::Feature, 1}}, &bv));
    NodeId s_tr = t.add(t.matmul(sn, Wsn), bsn);
    NodeId fb = t.add(t.matmul(accn, Wfbn), bfbn);
    NodeId e_in = t.add(t.add(ctxn, fb), s_tr);
    NodeId e = t.add(t.matmul(t.tanh(e_in), vn), bvn);
    NodeId an = t.softmax_over_spatial(e);
    NodeId acc2 = t.add(accn, an);
    NodeId attn = t.generic_attention(an, encn);
    put(t.value(attn), att);
    put(t.value(an), a);
    put(t.value(acc2), accum2);
    if (!grad) return 0;
    NodeId loss = sum_all(t, t.mul(attn, t.constant(make({{Axis::Batch, B}, {Axis::Feature, E}}, d_att))));
    if (d_accum) {
      Tensor tda = make({{Axis::Batch, B}, {Axis::Time, Ts}, {Axis::Feature, 1}}, d_accum);
      tda.set_seq_lens(lv);
      loss = t.add(loss, sum_all(t, t.mul(acc2, t.constant(tda))));
    }
    GradBuffer g = t.backward(loss);
    auto grads = t.param_gradients(g);
    put(grads.at("enc_ctx"), g_enc_ctx);
    put(grads.at("enc"), g_enc);
    put(grads.at("s"), g_s);
    put(grads.at("accum"), g_accum);
    put(grads.at("Ws"), g_Ws);
    put(grads.at("bs"), g_bs);
    put(grads.at("Wfb"), g_Wfb);
    put(grads.at("bfb"), g_bfb);
    put(grads.at("v"), g_v);
    put(grads.at("bv"), g_bv);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// An L-layer bidirectional LSTM stack, each layer's input the feature concat
// [fw ‖ bw] of the previous layer (compiler.cpp:600-608 with the Listing-1
// enc{i}_fw / enc{i}_bw topology, models.cpp).  params[l*6 + {0..5}] =
// W_fw, R_fw, b_fw, W_bw, R_bw, b_bw of layer l; D_l = D0 for l = 0 else 2H.
// grads (optional, same layout) receive parameter gradients; dx the input
// gradient.  dy is the upstream gradient of the top layer's [B, T, 2H] output.
int ref_blstm_stack(int L, int B, int T, int D0, int H, const double* x, const int* lens,
                    const double* const* params, const double* dy, double* y, double* dx,
                    double* const* grads, char* err, int errlen) {
  try {
    Tape t(dy != nullptr);
    Tensor xt = make({{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, D0}}, x);
    std::vector<std::int32_t> lv(lens, lens + B);
    xt.set_seq_lens(lv);
    NodeId in = dy ? t.param("x", xt) : t.constant(xt);
    for (int l = 0; l < L; ++l) {
      const int D = l == 0 ? D0 : 2 * H;
      NodeId outs[2];
      for (int d = 0; d < 2; ++d) {
        const std::string q = "enc" + std::to_string(l) + (d == 0 ? "_fw" : "_bw");
        const double* const* p = params + l * 6 + d * 3;
        NodeId Wn = t.param(q + "/W", make({{Axis::Feature, D}, {Axis::Other, 4 * H}}, p[0]));
        NodeId Rn = t.param(q + "/R", make({{Axis::Feature, H}, {Axis::Other, 4 * H}}, p[1]));
        NodeId bn = t.param(q + "/b", make({{Axis::Feature, 4 * H}}, p[2]));
        outs[d] = lstm_sequence(t, Wn, Rn, bn, in, d == 0 ? 1 : -1);
      }
      in = t.concat_feature(std::span<const NodeId>(outs, 2));
    }
    put(t.value(in), y);
    if (!dy) return 0;
    Tensor dyt = make({{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, 2 * H}}, dy);
    dyt.set_seq_lens(lv);
    NodeId loss = sum_all(t, t.mul(in, t.constant(dyt)));
    GradBuffer g = t.backward(loss);
    auto gr = t.param_gradients(g);
    put(gr.at("x"), dx);
    if (grads) {
      for (int l = 0; l < L; ++l) {
        for (int d = 0; d < 2; ++d) {
          const std::string q = "enc" + std::to_string(l) + (d == 0 ? "_fw" : "_bw");
          put(gr.at(q + "/W"), grads[l * 6 + d * 3 + 0]);
          put(gr.at(q + "/R"), grads[l * 6 + d * 3 + 1]);
          put(gr.at(q + "/b"), grads[l * 6 + d * 3 + 2]);
        }
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

}  // extern "C"
