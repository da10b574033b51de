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
