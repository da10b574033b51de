// Drop-in replacement for the reference's decoder cell:
//
//   Tape::LstmOut Tape::lstm_step(NodeId W, NodeId R, NodeId b, NodeId x, NodeId h_prev, NodeId c_prev)
//       reference core/include/seqloom/tape.hpp:123-129, core/src/tape.cpp:1074-1222
//       called by the RnnCell of the Listing-1 decoder (compiler.cpp:640-650) and by
//       lstm_sequence (layers.cpp:29)
//
// A maintainer removes the CPU definition (tape.cpp:1074-1222) and links this TU
// instead.  It is a member of Tape, so it records its tape
// closure exactly like the reference does — same validation and ShapeError
// messages (tape.cpp:1082-1094), same outputs (h, c with the shapes of h_prev /
// c_prev), same six inputs in the record, same GradBuffer::accumulate contract
// (tape.cpp:76-89, only for inputs that need gradients) — but Z = x W + h R + b,
// the gates, the cell update and the whole backward closure run on the GPU
// through the C ABI (sl_lstm_cell_fwd / sl_lstm_cell_bwd: fp32-class split-bf16
// tensor-core GEMMs + fused gate kernels).  The saved activations [B, 5H] stay
// on the device, captured by the closure as the reference captures its
// shared_ptr<vector> (tape.cpp:1112, 1143-1144).
#include "seqloom/tape.hpp"

#include "dropin_util.hpp"

namespace seqloom {

using namespace cuda_dropin;

Tape::LstmOut Tape::lstm_step(NodeId W, NodeId R, NodeId b, NodeId x, NodeId h_prev, NodeId c_prev) {
  const Tensor& tx = value(x);
  const Tensor& th = value(h_prev);
  const Tensor& tc = value(c_prev);
  const Tensor& tW = value(W);
  const Tensor& tR = value(R);
  const Tensor& tb = value(b);
  if (tx.shape().empty() || tx.shape().back().axis != Axis::Feature) {  // tape.cpp:1082-1084
    throw ShapeError("lstm_step: x must end in Feature axis");
  }
  const std::int64_t D = tx.shape().back().extent;
  const std::int64_t B = tx.size() / D;
  if (tR.shape().size() != 2) throw ShapeError("lstm_step: R must be rank 2");
  const std::int64_t H = tR.shape()[0].extent;
  if (tW.shape().size() != 2 || tW.shape()[0].extent != D || tW.shape()[1].extent != 4 * H ||
      tR.shape()[1].extent != 4 * H || tb.size() != 4 * H || th.size() != B * H || tc.size() != B * H) {
    throw ShapeError("lstm_step: inconsistent shapes: x=" + shape_to_string(tx.shape()) +
                     " W=" + shape_to_string(tW.shape()) + " R=" + shape_to_string(tR.shape()));
  }
  const int prec = precision_from_env();
  const bool ng = any_needs_grad({W, R, b, x, h_prev, c_prev});
  Buf dx = upload(tx), dh = upload(th), dc = upload(tc), dW = upload(tW), dR = upload(tR), db = upload(tb);
  Buf h = alloc((size_t)(B * H)), c = alloc((size_t)(B * H));
  Buf saved = ng ? alloc((size_t)(B * 5 * H)) : nullptr;
  rethrow(sl_lstm_cell_fwd((int32_t)B, (int32_t)D, (int32_t)H, prec, dx->f(), dh->f(), dc->f(), dW->f(), dR->f(),
                           db->f(), h->f(), c->f(), saved ? saved->f() : nullptr, nullptr),
          "lstm_step");
  // both outputs leave the device before the first emit: emit() may grow the node
  // vector, which invalidates the references tx / th / tc / tW / tR / tb
  Tensor h_out = download(*h, th.shape());
  Tensor c_out = download(*c, tc.shape());
  NodeId hid = emit(std::move(h_out), ng);
  NodeId cid = emit(std::move(c_out), ng);
  if (ng) {
    record({W, R, b, x, h_prev, c_prev}, {hid, cid}, [=](const Tape& tp, GradBuffer& g) {
      const Tensor* gh = g.get(hid);
      const Tensor* gc = g.get(cid);
      if (!gh && !gc) return;  // tape.cpp:1147
      Buf ghd = gh ? upload(*gh) : nullptr, gcd = gc ? upload(*gc) : nullptr;
      const bool nx = tp.needs_grad(x), nh = tp.needs_grad(h_prev), nc = tp.needs_grad(c_prev);
      const bool nW = tp.needs_grad(W), nR = tp.needs_grad(R), nb = tp.needs_grad(b);
      Buf gx = nx ? alloc((size_t)(B * D)) : nullptr, gh0 = nh ? alloc((size_t)(B * H)) : nullptr;
      Buf gc0 = nc ? alloc((size_t)(B * H)) : nullptr, gW = nW ? alloc((size_t)(D * 4 * H)) : nullptr;
      Buf gR = nR ? alloc((size_t)(H * 4 * H)) : nullptr, gb = nb ? alloc((size_t)(4 * H)) : nullptr;
      auto p = [](const Buf& q) { return q ? q->f() : nullptr; };
      rethrow(sl_lstm_cell_bwd((int32_t)B, (int32_t)D, (int32_t)H, prec, dx->f(), dh->f(), dc->f(), dW->f(),
                               dR->f(), saved->f(), p(ghd), p(gcd), p(gx), p(gh0), p(gc0), p(gW), p(gR), p(gb), 0,
                               nullptr),
              "lstm_step");
      if (nx) g.accumulate(x, download(*gx, tp.value(x).shape()));
      if (nh) g.accumulate(h_prev, download(*gh0, tp.value(h_prev).shape()));
      if (nc) g.accumulate(c_prev, download(*gc0, tp.value(c_prev).shape()));
      if (nW) g.accumulate(W, download(*gW, tp.value(W).shape()));
      if (nR) g.accumulate(R, download(*gR, tp.value(R).shape()));
      if (nb) g.accumulate(b, download(*gb, tp.value(b).shape()));
    });
  }
  return {hid, cid};
}

}  // namespace seqloom
