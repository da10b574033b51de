// Drop-in replacement for the reference's LSTM layer:
//
//   NodeId seqloom::lstm_sequence(Tape&, NodeId W, NodeId R, NodeId b, NodeId xs, int direction)
//       reference core/include/seqloom/layers.hpp:17, core/src/layers.cpp:8-37
//
// A maintainer links this file INSTEAD of the lstm_sequence definition in
// layers.cpp.  Same signature, same validation and error
// types (layers.cpp:10-16), same output (y [B, T, H], masked positions exactly
// 0, seq_lens carried), same gradients into the same GradBuffer slots — but
// the T per-step tape records of the reference (slice_time, lstm_step,
// stack_time, apply_time_mask, reverse_time_per_seq) become ONE record whose
// backward runs the fused CUDA BPTT through the C ABI (include/seqloom_cuda.h).
//
// The Tape's emit()/record() are private in the reference (tape.hpp:177-180);
// INTEGRATION.md shows the 4-line friend declaration a maintainer adds.  The
// test build (oracle/Makefile: dropin) compiles this TU with SEQLOOM_DROPIN_
// FRIEND_HACK, which exposes them without editing the reference sources.
//
// Precision: SEQLOOM_CUDA_PRECISION=bf16 selects SL_PREC_BF16, default fp32
// (fp32-class split-bf16 tensor cores).  Device buffers come from a process-wide
// pool (dropin_util.hpp): no cudaMalloc per call after warm-up.
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#ifdef SEQLOOM_DROPIN_FRIEND_HACK
// standard headers first, so the access hack only touches the reference's classes
#include <functional>
#include <map>
#include <optional>
#include <span>
#include "seqloom/rng.hpp"
#include "seqloom/tensor.hpp"
#define private public
#include "seqloom/tape.hpp"
#undef private
#endif
#include "seqloom/layers.hpp"
#include "seqloom_cuda.h"
#include "dropin_util.hpp"

namespace seqloom {

using namespace cuda_dropin;

NodeId lstm_sequence(Tape& tape, NodeId W, NodeId R, NodeId b, NodeId xs, int direction) {
  const Tensor& x = tape.value(xs);
  if (!x.has_axis(Axis::Time) || !x.has_axis(Axis::Batch)) {  // layers.cpp:10-13
    throw ShapeError("lstm_sequence: input needs Batch and Time axes, got " +
                     shape_to_string(x.shape()));
  }
  if (direction != 1 && direction != -1) {  // layers.cpp:14-16
    throw std::invalid_argument("lstm_sequence: direction must be +1 or -1");
  }
  const int64_t T = x.extent(Axis::Time);
  const int64_t B = x.extent(Axis::Batch);
  const int64_t D = x.shape().back().extent;
  const int64_t H = tape.value(R).shape()[0].extent;
  const Tensor& tW = tape.value(W);
  const Tensor& tR = tape.value(R);
  const Tensor& tb = tape.value(b);
  if (tW.size() != D * 4 * H || tR.size() != H * 4 * H || tb.size() != 4 * H) {  // tape.cpp:1089-1094
    throw ShapeError("lstm_step: inconsistent shapes: x=" + shape_to_string(x.shape()) +
                     " W=" + shape_to_string(tW.shape()) + " R=" + shape_to_string(tR.shape()));
  }
  std::vector<int32_t> lens = x.seq_lens() ? *x.seq_lens() : std::vector<int32_t>(B, (int32_t)T);

  sl_lstm_layer L{(int32_t)B, (int32_t)T, (int32_t)D, (int32_t)H, 1, direction,
                  precision_from_env(), 0};
  rethrow(sl_lstm_layer_check(&L), "lstm_sequence");
  const bool grad = tape.any_needs_grad({W, R, b, xs});
  auto dx_ = upload(x), dW_ = upload(tW), dR_ = upload(tR), db_ = upload(tb);
  auto dl_ = std::make_shared<DevBuf>(sizeof(int32_t) * B);  // (pool block of B int32)
  ck(cudaMemcpy(dl_->p, lens.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice), "H2D lens");
  auto y_ = alloc((size_t)(B * T * H));
  const size_t ws_bytes = sl_lstm_workspace_size(&L), rs_bytes = sl_lstm_reserve_size(&L);
  auto ws_ = std::make_shared<DevBuf>(ws_bytes);
  auto rs_ = grad ? std::make_shared<DevBuf>(rs_bytes) : nullptr;
  const float* Wp[1] = {dW_->f()};
  const float* Rp[1] = {dR_->f()};
  const float* bp[1] = {db_->f()};
  rethrow(sl_lstm_layer_fwd(&L, dx_->f(), static_cast<int32_t*>(dl_->p), Wp, Rp, bp, y_->f(),
                            nullptr, nullptr, rs_ ? rs_->p : nullptr, rs_ ? rs_bytes : 0, ws_->p,
                            ws_bytes, nullptr),
          "lstm_sequence");
  Tensor y = download(*y_, {{Axis::Batch, B}, {Axis::Time, T}, {Axis::Feature, H}});
  if (x.seq_lens()) y.set_seq_lens(*x.seq_lens());
  NodeId yid = tape.emit(std::move(y), grad);
  if (grad) {
    // ONE tape record for the whole sequence: its backward is the fused BPTT.
    tape.record({W, R, b, xs}, {yid}, [=](const Tape& tp, GradBuffer& g) {
      const Tensor* gy = g.get(yid);
      if (!gy) return;
      auto dy_ = upload(*gy);
      auto gx_ = alloc((size_t)(B * T * D)), gW_ = alloc((size_t)(D * 4 * H));
      auto gR_ = alloc((size_t)(H * 4 * H)), gb_ = alloc((size_t)(4 * H));
      const float* Wq[1] = {dW_->f()};
      const float* Rq[1] = {dR_->f()};
      float* gWq[1] = {gW_->f()};
      float* gRq[1] = {gR_->f()};
      float* gbq[1] = {gb_->f()};
      rethrow(sl_lstm_layer_bwd(&L, dx_->f(), static_cast<int32_t*>(dl_->p), Wq, Rq, dy_->f(),
                                nullptr, nullptr, gx_->f(), gWq, gRq, gbq, 0, rs_->p, rs_bytes,
                                ws_->p, ws_bytes, nullptr),
              "lstm_sequence");
      // GradBuffer::accumulate contract (tape.cpp:76-89), only for inputs needing grads
      if (tp.needs_grad(xs)) g.accumulate(xs, download(*gx_, tp.value(xs).shape()));
      if (tp.needs_grad(W)) g.accumulate(W, download(*gW_, tp.value(W).shape()));
      if (tp.needs_grad(R)) g.accumulate(R, download(*gR_, tp.value(R).shape()));
      if (tp.needs_grad(b)) g.accumulate(b, download(*gb_, tp.value(b).shape()));
    });
  }
  return yid;
}

}  // namespace seqloom
