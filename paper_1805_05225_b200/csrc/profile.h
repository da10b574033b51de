// Opt-in per-phase CUDA-event timing + launch counting behind sl_profile_*.
// Events are recorded on the stream the phase's kernels are launched on, so
// the bench's roofline numbers come from the launching stream.
#pragma once
#include "common.cuh"

namespace sl {

bool profile_enabled();
void count_launch(int n = 1);

// Records a start event on construction and a stop event on destruction
// (when profiling is enabled).  `flops` / `bytes` are the phase's
// ALGORITHMIC work, accumulated per name.
class Phase {
 public:
  Phase(cudaStream_t s, const char* name, double flops, double bytes = 0.0);
  ~Phase();
  Phase(const Phase&) = delete;
  Phase& operator=(const Phase&) = delete;

 private:
  cudaStream_t stream_;
  int slot_ = -1;
};

}  // namespace sl
