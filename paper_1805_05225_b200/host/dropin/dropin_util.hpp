// Shared host plumbing of the drop-in TUs (layers_cuda.cpp, tape_lstm_step_cuda.cpp):
// device buffers from a process-wide size-keyed pool (no cudaMalloc / cudaFree per
// tape op after warm-up), host <-> device copies of reference Tensors (Real = float:
// straight from the tensor's storage; Real = double: through an fp32 staging vector,
// the C ABI is fp32), and the C-ABI status -> reference exception mapping.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "seqloom/tensor.hpp"
#include "seqloom_cuda.h"

namespace seqloom {
namespace cuda_dropin {

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("seqloom cuda drop-in: ") + what + ": " +
                                                 cudaGetErrorString(e));
}

// C-ABI status -> the reference's exception types (layers.cpp:10-16, tape.cpp:1082-1094)
inline void rethrow(int rc, const char* op) {
  if (rc == SL_OK) return;
  const std::string msg = sl_last_error();
  if (rc == SL_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == SL_ERR_SHAPE) throw ShapeError(msg);
  throw std::runtime_error(std::string(op) + " (cuda): " + msg);
}

class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  void* take(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = free_.find(bytes);
    if (it != free_.end()) {
      void* p = it->second;
      free_.erase(it);
      return p;
    }
    void* p = nullptr;
    ck(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc");
    return p;
  }
  void give(void* p, size_t bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    free_.emplace(bytes, p);
  }

 private:
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  explicit DevBuf(size_t n) : p(Pool::get().take(n)), bytes(n) {}
  ~DevBuf() { Pool::get().give(p, bytes); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  float* f() const { return static_cast<float*>(p); }
};
using Buf = std::shared_ptr<DevBuf>;

inline Buf alloc(size_t floats) { return std::make_shared<DevBuf>(sizeof(float) * floats); }

inline Buf upload(const Tensor& t) {
  auto buf = alloc((size_t)t.size());
  if constexpr (std::is_same_v<Real, float>) {
    ck(cudaMemcpy(buf->p, t.data().data(), sizeof(float) * (size_t)t.size(), cudaMemcpyHostToDevice), "H2D");
  } else {
    std::vector<float> tmp(t.data().begin(), t.data().end());  // Real -> float
    ck(cudaMemcpy(buf->p, tmp.data(), sizeof(float) * tmp.size(), cudaMemcpyHostToDevice), "H2D");
  }
  return buf;
}

inline Tensor download(const DevBuf& d, Shape shape) {
  Tensor t = Tensor::zeros(std::move(shape));
  if constexpr (std::is_same_v<Real, float>) {
    ck(cudaMemcpy(t.data().data(), d.p, sizeof(float) * (size_t)t.size(), cudaMemcpyDeviceToHost), "D2H");
  } else {
    std::vector<float> tmp((size_t)t.size());
    ck(cudaMemcpy(tmp.data(), d.p, sizeof(float) * tmp.size(), cudaMemcpyDeviceToHost), "D2H");
    auto dst = t.data();
    for (size_t i = 0; i < tmp.size(); ++i) dst[i] = static_cast<Real>(tmp[i]);
  }
  return t;
}

// SEQLOOM_CUDA_PRECISION=bf16 selects SL_PREC_BF16; default SL_PREC_FP32 (the reference's precision)
inline int precision_from_env() {
  const char* p = std::getenv("SEQLOOM_CUDA_PRECISION");
  return (p && std::strcmp(p, "bf16") == 0) ? SL_PREC_BF16 : SL_PREC_FP32;
}

}  // namespace cuda_dropin
}  // namespace seqloom
