// C-ABI implementation (include/seqloom_cuda.h).  Orchestrates, per layer:
//   fwd:  K1  XW = X . W + b for ALL T at once (one GEMM per direction)
//         K2  persistent recurrence, both directions in one launch
//   bwd:  K3  persistent BPTT, both directions in one launch -> DZ [B*T, 4H]
//         K4  dX = sum_d DZ_d . W_d^T,  dW_d = X^T . DZ_d,  dR_d = Hprev_d^T . DZ_d
//             (db is reduced inside K3)
// replacing the reference's per-step Eigen GEMMs and per-step GradBuffer
// temporaries (tape.cpp:1103-1104, 1174-1215, 76-89).
#include <algorithm>
#include <string>
#include <vector>

#include "cell.h"
#include "gemm.h"
#include "profile.h"
#include "recurrence.h"

namespace sl {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

namespace {

constexpr size_t kAlign = 256;

// Bump allocator over a caller-owned buffer.
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* p) : base(static_cast<char*>(p)) {}
  template <typename T>
  T* take(size_t count) {
    off = round_up(off, kAlign);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

struct Dims {
  int B, T, D, H, nd;
  int64_t BT() const { return (int64_t)B * T; }
};

void validate(const sl_lstm_layer* L) {
  SL_REQUIRE(L != nullptr, SL_ERR_INVALID_ARGUMENT, "sl_lstm_layer: null descriptor");
  SL_REQUIRE(L->num_dirs == 1 || L->num_dirs == 2, SL_ERR_INVALID_ARGUMENT,
             "lstm_sequence: num_dirs must be 1 or 2");
  SL_REQUIRE(L->num_dirs == 2 || L->direction == 1 || L->direction == -1,
             SL_ERR_INVALID_ARGUMENT, "lstm_sequence: direction must be +1 or -1");
  SL_REQUIRE(L->batch > 0 && L->time > 0 && L->input_dim > 0 && L->hidden > 0, SL_ERR_SHAPE,
             "lstm_sequence: input needs Batch and Time axes, got B=" +
                 std::to_string(L->batch) + " T=" + std::to_string(L->time) +
                 " D=" + std::to_string(L->input_dim) + " H=" + std::to_string(L->hidden));
  SL_REQUIRE(L->precision == SL_PREC_FP32, SL_ERR_UNSUPPORTED,
             "precision " + std::to_string(L->precision) + " not supported by this build");
  SL_REQUIRE(L->flags == 0, SL_ERR_INVALID_ARGUMENT, "sl_lstm_layer.flags must be 0");
}

Dims dims(const sl_lstm_layer* L) {
  return Dims{L->batch, L->time, L->input_dim, L->hidden, L->num_dirs};
}

struct ReserveView {
  float* gates[2] = {nullptr, nullptr};
  float* cprev[2] = {nullptr, nullptr};
  float* hprev[2] = {nullptr, nullptr};
};

ReserveView carve_reserve(const Dims& d, void* p, size_t* bytes) {
  Carve c(p);
  ReserveView r;
  for (int k = 0; k < d.nd; ++k) {
    r.gates[k] = c.take<float>((size_t)d.BT() * 4 * d.H);
    r.cprev[k] = c.take<float>((size_t)d.BT() * d.H);
    r.hprev[k] = c.take<float>((size_t)d.BT() * d.H);
  }
  *bytes = c.off;
  return r;
}

struct FwdWork {
  float* xw[2] = {nullptr, nullptr};
  float* hbuf[2] = {nullptr, nullptr};
  float* cbuf[2] = {nullptr, nullptr};
  unsigned* bar = nullptr;
};

FwdWork carve_fwd(const Dims& d, void* p, size_t* bytes) {
  Carve c(p);
  FwdWork w;
  w.bar = c.take<unsigned>(64);
  for (int k = 0; k < d.nd; ++k) {
    w.xw[k] = c.take<float>((size_t)d.BT() * 4 * d.H);
    w.hbuf[k] = c.take<float>((size_t)2 * d.B * d.H);
    w.cbuf[k] = c.take<float>((size_t)d.B * d.H);
  }
  *bytes = c.off;
  return w;
}

struct BwdWork {
  float* dz[2] = {nullptr, nullptr};
  float* dzbuf[2] = {nullptr, nullptr};
  float* gcbuf[2] = {nullptr, nullptr};
  unsigned* bar = nullptr;
};

BwdWork carve_bwd(const Dims& d, void* p, size_t* bytes) {
  Carve c(p);
  BwdWork w;
  w.bar = c.take<unsigned>(64);
  for (int k = 0; k < d.nd; ++k) {
    w.dz[k] = c.take<float>((size_t)d.BT() * 4 * d.H);
    w.dzbuf[k] = c.take<float>((size_t)2 * d.B * 4 * d.H);
    w.gcbuf[k] = c.take<float>((size_t)d.B * d.H);
  }
  *bytes = c.off;
  return w;
}

int dir_sign(const sl_lstm_layer* L, int k) {
  return L->num_dirs == 2 ? (k == 0 ? 1 : -1) : L->direction;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    set_error("");
    return SL_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return SL_ERR_CUDA;
  }
}

}  // namespace
}  // namespace sl

using namespace sl;

extern "C" {

int sl_version(void) { return 100; }

const char* sl_last_error(void) { return g_last_error.c_str(); }

int sl_lstm_layer_check(const sl_lstm_layer* L) {
  return guarded([&] { validate(L); });
}

size_t sl_lstm_reserve_size(const sl_lstm_layer* L) {
  size_t bytes = 0;
  if (guarded([&] {
        validate(L);
        carve_reserve(dims(L), nullptr, &bytes);
      }) != SL_OK)
    return 0;
  return bytes;
}

size_t sl_lstm_workspace_size(const sl_lstm_layer* L) {
  size_t f = 0, b = 0;
  if (guarded([&] {
        validate(L);
        carve_fwd(dims(L), nullptr, &f);
        carve_bwd(dims(L), nullptr, &b);
      }) != SL_OK)
    return 0;
  return std::max(f, b);
}

int sl_lstm_layer_fwd(const sl_lstm_layer* L, const float* x, const int32_t* seq_lens,
                      const float* const* W, const float* const* R, const float* const* b,
                      float* y, float* h_last, float* c_last, void* reserve,
                      size_t reserve_bytes, void* workspace, size_t workspace_bytes,
                      sl_stream_t stream_) {
  return guarded([&] {
    validate(L);
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    const Dims d = dims(L);
    SL_REQUIRE(x && seq_lens && W && R && b && y, SL_ERR_INVALID_ARGUMENT,
               "sl_lstm_layer_fwd: null pointer argument");
    size_t need_w = 0, need_r = 0;
    FwdWork w = carve_fwd(d, workspace, &need_w);
    SL_REQUIRE(workspace && workspace_bytes >= need_w, SL_ERR_WORKSPACE,
               "sl_lstm_layer_fwd: workspace too small");
    ReserveView rv;
    if (reserve) {
      rv = carve_reserve(d, reserve, &need_r);
      SL_REQUIRE(reserve_bytes >= need_r, SL_ERR_WORKSPACE, "sl_lstm_layer_fwd: reserve too small");
    }
    SL_CUDA_TRY(cudaMemsetAsync(w.bar, 0, 64 * sizeof(unsigned), stream));
    RecFwdArgs a{};
    a.B = d.B;
    a.T = d.T;
    a.H = d.H;
    a.nd = d.nd;
    rec_partition(d.H, d.nd, &a.U, &a.ctas_per_dir);
    a.lens = seq_lens;
    a.xw_ld = 4 * d.H;
    a.y = y;
    a.y_ld = (int64_t)d.nd * d.H;
    a.h_last = h_last;
    a.c_last = c_last;
    a.bar = w.bar;
    for (int k = 0; k < d.nd; ++k) {
      SL_REQUIRE(W[k] && R[k] && b[k], SL_ERR_INVALID_ARGUMENT,
                 "sl_lstm_layer_fwd: null weight pointer");
      {  // K1: XW = X W + b over all B*T rows (replaces tape.cpp:1103-1109 per step).
        Phase ph(stream, "k1_xw_gemm", 2.0 * d.BT() * d.D * 4.0 * d.H);
        gemm_f32(false, false, (int)d.BT(), 4 * d.H, d.D, 1.f, x, d.D, W[k], 4 * d.H, 0.f,
                 w.xw[k], 4 * d.H, b[k], stream);
      }
      SL_CUDA_TRY(cudaMemsetAsync(w.hbuf[k], 0, sizeof(float) * d.B * d.H, stream));
      SL_CUDA_TRY(cudaMemsetAsync(w.cbuf[k], 0, sizeof(float) * d.B * d.H, stream));
      a.dirsign[k] = dir_sign(L, k);
      a.xw[k] = w.xw[k];
      a.R[k] = R[k];
      a.hbuf[k] = w.hbuf[k];
      a.cbuf[k] = w.cbuf[k];
      a.gates[k] = rv.gates[k];
      a.cprev[k] = rv.cprev[k];
      a.hprev[k] = rv.hprev[k];
    }
    {
      Phase ph(stream, "k2_rec_fwd", 2.0 * d.BT() * d.H * 4.0 * d.H * d.nd);
      rec_fwd_f32(a, stream);
    }
  });
}

int sl_lstm_layer_bwd(const sl_lstm_layer* L, const float* x, const int32_t* seq_lens,
                      const float* const* W, const float* const* R, const float* dy,
                      const float* dh_last, const float* dc_last, float* dx, float* const* dW,
                      float* const* dR, float* const* db, int accumulate, const void* reserve,
                      size_t reserve_bytes, void* workspace, size_t workspace_bytes,
                      sl_stream_t stream_) {
  return guarded([&] {
    validate(L);
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    const Dims d = dims(L);
    SL_REQUIRE(x && seq_lens && W && R && dy && reserve, SL_ERR_INVALID_ARGUMENT,
               "sl_lstm_layer_bwd: null pointer argument");
    size_t need_w = 0, need_r = 0;
    BwdWork w = carve_bwd(d, workspace, &need_w);
    SL_REQUIRE(workspace && workspace_bytes >= need_w, SL_ERR_WORKSPACE,
               "sl_lstm_layer_bwd: workspace too small");
    ReserveView rv = carve_reserve(d, const_cast<void*>(reserve), &need_r);
    SL_REQUIRE(reserve_bytes >= need_r, SL_ERR_WORKSPACE, "sl_lstm_layer_bwd: reserve too small");
    SL_CUDA_TRY(cudaMemsetAsync(w.bar, 0, 64 * sizeof(unsigned), stream));
    RecBwdArgs a{};
    a.B = d.B;
    a.T = d.T;
    a.H = d.H;
    a.nd = d.nd;
    rec_partition(d.H, d.nd, &a.U, &a.ctas_per_dir);
    a.lens = seq_lens;
    a.dy = dy;
    a.dy_ld = (int64_t)d.nd * d.H;
    a.dh_last = dh_last;
    a.dc_last = dc_last;
    a.accumulate = accumulate;
    a.bar = w.bar;
    for (int k = 0; k < d.nd; ++k) {
      a.dirsign[k] = dir_sign(L, k);
      a.R[k] = R[k];
      a.gates[k] = rv.gates[k];
      a.cprev[k] = rv.cprev[k];
      a.dz[k] = w.dz[k];
      a.dzbuf[k] = w.dzbuf[k];
      a.gcbuf[k] = w.gcbuf[k];
      a.db[k] = db ? db[k] : nullptr;
      SL_CUDA_TRY(cudaMemsetAsync(w.dzbuf[k], 0, sizeof(float) * 2 * d.B * 4 * d.H, stream));
      SL_CUDA_TRY(cudaMemsetAsync(w.gcbuf[k], 0, sizeof(float) * d.B * d.H, stream));
    }
    {
      Phase ph(stream, "k3_rec_bwd", 2.0 * d.BT() * d.H * 4.0 * d.H * d.nd);
      rec_bwd_f32(a, stream);
    }
    const float beta = accumulate ? 1.f : 0.f;
    const int M = (int)d.BT(), G = 4 * d.H;
    for (int k = 0; k < d.nd; ++k) {
      // K4: hoisted weight / input gradients over all B*T rows (tape.cpp:1174-1205).
      const double f = 2.0 * M * G * (double)d.D;
      if (dx) {
        Phase ph(stream, "k4_dx_gemm", f);
        gemm_f32(false, true, M, d.D, G, 1.f, w.dz[k], G, W[k], G, k == 0 ? beta : 1.f, dx, d.D,
                 nullptr, stream);
      }
      if (dW && dW[k]) {
        Phase ph(stream, "k4_dw_gemm", f);
        gemm_f32(true, false, d.D, G, M, 1.f, x, d.D, w.dz[k], G, beta, dW[k], G, nullptr, stream);
      }
      if (dR && dR[k]) {
        Phase ph(stream, "k4_dr_gemm", 2.0 * M * G * (double)d.H);
        gemm_f32(true, false, d.H, G, M, 1.f, rv.hprev[k], d.H, w.dz[k], G, beta, dR[k], G,
                 nullptr, stream);
      }
    }
  });
}

int sl_lstm_cell_fwd(int32_t B, int32_t D, int32_t H, int32_t precision, const float* x,
                     const float* h0, const float* c0, const float* W, const float* R,
                     const float* b, float* h, float* c, float* saved, sl_stream_t stream) {
  return guarded([&] {
    SL_REQUIRE(B > 0 && D > 0 && H > 0, SL_ERR_SHAPE, "lstm_step: inconsistent shapes");
    SL_REQUIRE(precision == SL_PREC_FP32, SL_ERR_UNSUPPORTED, "precision not supported");
    SL_REQUIRE(x && h0 && c0 && W && R && b && h && c, SL_ERR_INVALID_ARGUMENT,
               "sl_lstm_cell_fwd: null pointer argument");
    Phase ph(reinterpret_cast<cudaStream_t>(stream), "k5_cell_fwd", 2.0 * B * (D + H) * 4.0 * H);
    cell_fwd(B, D, H, x, h0, c0, W, R, b, h, c, saved, reinterpret_cast<cudaStream_t>(stream));
  });
}

int sl_lstm_cell_bwd(int32_t B, int32_t D, int32_t H, int32_t precision, const float* x,
                     const float* h0, const float* c0, const float* W, const float* R,
                     const float* saved, const float* gh, const float* gc, float* dx, float* dh0,
                     float* dc0, float* dW, float* dR, float* db, int accumulate,
                     sl_stream_t stream) {
  return guarded([&] {
    SL_REQUIRE(B > 0 && D > 0 && H > 0, SL_ERR_SHAPE, "lstm_step: inconsistent shapes");
    SL_REQUIRE(precision == SL_PREC_FP32, SL_ERR_UNSUPPORTED, "precision not supported");
    SL_REQUIRE(x && h0 && c0 && W && R && saved, SL_ERR_INVALID_ARGUMENT,
               "sl_lstm_cell_bwd: null pointer argument");
    Phase ph(reinterpret_cast<cudaStream_t>(stream), "k5_cell_bwd", 4.0 * B * (D + H) * 4.0 * H);
    cell_bwd(B, D, H, x, h0, c0, W, R, saved, gh, gc, dx, dh0, dc0, dW, dR, db, accumulate,
             reinterpret_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
