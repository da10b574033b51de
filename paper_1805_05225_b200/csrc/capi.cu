// C-ABI implementation (include/seqloom_cuda.h).  Orchestrates, per layer:
//   fwd:  K1  XW = X . W + b for ALL T at once (one GEMM per direction)
//         K2  persistent recurrence, both directions in one launch
//   bwd:  K3  persistent BPTT, both directions in one launch -> DZ [B*T, 4H]
//         K4  dX = sum_d DZ_d . W_d^T,  dW_d = X^T . DZ_d,  dR_d = Hprev_d^T . DZ_d
//             (db is reduced inside K3)
// replacing the reference's per-step Eigen GEMMs and per-step GradBuffer
// temporaries (tape.cpp:1103-1104, 1174-1215, 76-89).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "adam.h"
#include "attention.h"
#include "embedding.h"
#include "cell.h"
#include "decoder.h"
#include "dropout.h"
#include "convert.h"
#include "gemm.h"
#include "profile.h"
#include "rec_tc.h"
#include "softmax_ce.h"
#include "recurrence.h"

namespace sl {

static thread_local std::string g_last_error;
static unsigned long long* g_rec_trace = nullptr;  // debug: sl_debug_set_trace
static int g_rec_trace_cta = 0;
static int g_rec_debug_flags = 0;  // experiments only (sl_debug_set_flags)
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
  int flags = 0;
  int64_t BT() const { return (int64_t)B * T; }
  bool x_bf16() const { return flags & SL_LAYER_X_BF16; }
  bool y_bf16() const { return flags & SL_LAYER_Y_BF16; }
  bool x_x3() const { return flags & SL_LAYER_X_X3; }
  bool y_x3() const { return flags & SL_LAYER_Y_X3; }
};

struct Dims;
Dims dims(const sl_lstm_layer* L);
bool use_x3(const Dims& d, int prec);

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
  SL_REQUIRE(L->precision == SL_PREC_FP32 || L->precision == SL_PREC_BF16, SL_ERR_UNSUPPORTED,
             "precision " + std::to_string(L->precision) + " not supported by this build");
  SL_REQUIRE((L->flags & ~(SL_LAYER_X_BF16 | SL_LAYER_Y_BF16 | SL_LAYER_X_X3 | SL_LAYER_Y_X3)) == 0,
             SL_ERR_INVALID_ARGUMENT, "sl_lstm_layer.flags: unknown bits " + std::to_string(L->flags));
  SL_REQUIRE((L->flags & (SL_LAYER_X_BF16 | SL_LAYER_Y_BF16)) == 0 || L->precision == SL_PREC_BF16,
             SL_ERR_UNSUPPORTED, "sl_lstm_layer.flags: bf16 activations need precision SL_PREC_BF16");
  SL_REQUIRE((L->flags & (SL_LAYER_X_X3 | SL_LAYER_Y_X3)) == 0 ||
                 (L->precision == SL_PREC_FP32 && use_x3(dims(L), L->precision)),
             SL_ERR_UNSUPPORTED,
             "sl_lstm_layer.flags: split-image (x3) activations need precision SL_PREC_FP32 on the "
             "tensor-core path");
}

Dims dims(const sl_lstm_layer* L) {
  return Dims{L->batch, L->time, L->input_dim, L->hidden, L->num_dirs, L->flags};
}

int sm_count();

// SL_PREC_FP32 runs on the tensor cores as split-bf16 ("x3": every product
// A B = A_hi B_hi + A_lo B_hi + A_hi B_lo, fp32 accumulation) whenever the x3
// recurrences support the hidden size; the SIMT fp32 kernels cover the rest.
bool use_x3(const Dims& d, int prec) {
  return prec == SL_PREC_FP32 && tc_rec_fwd_x3_shape(d.H, sm_count()).C > 0 &&
         tc_rec_bwd_x3_shape(d.H, sm_count()).C > 0;
}
int64_t g4(const Dims& d) { return 4 * (int64_t)d.H; }
// row stride of the DZ image: the K4 weight-gradient GEMMs read one direction's
// column slice as 64-wide MN-major blocks, which may run up to 64 columns past it
int64_t dzi_ld(const Dims& d) { return x3_img_ld(d.nd * 4 * d.H) + 64; }

size_t x3_gemm_ws(const Dims& d, bool bwd) {
  const int M = (int)d.BT(), G = 4 * d.H, Gc = d.nd * G;
  if (!bwd) return gemm_f32x3_workspace_bytes(false, false, M, Gc, d.D, false);
  return std::max({gemm_f32x3_workspace_bytes(false, true, M, d.D, Gc, false),   // dX = DZ Wcat^T
                   gemm_f32x3_workspace_bytes(true, false, d.D, G, M, true),     // [dW; db] = [X | 1]^T DZ_d
                   gemm_f32x3_workspace_bytes(true, false, d.H, G, M, false)});  // dR = Hprev^T DZ_d
}

struct ReserveView {
  float* gates[2] = {nullptr, nullptr};
  float* cprev[2] = {nullptr, nullptr};
  float* hprev[2] = {nullptr, nullptr};  // fp32 SIMT path: h_{s-1} [B*T, H]
  __nv_bfloat16* hprevi[2] = {nullptr, nullptr};  // x3 path: h_{s-1} as its split image [2][B*T][x3_img_ld(H)]
  __nv_bfloat16* xb = nullptr;    // bf16 path: x in bf16 [B*T, Dp]
  __nv_bfloat16* wcat = nullptr;  // bf16 path: [W_fw | W_bw] bf16 [D, nd*G4p]
  __nv_bfloat16* hprevb[2] = {nullptr, nullptr};  // bf16 path: h_{s-1} [B*T, Hp]
  __nv_bfloat16* gatesb[2] = {nullptr, nullptr};  // bf16 path: saved (i,f,g,o), step-major (rec_tc.h)
  __nv_bfloat16* cprevb[2] = {nullptr, nullptr};  // bf16 path: saved c_{s-1}, step-major
  __nv_bfloat16* rt[2] = {nullptr, nullptr};      // bf16 path: packed R^T slices
  __nv_bfloat16* wimg = nullptr;  // x3 path: split image of [W_fw | W_bw] [D, nd*4H] (K1 and K4-dX)
  __nv_bfloat16* ximg = nullptr;  // x3 path: split image of [X | 1] [B*T, D + 1] (K1 and K4-dW)
};

// x3 operand images kept from the forward for the backward (gemm.h x3_split_into)
int64_t wimg_ld(const Dims& d) { return x3_img_ld(d.nd * 4 * d.H); }
int64_t ximg_ld(const Dims& d) { return x3_img_ld(d.D + 1); }
size_t wimg_elems(const Dims& d) { return (size_t)2 * d.D * wimg_ld(d); }
size_t ximg_elems(const Dims& d) { return (size_t)2 * d.BT() * ximg_ld(d); }

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 148;  // sizing only (no device yet): B200
  }
  return n;
}

// Padded extents of the bf16 path (TMA needs 16 B aligned rows).
struct Pad {
  int64_t Dp, Hp, G4p, Gc;  // Gc = nd * G4p (concatenated gate columns)
};
Pad pads(const Dims& d) {
  Pad p;
  // 64-element multiples: the GEMM reads MN-major operands in whole 64-wide
  // blocks (one 3-D TMA box per stage), and every row stays 16 B aligned
  p.Dp = round_up(d.D + 1, 64);  // + a ones column (db from the dW GEMM)
  p.Hp = round_up(d.H, 64);
  p.G4p = round_up(4 * (int64_t)d.H, 64);
  p.Gc = d.nd * p.G4p;
  return p;
}

ReserveView carve_reserve(const Dims& d, int prec, void* p, size_t* bytes) {
  Carve c(p);
  ReserveView r;
  for (int k = 0; k < d.nd; ++k) {
    if (prec == SL_PREC_BF16) {
      r.gatesb[k] = c.take<__nv_bfloat16>((size_t)d.BT() * 4 * save_hq(d.H));  // step-major, rec_tc.h
      r.cprevb[k] = c.take<__nv_bfloat16>((size_t)d.BT() * save_hq(d.H));
    } else if (use_x3(d, prec)) {  // x3: the same step-major saves in fp32
      r.gates[k] = c.take<float>((size_t)d.BT() * 4 * save_hq(d.H));
      r.cprev[k] = c.take<float>((size_t)d.BT() * save_hq(d.H));
      r.hprevi[k] = c.take<__nv_bfloat16>(x3_img_elems((int)d.BT(), d.H));
    } else {
      r.gates[k] = c.take<float>((size_t)d.BT() * 4 * d.H);
      r.cprev[k] = c.take<float>((size_t)d.BT() * d.H);
      r.hprev[k] = c.take<float>((size_t)d.BT() * d.H);
    }
  }
  if (use_x3(d, prec)) {
    r.wimg = c.take<__nv_bfloat16>(wimg_elems(d));
    if (!d.x_x3()) r.ximg = c.take<__nv_bfloat16>(ximg_elems(d));  // else the caller's x image
  }
  if (prec == SL_PREC_BF16) {
    const Pad pd = pads(d);
    const TcFwdShape sh = tc_rec_fwd_shape(d.H, d.nd, sm_count());
    SL_REQUIRE(sh.C > 0, SL_ERR_UNSUPPORTED, "bf16 recurrence: hidden size too large for one launch");
    if (!d.x_bf16()) r.xb = c.take<__nv_bfloat16>((size_t)d.BT() * pd.Dp);  // else the caller's x
    r.wcat = c.take<__nv_bfloat16>((size_t)d.D * pd.Gc);
    for (int k = 0; k < d.nd; ++k) {
      r.hprevb[k] = c.take<__nv_bfloat16>((size_t)d.BT() * pd.Hp);
      r.rt[k] = c.take<__nv_bfloat16>(tc_rec_pack_elems(sh));
    }
  }
  *bytes = c.off;
  return r;
}

struct FwdWork {
  float* xw[2] = {nullptr, nullptr};
  __nv_bfloat16* xwb[2] = {nullptr, nullptr};  // bf16 path: K1 output in bf16
  int64_t xw_ld = 0;
  float* hbuf[2] = {nullptr, nullptr};
  float* cbuf[2] = {nullptr, nullptr};
  float* bcat = nullptr;  // bf16 path: concatenated bias [nd*G4p]
  __nv_bfloat16* xb = nullptr;    // bf16 inference (no reserve)
  __nv_bfloat16* wcat = nullptr;
  __nv_bfloat16* rt[2] = {nullptr, nullptr};
  __nv_bfloat16* hbufb[2] = {nullptr, nullptr};  // bf16 path: h ring [2][B][Kp]
  __nv_bfloat16* hbuflo[2] = {nullptr, nullptr};  // x3 path: lo halves of h, same ring layout
  __nv_bfloat16* rtx3[2] = {nullptr, nullptr};    // x3 path: packed R^T hi + lo
  __nv_bfloat16* wimg = nullptr;                  // x3 path without a reserve: the K1 operand images
  __nv_bfloat16* ximg = nullptr;
  void* gws = nullptr;                            // x3 path: split-bf16 GEMM scratch
  unsigned* bar = nullptr;
};

FwdWork carve_fwd(const Dims& d, int prec, void* p, size_t* bytes) {
  Carve c(p);
  FwdWork w;
  w.bar = c.take<unsigned>(rec_bar_count(d.B));
  if (prec == SL_PREC_BF16) {
    const Pad pd = pads(d);
    __nv_bfloat16* xw = c.take<__nv_bfloat16>((size_t)d.BT() * pd.Gc);
    w.xw_ld = pd.Gc;
    for (int k = 0; k < d.nd; ++k) w.xwb[k] = xw ? xw + k * pd.G4p : nullptr;
    w.bcat = c.take<float>((size_t)pd.Gc);
    if (!d.x_bf16()) w.xb = c.take<__nv_bfloat16>((size_t)d.BT() * pd.Dp);
    w.wcat = c.take<__nv_bfloat16>((size_t)d.D * pd.Gc);
    const TcFwdShape sh = tc_rec_fwd_shape(d.H, d.nd, sm_count());
    SL_REQUIRE(sh.C > 0, SL_ERR_UNSUPPORTED, "bf16 recurrence: hidden size too large for one launch");
    for (int k = 0; k < d.nd; ++k) {
      w.rt[k] = c.take<__nv_bfloat16>(tc_rec_pack_elems(sh));
      w.hbufb[k] = c.take<__nv_bfloat16>(tc_rec_hbuf_elems(d.B, sh));
    }
  } else if (use_x3(d, prec)) {
    const TcFwdShape sh = tc_rec_fwd_x3_shape(d.H, sm_count(), d.nd);
    w.xw_ld = d.nd * g4(d);
    float* xw = c.take<float>((size_t)d.BT() * w.xw_ld);
    for (int k = 0; k < d.nd; ++k) w.xw[k] = xw ? xw + k * g4(d) : nullptr;
    w.bcat = c.take<float>((size_t)w.xw_ld);
    w.wimg = c.take<__nv_bfloat16>(wimg_elems(d));
    if (!d.x_x3()) w.ximg = c.take<__nv_bfloat16>(ximg_elems(d));
    w.gws = c.take<char>(x3_gemm_ws(d, false));
    for (int k = 0; k < d.nd; ++k) {
      w.rtx3[k] = c.take<__nv_bfloat16>(tc_rec_x3_pack_elems(sh));
      w.hbufb[k] = c.take<__nv_bfloat16>(tc_rec_hbuf_elems(d.B, sh));
      w.hbuflo[k] = c.take<__nv_bfloat16>(tc_rec_hbuf_elems(d.B, sh));
    }
  } else {
    w.xw_ld = 4 * d.H;
    for (int k = 0; k < d.nd; ++k) {
      w.xw[k] = c.take<float>((size_t)d.BT() * 4 * d.H);
      w.hbuf[k] = c.take<float>((size_t)2 * d.B * d.H);
      w.cbuf[k] = c.take<float>((size_t)d.B * d.H);
    }
  }
  *bytes = c.off;
  return w;
}

struct BwdWork {
  float* dz[2] = {nullptr, nullptr};      // fp32 path
  float* dzbuf[2] = {nullptr, nullptr};   // fp32 path
  float* gcbuf[2] = {nullptr, nullptr};   // fp32 path
  __nv_bfloat16* dzb = nullptr;           // bf16 path: DZ of both directions [B*T, nd*G4p]
  __nv_bfloat16* dzring[2] = {nullptr, nullptr};  // bf16 path: DZ ring (rec_tc.h dz_ring_off)
  __nv_bfloat16* rb[2] = {nullptr, nullptr};      // bf16 path: packed R row slices
  __nv_bfloat16* dzringlo[2] = {nullptr, nullptr};  // x3 path: lo halves of DZ, same ring layout
  __nv_bfloat16* dzi = nullptr;  // x3 path: DZ of both directions as its split image (hi, lo) [B*T, dzi_ld]
  void* gws = nullptr;                            // x3 path: split-bf16 GEMM scratch
  unsigned* bar = nullptr;
};

BwdWork carve_bwd(const Dims& d, int prec, void* p, size_t* bytes) {
  Carve c(p);
  BwdWork w;
  w.bar = c.take<unsigned>(rec_bar_count(d.B));
  if (prec == SL_PREC_BF16) {
    const Pad pd = pads(d);
    const TcBwdShape sh = tc_rec_bwd_shape(d.H, d.nd, sm_count());
    SL_REQUIRE(sh.C > 0, SL_ERR_UNSUPPORTED, "bf16 recurrence: hidden size too large for one launch");
    w.dzb = c.take<__nv_bfloat16>((size_t)d.BT() * pd.Gc);
    for (int k = 0; k < d.nd; ++k) {
      w.dzring[k] = c.take<__nv_bfloat16>((size_t)2 * dz_ring_bp(d.B) * sh.Kz);
      w.rb[k] = c.take<__nv_bfloat16>(tc_rec_bwd_pack_elems(sh));
    }
  } else if (use_x3(d, prec)) {
    const TcBwdShape sh = tc_rec_bwd_x3_shape(d.H, sm_count(), d.nd);
    w.dzi = c.take<__nv_bfloat16>((size_t)2 * d.BT() * dzi_ld(d));
    w.gws = c.take<char>(x3_gemm_ws(d, true));
    for (int k = 0; k < d.nd; ++k) {
      w.dzring[k] = c.take<__nv_bfloat16>((size_t)2 * dz_ring_bp(d.B) * sh.Kz);
      w.dzringlo[k] = c.take<__nv_bfloat16>((size_t)2 * dz_ring_bp(d.B) * sh.Kz);
      w.rb[k] = c.take<__nv_bfloat16>(tc_rec_bwd_x3_pack_elems(sh));
    }
  } else {
    for (int k = 0; k < d.nd; ++k) {
      w.dz[k] = c.take<float>((size_t)d.BT() * 4 * d.H);
      w.dzbuf[k] = c.take<float>((size_t)2 * d.B * 4 * d.H);
      w.gcbuf[k] = c.take<float>((size_t)d.B * d.H);
    }
  }
  *bytes = c.off;
  return w;
}

int dir_sign(const sl_lstm_layer* L, int k) {
  return L->num_dirs == 2 ? (k == 0 ? 1 : -1) : L->direction;
}


// out[c] = beta * out[c] + sum_r x[r * ld + c] (ascending r)
__global__ void colsum_img_kernel(int rows, int cols, const __nv_bfloat16* __restrict__ hi, int64_t ld, int64_t lo,
                                  float beta, float* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int r = 0; r < rows; ++r) {
    const int64_t i = (int64_t)r * ld + c;
    s += __bfloat162float(hi[i]) + __bfloat162float(hi[lo + i]);
  }
  out[c] = beta != 0.f ? beta * out[c] + s : s;
}

// ---- SL_PREC_FP32 on the tensor cores (split-bf16 "x3") ------------------------
// K1: XW = X [W_fw | W_bw] + [b_fw | b_bw] as ONE fp32-class GEMM (fp32 out);
// K2: the x3 pair recurrence, one launch per direction.
void fwd_x3(const sl_lstm_layer* L, const Dims& d, const float* x, const int32_t* lens, const float* const* W,
            const float* const* R, const float* const* b, float* y, float* h_last, float* c_last,
            const ReserveView& rv, const FwdWork& w, cudaStream_t st) {
  const int64_t G = g4(d), Gc = d.nd * G;
  // the split images of [W_fw | W_bw] (each direction straight into its column block)
  // and of [X | 1]; with a reserve they stay there for the backward's dX and dW GEMMs
  // (SL_LAYER_X_X3: x already is that image, written by the previous layer's K2)
  __nv_bfloat16* wi = rv.wimg ? rv.wimg : w.wimg;
  __nv_bfloat16* xi = d.x_x3() ? reinterpret_cast<__nv_bfloat16*>(const_cast<float*>(x))
                               : (rv.ximg ? rv.ximg : w.ximg);
  const int64_t wl = wimg_ld(d), xl = ximg_ld(d), M = d.BT();
  for (int k = 0; k < d.nd; ++k) {
    x3_split_into(W[k], G, d.D, (int)G, -1, wi + k * G, wl, G, (int64_t)d.D * wl, st);
    SL_CUDA_TRY(cudaMemcpyAsync(w.bcat + k * G, b[k], G * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  if (!d.x_x3()) x3_split_into(x, d.D, (int)M, d.D, d.D, xi, xl, xl, M * xl, st);
  // SL_LAYER_Y_X3: K2 writes y as the next layer's x image (its ones column set here)
  __nv_bfloat16* yimg = d.y_x3() ? reinterpret_cast<__nv_bfloat16*>(y) : nullptr;
  const int64_t yl = x3_img_ld(d.nd * d.H + 1);
  if (yimg) fill_col_bf16(d.BT(), d.nd * d.H, yimg, yl, 1.f, st);
  {
    Phase ph(st, "k1_xw_gemm", 2.0 * d.BT() * d.D * (double)Gc);
    gemm_f32x3_ex(false, false, (int)M, (int)Gc, d.D, nullptr, 0, xi, nullptr, 0, wi, 0.f, w.xw[0], Gc, w.bcat,
                  nullptr, 0, w.gws, st, xl, M * xl, wl, (int64_t)d.D * wl);
  }
  const TcFwdShape sh = tc_rec_fwd_x3_shape(d.H, sm_count(), d.nd);
  const int per_launch = sh.pair == 2 ? d.nd : 1;  // both directions at once, or one per launch
  SL_CUDA_TRY(cudaMemsetAsync(w.bar, 0, rec_bar_count(d.B) * sizeof(unsigned), st));
  for (int k0 = 0; k0 < d.nd; k0 += per_launch) {
    TcRecFwdArgs a{};
    a.B = d.B;
    a.T = d.T;
    a.H = d.H;
    a.nd = per_launch;
    a.dir0 = sh.pair == 2 ? 0 : k0;
    a.lens = lens;
    a.xw_ld = Gc;
    a.y = yimg ? nullptr : y;
    a.y_ld = (int64_t)d.nd * d.H;
    a.yimg = yimg;
    a.yimg_ld = yl;
    a.yimg_lo = M * yl;
    a.h_last = h_last;
    a.c_last = c_last;
    a.hprev_ld = x3_img_ld(d.H);  // h_{s-1} image rows
    a.hprevi_lo = d.BT() * x3_img_ld(d.H);
    a.bar = w.bar;
    a.trace = g_rec_trace;  // (experiments builds stamp it; null otherwise)
    a.trace_cta = g_rec_trace_cta;
    const __nv_bfloat16* rt[2] = {nullptr, nullptr};
    for (int j = 0; j < per_launch; ++j) {
      const int k = k0 + j;
      a.dirsign[j] = dir_sign(L, k);
      a.xwf[j] = w.xw[k];
      a.gatesf[j] = rv.gates[k];
      a.cprevf[j] = rv.cprev[k];
      a.hprevi[j] = rv.hprevi[k];
      a.hbuf[j] = w.hbufb[k];
      a.hbuf_lo[j] = w.hbuflo[k];
      tc_rec_x3_pack(R[k], d.H, sh, w.rtx3[k], st);
      rt[j] = w.rtx3[k];
      SL_CUDA_TRY(cudaMemsetAsync(w.hbufb[k], 0, sizeof(__nv_bfloat16) * tc_rec_hbuf_elems(d.B, sh), st));
      SL_CUDA_TRY(cudaMemsetAsync(w.hbuflo[k], 0, sizeof(__nv_bfloat16) * tc_rec_hbuf_elems(d.B, sh), st));
    }
    if (k0 > 0) SL_CUDA_TRY(cudaMemsetAsync(w.bar, 0, rec_bar_count(d.B) * sizeof(unsigned), st));
    Phase ph(st, "k2_rec_fwd", 2.0 * d.BT() * d.H * 4.0 * d.H * per_launch);
    rec_fwd_pair_x3(a, sh, rt, st);
  }
}

// K3: the x3 BPTT, one launch per direction, DZ of both directions side by side in
// fp32; K4: dX = DZ Wcat^T, [dW; db] = [X | 1]^T DZ_d, dR = Hprev_d^T DZ_d, fp32-class.
void bwd_x3(const sl_lstm_layer* L, const Dims& d, const float* x, const int32_t* lens, const float* const* W,
            const float* const* R, const float* dy, const float* dh_last, const float* dc_last, float* dx,
            float* const* dW, float* const* dR, float* const* db, float beta, const ReserveView& rv,
            const BwdWork& w, cudaStream_t st) {
  const int64_t G = g4(d), Gc = d.nd * G;
  const int M = (int)d.BT();
  const TcBwdShape sh = tc_rec_bwd_x3_shape(d.H, sm_count(), d.nd);
  const int per_launch = sh.pair == 2 ? d.nd : 1;  // both directions at once, or one per launch
  for (int k0 = 0; k0 < d.nd; k0 += per_launch) {
    TcRecBwdArgs a{};
    a.B = d.B;
    a.T = d.T;
    a.H = d.H;
    a.nd = per_launch;
    a.dir0 = sh.pair == 2 ? 0 : k0;
    a.lens = lens;
    a.dy = dy;
    a.dy_ld = (int64_t)d.nd * d.H;
    a.dh_last = dh_last;
    a.dc_last = dc_last;
    a.dzimg = w.dzi;
    a.dzimg_rows = M;
    a.trace = g_rec_trace;  // (experiments builds stamp it; null otherwise)
    a.debug_flags = g_rec_debug_flags;
    a.dzcat_ld = dzi_ld(d);
    a.dz_dir_off = G;
    a.bar = w.bar;
    const __nv_bfloat16* rb[2] = {nullptr, nullptr};
    for (int j = 0; j < per_launch; ++j) {
      const int k = k0 + j;
      a.dirsign[j] = dir_sign(L, k);
      a.gatesf[j] = rv.gates[k];
      a.cprevf[j] = rv.cprev[k];
      a.dzring[j] = w.dzring[k];
      a.dzring_lo[j] = w.dzringlo[k];
      tc_rec_bwd_x3_pack(R[k], d.H, sh, w.rb[k], st);
      rb[j] = w.rb[k];
      SL_CUDA_TRY(cudaMemsetAsync(w.dzring[k], 0, sizeof(__nv_bfloat16) * 2 * dz_ring_bp(d.B) * sh.Kz, st));
      SL_CUDA_TRY(cudaMemsetAsync(w.dzringlo[k], 0, sizeof(__nv_bfloat16) * 2 * dz_ring_bp(d.B) * sh.Kz, st));
    }
    SL_CUDA_TRY(cudaMemsetAsync(w.bar, 0, rec_bar_count(d.B) * sizeof(unsigned), st));
    Phase ph(st, "k3_rec_bwd", 2.0 * d.BT() * d.H * 4.0 * d.H * per_launch);
    rec_bwd_x3(a, sh, rb, st);
  }
  const int64_t wl = wimg_ld(d), xl = ximg_ld(d);
  if (dx) {  // dX = DZ [W_fw | W_bw]^T from the forward's image of the weights
    Phase ph(st, "k4_dx_gemm", 2.0 * M * (double)Gc * d.D);
    gemm_f32x3_ex(false, true, M, d.D, (int)Gc, nullptr, 0, w.dzi, nullptr, 0, rv.wimg, beta, dx, d.D, nullptr,
                  nullptr, 0, w.gws, st, dzi_ld(d), (int64_t)M * dzi_ld(d), wl, (int64_t)d.D * wl);
  }
  // the weight gradients read direction k's column slice of the same DZ image
  const int64_t zl = dzi_ld(d), zlo = (int64_t)M * zl;
  for (int k = 0; k < d.nd; ++k) {
    float* dbk = db ? db[k] : nullptr;
    const bool want_w = dW && dW[k], want_r = dR && dR[k];
    const __nv_bfloat16* zk = w.dzi + k * G;
    if (want_w || dbk) {
      Phase ph(st, "k4_dw_gemm", 2.0 * M * (double)G * d.D);
      if (want_w) {
        const __nv_bfloat16* xi = d.x_x3() ? reinterpret_cast<const __nv_bfloat16*>(x) : rv.ximg;
        gemm_f32x3_ex(true, false, d.D, (int)G, M, nullptr, 0, xi, nullptr, 0, zk, beta, dW[k], G, nullptr,
                      dbk, G, w.gws, st, xl, (int64_t)M * xl, zl, zlo);
      } else {  // db alone: fixed-order column sums of DZ_d (hi + lo)
        colsum_img_kernel<<<(unsigned)ceil_div(G, 256), 256, 0, st>>>(M, (int)G, zk, zl, zlo, beta, dbk);
        SL_CUDA_TRY(cudaGetLastError());
        count_launch();
      }
    }
    if (want_r) {
      Phase ph(st, "k4_dr_gemm", 2.0 * M * (double)G * d.H);
      gemm_f32x3_ex(true, false, d.H, (int)G, M, nullptr, 0, rv.hprevi[k], nullptr, 0, zk, beta, dR[k], G, nullptr,
                    nullptr, 0, w.gws, st, x3_img_ld(d.H), (int64_t)M * x3_img_ld(d.H), zl, zlo);
    }
  }
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

int64_t sl_lstm_bf16_pitch(int32_t features) { return round_up((int64_t)features + 1, 64); }

size_t sl_adam_scratch_size(void) { return sizeof(AdamScratch); }

static void check_attention(const sl_attention* at) {
  SL_REQUIRE(at != nullptr, SL_ERR_INVALID_ARGUMENT, "attention: null descriptor");
  SL_REQUIRE(at->batch > 0 && at->src_time > 0 && at->key_dim > 0 && at->enc_dim > 0 && at->state_dim > 0,
             SL_ERR_SHAPE, "softmax_over_spatial: needs Batch and Time axes (all extents > 0)");
}

size_t sl_attention_workspace_size(const sl_attention* at) {
  if (!at || at->batch <= 0 || at->key_dim <= 0 || at->state_dim <= 0) return 0;
  return attention_workspace_bytes(at->batch, at->key_dim, at->state_dim, at->src_time);
}

static AttnArgs attn_args(const sl_attention* at, const int32_t* lens, const float* enc_ctx, const float* enc,
                          const float* accum, const float* W_fb, const float* b_fb, const float* v) {
  AttnArgs p{};
  p.B = at->batch;
  p.Ts = at->src_time;
  p.K = at->key_dim;
  p.E = at->enc_dim;
  p.H = at->state_dim;
  p.lens = lens;
  p.enc_ctx = enc_ctx;
  p.enc = enc;
  p.accum = accum;
  p.W_fb = W_fb;
  p.b_fb = b_fb;
  p.v = v;
  return p;
}

int sl_attention_step_fwd(const sl_attention* at, const int32_t* src_lens, const float* enc_ctx,
                          const float* enc, const float* s, const float* accum, const float* W_s,
                          const float* b_s, const float* W_fb, const float* b_fb, const float* v,
                          const float* b_v, float* att_out, float* a, float* accum_out, void* workspace,
                          size_t workspace_bytes, sl_stream_t stream) {
  return guarded([&] {
    check_attention(at);
    SL_REQUIRE(src_lens && enc_ctx && enc && s && accum && W_s && b_s && W_fb && b_fb && v && b_v && att_out &&
                   a && accum_out,
               SL_ERR_INVALID_ARGUMENT, "attention fwd: null pointer argument");
    SL_REQUIRE(workspace && workspace_bytes >= attention_workspace_bytes(at->batch, at->key_dim, at->state_dim, at->src_time),
               SL_ERR_WORKSPACE, "attention: workspace too small");
    AttnArgs p = attn_args(at, src_lens, enc_ctx, enc, accum, W_fb, b_fb, v);
    p.b_v = b_v;
    p.att = att_out;
    p.a = a;
    p.accum_out = accum_out;
    attention_fwd(p, s, W_s, b_s, workspace, reinterpret_cast<cudaStream_t>(stream));
  });
}

int sl_attention_step_bwd(const sl_attention* at, const int32_t* src_lens, const float* enc_ctx,
                          const float* enc, const float* s, const float* accum, const float* W_s,
                          const float* b_s, const float* W_fb, const float* b_fb, const float* v,
                          const float* a, const float* d_att, const float* d_accum_out, float* d_enc_ctx,
                          float* d_enc, float* d_s, float* d_accum, float* d_W_s, float* d_b_s, float* d_W_fb,
                          float* d_b_fb, float* d_v, float* d_b_v, int accumulate, void* workspace,
                          size_t workspace_bytes, sl_stream_t stream) {
  return guarded([&] {
    check_attention(at);
    SL_REQUIRE(src_lens && enc_ctx && enc && s && accum && W_s && b_s && W_fb && b_fb && v && a && d_att &&
                   d_enc_ctx && d_enc && d_accum && d_W_fb && d_b_fb && d_v && d_b_v,
               SL_ERR_INVALID_ARGUMENT, "attention bwd: null pointer argument");
    SL_REQUIRE(workspace && workspace_bytes >= attention_workspace_bytes(at->batch, at->key_dim, at->state_dim, at->src_time),
               SL_ERR_WORKSPACE, "attention: workspace too small");
    AttnArgs p = attn_args(at, src_lens, enc_ctx, enc, accum, W_fb, b_fb, v);
    p.a_saved = a;
    p.d_att = d_att;
    p.d_accum_out = d_accum_out;
    p.d_enc_ctx = d_enc_ctx;
    p.d_enc = d_enc;
    p.d_accum = d_accum;
    p.d_W_fb = d_W_fb;
    p.d_b_fb = d_b_fb;
    p.d_v = d_v;
    p.d_b_v = d_b_v;
    p.accumulate = accumulate != 0;
    attention_bwd(p, s, W_s, b_s, d_s, d_W_s, d_b_s, workspace, reinterpret_cast<cudaStream_t>(stream));
  });
}

size_t sl_output_ce_workspace_size(int32_t batch, int32_t time, int32_t input_dim, int32_t vocab) {
  if (batch <= 0 || time <= 0 || input_dim <= 0 || vocab <= 0) return 0;
  return output_ce_workspace_bytes(batch, time, input_dim, vocab);
}

int sl_output_ce(int32_t batch, int32_t time, int32_t input_dim, int32_t vocab, const float* x,
                 const int32_t* targets, const int32_t* seq_lens, const float* W, const float* b,
                 float epsilon, float* loss, float* dx, float* dW, float* db, int accumulate,
                 void* workspace, size_t workspace_bytes, int32_t* bad_target, sl_stream_t stream) {
  return guarded([&] {
    SL_REQUIRE(epsilon >= 0.f && epsilon < 1.f, SL_ERR_INVALID_ARGUMENT,
               "label smoothing epsilon must be in [0, 1)");  // reference tape.cpp:1226-1228
    SL_REQUIRE(batch > 0 && time > 0 && input_dim > 0 && vocab > 0, SL_ERR_SHAPE,
               "output_ce: log_probs must end in Feature axis (B, T, D, V > 0)");
    SL_REQUIRE(x && targets && seq_lens && W && b && loss && bad_target, SL_ERR_INVALID_ARGUMENT,
               "output_ce: null pointer argument");
    SL_REQUIRE(workspace && workspace_bytes >= output_ce_workspace_bytes(batch, time, input_dim, vocab),
               SL_ERR_WORKSPACE, "output_ce: workspace too small");
    output_ce(batch, time, input_dim, vocab, x, targets, seq_lens, W, b, epsilon, loss, dx, dW, db,
              accumulate != 0, workspace, bad_target, reinterpret_cast<cudaStream_t>(stream));
  });
}

size_t sl_output_ce_f32_workspace_size(int32_t batch, int32_t time, int32_t input_dim, int32_t vocab) {
  if (batch <= 0 || time <= 0 || input_dim <= 0 || vocab <= 0) return 0;
  return output_ce_f32_workspace_bytes(batch, time, input_dim, vocab);
}

int sl_output_ce_f32(int32_t batch, int32_t time, int32_t input_dim, int32_t vocab, const float* x,
                     const int32_t* targets, const int32_t* seq_lens, const float* W, const float* b,
                     float epsilon, float* loss, float* dx, float* dW, float* db, int accumulate,
                     void* workspace, size_t workspace_bytes, int32_t* bad_target, sl_stream_t stream) {
  return guarded([&] {
    SL_REQUIRE(epsilon >= 0.f && epsilon < 1.f, SL_ERR_INVALID_ARGUMENT,
               "label smoothing epsilon must be in [0, 1)");  // reference tape.cpp:1226-1228
    SL_REQUIRE(batch > 0 && time > 0 && input_dim > 0 && vocab > 0, SL_ERR_SHAPE,
               "output_ce: log_probs must end in Feature axis (B, T, D, V > 0)");
    SL_REQUIRE(x && targets && seq_lens && W && b && loss && bad_target, SL_ERR_INVALID_ARGUMENT,
               "output_ce: null pointer argument");
    SL_REQUIRE(workspace && workspace_bytes >= output_ce_f32_workspace_bytes(batch, time, input_dim, vocab),
               SL_ERR_WORKSPACE, "output_ce: workspace too small");
    output_ce_f32(batch, time, input_dim, vocab, x, targets, seq_lens, W, b, epsilon, loss, dx, dW, db,
                  accumulate != 0, workspace, bad_target, reinterpret_cast<cudaStream_t>(stream));
  });
}

size_t sl_embedding_workspace_size(int64_t n_ids, int32_t vocab) {
  if (n_ids < 0 || vocab <= 0) return 0;
  return embedding_workspace_bytes(n_ids, vocab);
}

static void check_embedding(int64_t n, int32_t vocab, int32_t dim) {
  SL_REQUIRE(vocab > 0 && dim > 0 && n >= 0 && n < INT32_MAX, SL_ERR_SHAPE,
             "gather_rows: table must be [Feature=V, Other=D] (V, D > 0)");  // tape.cpp:451-453
}

int sl_embedding_fwd(int64_t n_ids, const int32_t* ids, int32_t vocab, int32_t dim, const float* table,
                     float* out, int64_t out_ld, int flags, int32_t* bad_row, sl_stream_t stream) {
  return guarded([&] {
    check_embedding(n_ids, vocab, dim);
    SL_REQUIRE((ids && table && out) || n_ids == 0, SL_ERR_INVALID_ARGUMENT, "embedding: null pointer argument");
    SL_REQUIRE(bad_row, SL_ERR_INVALID_ARGUMENT, "embedding: null bad_row");
    SL_REQUIRE(out_ld >= dim && (flags & ~SL_EMB_NEGATIVE_ZERO) == 0, SL_ERR_INVALID_ARGUMENT,
               "embedding: out_ld < dim or unsupported flags");
    embedding_fwd(n_ids, ids, vocab, dim, table, out, out_ld, flags, bad_row, reinterpret_cast<cudaStream_t>(stream));
  });
}

int sl_embedding_fwd_bf16(int64_t n_ids, const int32_t* ids, int32_t vocab, int32_t dim, const float* table,
                          void* out_bf16, int64_t out_ld, int flags, int32_t* bad_row, sl_stream_t stream) {
  return guarded([&] {
    check_embedding(n_ids, vocab, dim);
    SL_REQUIRE((ids && table && out_bf16) || n_ids == 0, SL_ERR_INVALID_ARGUMENT,
               "embedding: null pointer argument");
    SL_REQUIRE(bad_row, SL_ERR_INVALID_ARGUMENT, "embedding: null bad_row");
    SL_REQUIRE(out_ld >= dim + ((flags & SL_EMB_ONES_COLUMN) ? 1 : 0) &&
                   (flags & ~(SL_EMB_ONES_COLUMN | SL_EMB_NEGATIVE_ZERO)) == 0,
               SL_ERR_INVALID_ARGUMENT, "embedding: out_ld too small (ones column) or unsupported flags");
    embedding_fwd_bf16(n_ids, ids, vocab, dim, table, static_cast<__nv_bfloat16*>(out_bf16), out_ld, flags,
                       bad_row, reinterpret_cast<cudaStream_t>(stream));
  });
}

int sl_embedding_bwd(int64_t n_ids, const int32_t* ids, int32_t vocab, int32_t dim, const float* d_out,
                     int64_t d_out_ld, float* d_table, int accumulate, void* workspace, size_t workspace_bytes,
                     sl_stream_t stream) {
  return guarded([&] {
    check_embedding(n_ids, vocab, dim);
    SL_REQUIRE(d_table && ((ids && d_out) || n_ids == 0), SL_ERR_INVALID_ARGUMENT,
               "embedding: null pointer argument");
    SL_REQUIRE(d_out_ld >= dim, SL_ERR_INVALID_ARGUMENT, "embedding: d_out_ld < dim");
    SL_REQUIRE(workspace && workspace_bytes >= embedding_workspace_bytes(n_ids, vocab), SL_ERR_WORKSPACE,
               "embedding: workspace too small");
    embedding_bwd(n_ids, ids, vocab, dim, d_out, d_out_ld, d_table, accumulate != 0, workspace,
                  reinterpret_cast<cudaStream_t>(stream));
  });
}

static DecDims dec_dims(const sl_attn_decoder* d) {
  SL_REQUIRE(d, SL_ERR_INVALID_ARGUMENT, "attn_decoder: null descriptor");
  return DecDims{d->batch, d->src_time, d->trg_time, d->embed_dim, d->enc_dim, d->hidden, d->key_dim,
                 d->readout_dim, d->trg_vocab};
}
static DecParams dec_params(const sl_attn_decoder_params* p) {
  SL_REQUIRE(p, SL_ERR_INVALID_ARGUMENT, "attn_decoder: null params");
  const float* all[] = {p->enc_ctx_W, p->enc_ctx_b, p->s_W, p->s_R, p->s_b, p->fb_W, p->fb_b,
                        p->s_tr_W, p->s_tr_b, p->e_W, p->e_b, p->readout_W, p->readout_b, p->trg_W};
  for (const float* q : all)
    SL_REQUIRE(q && ((uintptr_t)q & 15) == 0, SL_ERR_INVALID_ARGUMENT,
               "attn_decoder: parameter pointers must be non-null and 16 B aligned");
  return DecParams{p->enc_ctx_W, p->enc_ctx_b, p->s_W, p->s_R, p->s_b, p->fb_W, p->fb_b,
                   p->s_tr_W, p->s_tr_b, p->e_W, p->e_b, p->readout_W, p->readout_b, p->trg_W};
}

size_t sl_attn_decoder_workspace_size(const sl_attn_decoder* dec) {
  try {
    const DecDims d = dec_dims(dec);
    decoder_check(d);
    set_error("");
    return decoder_workspace_bytes(d);
  } catch (const Error& e) {
    set_error(e.msg);
    return 0;
  }
}

int sl_attn_decoder_fwd(const sl_attn_decoder* dec, const sl_attn_decoder_params* params, const void* enc_bf16,
                        int64_t enc_ld, const int32_t* src_lens, const int32_t* prev_ids, float* readout,
                        int32_t* bad_row, void* workspace, size_t workspace_bytes, sl_stream_t stream) {
  return guarded([&] {
    const DecDims d = dec_dims(dec);
    decoder_check(d);
    const DecParams p = dec_params(params);
    SL_REQUIRE(enc_bf16 && src_lens && prev_ids && readout && bad_row, SL_ERR_INVALID_ARGUMENT,
               "attn_decoder: null pointer argument");
    SL_REQUIRE(workspace && workspace_bytes >= decoder_workspace_bytes(d), SL_ERR_WORKSPACE,
               "attn_decoder: workspace too small");
    decoder_fwd(d, p, static_cast<const __nv_bfloat16*>(enc_bf16), enc_ld, src_lens, prev_ids, readout, bad_row,
                workspace, reinterpret_cast<cudaStream_t>(stream));
  });
}

int sl_attn_decoder_bwd(const sl_attn_decoder* dec, const sl_attn_decoder_params* params,
                        const sl_attn_decoder_grads* grads, const void* enc_bf16, int64_t enc_ld,
                        const int32_t* src_lens, const int32_t* prev_ids, const float* readout,
                        const float* d_readout, float* d_enc, void* workspace, size_t workspace_bytes,
                        sl_stream_t stream) {
  return guarded([&] {
    const DecDims d = dec_dims(dec);
    decoder_check(d);
    const DecParams p = dec_params(params);
    SL_REQUIRE(grads, SL_ERR_INVALID_ARGUMENT, "attn_decoder: null grads");
    const sl_attn_decoder_grads& q = *grads;
    float* all[] = {q.enc_ctx_W, q.enc_ctx_b, q.s_W, q.s_R, q.s_b, q.fb_W, q.fb_b,
                    q.s_tr_W, q.s_tr_b, q.e_W, q.e_b, q.readout_W, q.readout_b, q.trg_W};
    for (float* x : all)
      SL_REQUIRE(x && ((uintptr_t)x & 15) == 0, SL_ERR_INVALID_ARGUMENT,
                 "attn_decoder: gradient pointers must be non-null and 16 B aligned");
    SL_REQUIRE(enc_bf16 && src_lens && prev_ids && readout && d_readout && d_enc, SL_ERR_INVALID_ARGUMENT,
               "attn_decoder: null pointer argument");
    SL_REQUIRE(workspace && workspace_bytes >= decoder_workspace_bytes(d), SL_ERR_WORKSPACE,
               "attn_decoder: workspace too small");
    const DecGrads g{q.enc_ctx_W, q.enc_ctx_b, q.s_W, q.s_R, q.s_b, q.fb_W, q.fb_b,
                     q.s_tr_W, q.s_tr_b, q.e_W, q.e_b, q.readout_W, q.readout_b, q.trg_W};
    decoder_bwd(d, p, g, static_cast<const __nv_bfloat16*>(enc_bf16), enc_ld, src_lens, prev_ids, readout,
                d_readout, d_enc, workspace, reinterpret_cast<cudaStream_t>(stream));
  });
}

size_t sl_attn_decoder_f32_workspace_size(const sl_attn_decoder* dec) {
  try {
    const DecDims d = dec_dims(dec);
    decoder_f32_check(d);
    set_error("");
    return decoder_f32_workspace_bytes(d);
  } catch (const Error& e) {
    set_error(e.msg);
    return 0;
  }
}

int sl_attn_decoder_fwd_f32(const sl_attn_decoder* dec, const sl_attn_decoder_params* params, const float* enc,
                            const int32_t* src_lens, const int32_t* prev_ids, float* readout, int32_t* bad_row,
                            void* workspace, size_t workspace_bytes, sl_stream_t stream) {
  return guarded([&] {
    const DecDims d = dec_dims(dec);
    decoder_f32_check(d);
    const DecParams p = dec_params(params);
    SL_REQUIRE(enc && src_lens && prev_ids && readout && bad_row, SL_ERR_INVALID_ARGUMENT,
               "attn_decoder: null pointer argument");
    SL_REQUIRE(workspace && workspace_bytes >= decoder_f32_workspace_bytes(d), SL_ERR_WORKSPACE,
               "attn_decoder: workspace too small");
    decoder_f32_fwd(d, p, enc, src_lens, prev_ids, readout, bad_row, workspace, reinterpret_cast<cudaStream_t>(stream));
  });
}

int sl_attn_decoder_bwd_f32(const sl_attn_decoder* dec, const sl_attn_decoder_params* params,
                            const sl_attn_decoder_grads* grads, const float* enc, const int32_t* src_lens,
                            const int32_t* prev_ids, const float* readout, const float* d_readout, float* d_enc,
                            void* workspace, size_t workspace_bytes, sl_stream_t stream) {
  return guarded([&] {
    const DecDims d = dec_dims(dec);
    decoder_f32_check(d);
    const DecParams p = dec_params(params);
    SL_REQUIRE(grads, SL_ERR_INVALID_ARGUMENT, "attn_decoder: null grads");
    const sl_attn_decoder_grads& q = *grads;
    float* all[] = {q.enc_ctx_W, q.enc_ctx_b, q.s_W, q.s_R, q.s_b, q.fb_W, q.fb_b,
                    q.s_tr_W, q.s_tr_b, q.e_W, q.e_b, q.readout_W, q.readout_b, q.trg_W};
    for (float* x : all)
      SL_REQUIRE(x && ((uintptr_t)x & 15) == 0, SL_ERR_INVALID_ARGUMENT,
                 "attn_decoder: gradient pointers must be non-null and 16 B aligned");
    SL_REQUIRE(enc && src_lens && prev_ids && readout && d_readout && d_enc, SL_ERR_INVALID_ARGUMENT,
               "attn_decoder: null pointer argument");
    SL_REQUIRE(workspace && workspace_bytes >= decoder_f32_workspace_bytes(d), SL_ERR_WORKSPACE,
               "attn_decoder: workspace too small");
    const DecGrads g{q.enc_ctx_W, q.enc_ctx_b, q.s_W, q.s_R, q.s_b, q.fb_W, q.fb_b,
                     q.s_tr_W, q.s_tr_b, q.e_W, q.e_b, q.readout_W, q.readout_b, q.trg_W};
    decoder_f32_bwd(d, p, g, enc, src_lens, prev_ids, readout, d_readout, d_enc, workspace,
                    reinterpret_cast<cudaStream_t>(stream));
  });
}

static int dropout_call(int32_t B, int32_t T, int32_t F, float rate, uint64_t key0, const int32_t* counter,
                        int64_t counter_value, const float* in, float* out, sl_stream_t stream) {
  return guarded([&] {
    SL_REQUIRE(rate >= 0.f && rate < 1.f, SL_ERR_INVALID_ARGUMENT,
               "dropout rate must be in [0, 1), got " + std::to_string(rate));  // tape.cpp:541-544
    SL_REQUIRE(B >= 0 && T >= 0 && F >= 0, SL_ERR_SHAPE, "dropout: negative extent");
    SL_REQUIRE((in && out) || (int64_t)B * T * F == 0, SL_ERR_INVALID_ARGUMENT, "dropout: null pointer argument");
    dropout_apply(B, T, F, rate, key0, counter, counter_value, in, out, reinterpret_cast<cudaStream_t>(stream));
  });
}
int sl_dropout_fwd(int32_t batch, int32_t time, int32_t features, float rate, uint64_t key0,
                   const int32_t* counter, int64_t counter_value, const float* x, float* y, sl_stream_t stream) {
  return dropout_call(batch, time, features, rate, key0, counter, counter_value, x, y, stream);
}
int sl_dropout_bwd(int32_t batch, int32_t time, int32_t features, float rate, uint64_t key0,
                   const int32_t* counter, int64_t counter_value, const float* dy, float* dx, sl_stream_t stream) {
  return dropout_call(batch, time, features, rate, key0, counter, counter_value, dy, dx, stream);
}

int sl_adam_step(int64_t n, float* params, const float* grads, float* m, float* v, int32_t step,
                 float lr, float beta1, float beta2, float eps, float grad_scale, float clip_norm,
                 void* scratch, float* grad_norm_out, int32_t* nonfinite_out, sl_stream_t stream) {
  return guarded([&] {
    SL_REQUIRE(step >= 0, SL_ERR_INVALID_ARGUMENT, "adam_step: step counts from 1 (0 = device counter)");
    SL_REQUIRE(lr > 0.f && beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f && eps > 0.f,
               SL_ERR_INVALID_ARGUMENT, "adam_step: hyperparameters out of range");
    AdamHyper h{lr, beta1, beta2, eps, grad_scale, clip_norm, step};
    adam_step(n, params, grads, m, v, h, static_cast<AdamScratch*>(scratch), grad_norm_out, nonfinite_out,
              reinterpret_cast<cudaStream_t>(stream));
  });
}

const char* sl_last_error(void) { return g_last_error.c_str(); }

int sl_lstm_layer_path(const sl_lstm_layer* L) {
  int path = 0;
  if (guarded([&] {
        validate(L);
        const Dims d = dims(L);
        path = L->precision == SL_PREC_BF16 ? SL_PATH_BF16_TC : use_x3(d, L->precision) ? SL_PATH_FP32_X3_TC
                                                                                        : SL_PATH_FP32_SIMT;
      }) != SL_OK)
    return 0;
  return path;
}

int sl_lstm_layer_check(const sl_lstm_layer* L) {
  return guarded([&] { validate(L); });
}

size_t sl_lstm_reserve_size(const sl_lstm_layer* L) {
  size_t bytes = 0;
  if (guarded([&] {
        validate(L);
        carve_reserve(dims(L), L->precision, nullptr, &bytes);
      }) != SL_OK)
    return 0;
  return bytes;
}

size_t sl_lstm_workspace_size(const sl_lstm_layer* L) {
  size_t f = 0, b = 0;
  if (guarded([&] {
        validate(L);
        carve_fwd(dims(L), L->precision, nullptr, &f);
        carve_bwd(dims(L), L->precision, nullptr, &b);
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
    const int prec = L->precision;
    SL_REQUIRE(x && seq_lens && W && R && b && y, SL_ERR_INVALID_ARGUMENT,
               "sl_lstm_layer_fwd: null pointer argument");
    for (int k = 0; k < d.nd; ++k)
      SL_REQUIRE(W[k] && R[k] && b[k], SL_ERR_INVALID_ARGUMENT,
                 "sl_lstm_layer_fwd: null weight pointer");
    size_t need_w = 0, need_r = 0;
    FwdWork w = carve_fwd(d, prec, workspace, &need_w);
    SL_REQUIRE(workspace && workspace_bytes >= need_w, SL_ERR_WORKSPACE,
               "sl_lstm_layer_fwd: workspace too small");
    ReserveView rv;
    if (reserve) {
      rv = carve_reserve(d, prec, reserve, &need_r);
      SL_REQUIRE(reserve_bytes >= need_r, SL_ERR_WORKSPACE, "sl_lstm_layer_fwd: reserve too small");
    }
    if (use_x3(d, prec)) {
      fwd_x3(L, d, x, seq_lens, W, R, b, y, h_last, c_last, rv, w, stream);
      return;
    }
    SL_CUDA_TRY(cudaMemsetAsync(w.bar, 0, rec_bar_count(d.B) * sizeof(unsigned), stream));
    const double k1_flops = 2.0 * d.BT() * d.D * 4.0 * d.H * d.nd;
    if (prec == SL_PREC_BF16) {
      // Pack [W_fw | W_bw] and x to bf16 (kept in the reserve for the backward
      // GEMMs), then K1 for both directions as ONE tcgen05 GEMM.
      const Pad pd = pads(d);
      __nv_bfloat16* xb = d.x_bf16() ? reinterpret_cast<__nv_bfloat16*>(const_cast<float*>(x))
                                     : (rv.xb ? rv.xb : w.xb);
      __nv_bfloat16* wcat = rv.wcat ? rv.wcat : w.wcat;
      if (pd.G4p != 4 * d.H) {
        SL_CUDA_TRY(cudaMemsetAsync(wcat, 0, sizeof(__nv_bfloat16) * d.D * pd.Gc, stream));
        SL_CUDA_TRY(cudaMemsetAsync(w.bcat, 0, sizeof(float) * pd.Gc, stream));
      }
      for (int k = 0; k < d.nd; ++k) {
        f32_to_bf16(d.D, 4 * d.H, W[k], 4 * d.H, wcat + k * pd.G4p, pd.Gc, stream);
        SL_CUDA_TRY(cudaMemcpyAsync(w.bcat + k * pd.G4p, b[k], sizeof(float) * 4 * d.H,
                                    cudaMemcpyDeviceToDevice, stream));
      }
      if (!d.x_bf16()) {
        f32_to_bf16(d.BT(), d.D, x, d.D, xb, pd.Dp, stream);
        fill_col_bf16(d.BT(), d.D, xb, pd.Dp, 1.f, stream);
      }
      Phase ph(stream, "k1_xw_gemm", k1_flops);
      TcGemm g{(int)d.BT(), (int)pd.Gc, d.D, xb, pd.Dp, false, wcat, pd.Gc, true,
               nullptr, pd.Gc, 1.f, 0.f, w.bcat};
      g.Cb = w.xwb[0];  // XW in bf16: half the bytes K1 writes and K2 reads
      gemm_bf16_tc(g, stream);
    } else {
      Phase ph(stream, "k1_xw_gemm", k1_flops);
      for (int k = 0; k < d.nd; ++k)  // K1: XW = X W + b over all B*T rows (tape.cpp:1103-1109)
        gemm_f32(false, false, (int)d.BT(), 4 * d.H, d.D, 1.f, x, d.D, W[k], 4 * d.H, 0.f,
                 w.xw[k], 4 * d.H, b[k], stream);
    }
    if (prec == SL_PREC_BF16) {
      const Pad pd = pads(d);
      TcRecFwdArgs a{};
      a.B = d.B;
      a.T = d.T;
      a.H = d.H;
      a.nd = d.nd;
      const TcFwdShape sh = tc_rec_fwd_shape(d.H, d.nd, sm_count());
      a.lens = seq_lens;
      a.xw_ld = w.xw_ld;
      if (d.y_bf16()) {  // the next layer's padded bf16 input, with its ones column
        a.ybf = reinterpret_cast<__nv_bfloat16*>(y);
        a.ybf_ld = round_up((int64_t)d.nd * d.H + 1, 64);
        fill_col_bf16(d.BT(), d.nd * d.H, a.ybf, a.ybf_ld, 1.f, stream);
      } else {
        a.y = y;
        a.y_ld = (int64_t)d.nd * d.H;
      }
      a.h_last = h_last;
      a.c_last = c_last;
      a.hprev_ld = pd.Hp;
      a.bar = w.bar;
      __nv_bfloat16* rt[2] = {nullptr, nullptr};
      for (int k = 0; k < d.nd; ++k) {
        rt[k] = rv.rt[k] ? rv.rt[k] : w.rt[k];
        tc_rec_pack(R[k], d.H, sh, rt[k], stream);
        SL_CUDA_TRY(cudaMemsetAsync(w.hbufb[k], 0, sizeof(__nv_bfloat16) * tc_rec_hbuf_elems(d.B, sh),
                                    stream));
        a.dirsign[k] = dir_sign(L, k);
        a.xw[k] = w.xwb[k];
        a.hbuf[k] = w.hbufb[k];
        a.gates[k] = rv.gatesb[k];
        a.cprev[k] = rv.cprevb[k];
        a.hprev[k] = rv.hprevb[k];
      }
      a.trace = g_rec_trace;
      a.trace_cta = g_rec_trace_cta;
      a.debug_flags = g_rec_debug_flags;
      Phase ph(stream, "k2_rec_fwd", 2.0 * d.BT() * d.H * 4.0 * d.H * d.nd);
      rec_fwd_tc(a, sh, rt, stream);
      return;
    }
    RecFwdArgs a{};
    a.B = d.B;
    a.T = d.T;
    a.H = d.H;
    a.nd = d.nd;
    rec_partition(d.H, d.nd, &a.U, &a.ctas_per_dir);
    a.lens = seq_lens;
    a.xw_ld = w.xw_ld;
    a.y = y;
    a.y_ld = (int64_t)d.nd * d.H;
    a.h_last = h_last;
    a.c_last = c_last;
    a.bar = w.bar;
    for (int k = 0; k < d.nd; ++k) {
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
    const int prec = L->precision;
    SL_REQUIRE(x && seq_lens && W && R && dy && reserve, SL_ERR_INVALID_ARGUMENT,
               "sl_lstm_layer_bwd: null pointer argument");
    size_t need_w = 0, need_r = 0;
    BwdWork w = carve_bwd(d, prec, workspace, &need_w);
    SL_REQUIRE(workspace && workspace_bytes >= need_w, SL_ERR_WORKSPACE,
               "sl_lstm_layer_bwd: workspace too small");
    ReserveView rv = carve_reserve(d, prec, const_cast<void*>(reserve), &need_r);
    SL_REQUIRE(reserve_bytes >= need_r, SL_ERR_WORKSPACE, "sl_lstm_layer_bwd: reserve too small");
    const float beta = accumulate ? 1.f : 0.f;
    if (use_x3(d, prec)) {
      bwd_x3(L, d, x, seq_lens, W, R, dy, dh_last, dc_last, dx, dW, dR, db, beta, rv, w, stream);
      return;
    }
    SL_CUDA_TRY(cudaMemsetAsync(w.bar, 0, rec_bar_count(d.B) * sizeof(unsigned), stream));
    const int M = (int)d.BT(), G = 4 * d.H;
    const double fx = 2.0 * M * G * (double)d.D;
    const double rec_flops = 2.0 * d.BT() * d.H * 4.0 * d.H * d.nd;
    if (prec == SL_PREC_BF16) {
      const Pad pd = pads(d);
      TcRecBwdArgs a{};
      a.B = d.B;
      a.T = d.T;
      a.H = d.H;
      a.nd = d.nd;
      const TcBwdShape sh = tc_rec_bwd_shape(d.H, d.nd, sm_count());
      a.U = sh.U;
      a.P = sh.P;
      a.Kz = sh.Kz;
      a.lens = seq_lens;
      a.dy = dy;
      a.dy_ld = (int64_t)d.nd * d.H;
      a.dh_last = dh_last;
      a.dc_last = dc_last;
      a.dzcat = w.dzb;
      a.dzcat_ld = pd.Gc;
      a.dz_dir_off = pd.G4p;
      a.bar = w.bar;
      a.trace = g_rec_trace;
      a.trace_cta = g_rec_trace_cta;
      a.debug_flags = g_rec_debug_flags;
      if (pd.G4p != G) SL_CUDA_TRY(cudaMemsetAsync(w.dzb, 0, sizeof(__nv_bfloat16) * M * pd.Gc, stream));
      for (int k = 0; k < d.nd; ++k) {
        tc_rec_bwd_pack(R[k], d.H, sh, w.rb[k], stream);
        SL_CUDA_TRY(cudaMemsetAsync(w.dzring[k], 0, sizeof(__nv_bfloat16) * 2 * dz_ring_bp(d.B) * a.Kz,
                                    stream));
        a.dirsign[k] = dir_sign(L, k);
        a.gates[k] = rv.gatesb[k];
        a.cprev[k] = rv.cprevb[k];
        a.dzring[k] = w.dzring[k];
      }
      {
        Phase ph(stream, "k3_rec_bwd", rec_flops);
        rec_bwd_tc(a, sh, w.rb, stream);
      }
      // K4 on tensor cores: DZ of both directions side by side -> one dX GEMM;
      // dW and db from ONE GEMM over [X | 1] (the ones column yields colsum(DZ)).
      if (dx) {
        Phase ph(stream, "k4_dx_gemm", fx * d.nd);
        TcGemm g{M, d.D, (int)pd.Gc, w.dzb, pd.Gc, false, rv.wcat, pd.Gc, false, dx, d.D, 1.f,
                 beta, nullptr};
        gemm_bf16_tc(g, stream);
      }
      for (int k = 0; k < d.nd; ++k) {
        float* dbk = db ? db[k] : nullptr;
        if ((dW && dW[k]) || dbk) {
          Phase ph(stream, "k4_dw_gemm", fx);
          const __nv_bfloat16* xb =
              d.x_bf16() ? reinterpret_cast<const __nv_bfloat16*>(x) : rv.xb;
          TcGemm g{d.D + 1, G, M, xb, pd.Dp, true, w.dzb + k * pd.G4p, pd.Gc, true,
                   dW ? dW[k] : nullptr, G, 1.f, beta, nullptr};
          g.m_split = d.D;
          g.C2 = dbk;
          g.ldc2 = G;
          if (!dbk) g.M = d.D;
          gemm_bf16_tc(g, stream);
        }
        if (dR && dR[k]) {
          Phase ph(stream, "k4_dr_gemm", 2.0 * M * G * (double)d.H);
          TcGemm g{d.H, G, M, rv.hprevb[k], pd.Hp, true, w.dzb + k * pd.G4p, pd.Gc, true, dR[k],
                   G, 1.f, beta, nullptr};
          gemm_bf16_tc(g, stream);
        }
      }
      return;
    }
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
      Phase ph(stream, "k3_rec_bwd", rec_flops);
      rec_bwd_f32(a, stream);
    }
    for (int k = 0; k < d.nd; ++k) {
      // K4: hoisted weight / input gradients over all B*T rows (tape.cpp:1174-1205).
      if (dx) {
        Phase ph(stream, "k4_dx_gemm", fx);
        gemm_f32(false, true, M, d.D, G, 1.f, w.dz[k], G, W[k], G, k == 0 ? beta : 1.f, dx, d.D,
                 nullptr, stream);
      }
      if (dW && dW[k]) {
        Phase ph(stream, "k4_dw_gemm", fx);
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
    SL_REQUIRE(precision == SL_PREC_FP32 || precision == SL_PREC_BF16, SL_ERR_UNSUPPORTED,
               "precision not supported");
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
    SL_REQUIRE(precision == SL_PREC_FP32 || precision == SL_PREC_BF16, SL_ERR_UNSUPPORTED,
               "precision not supported");
    SL_REQUIRE(x && h0 && c0 && W && R && saved, SL_ERR_INVALID_ARGUMENT,
               "sl_lstm_cell_bwd: null pointer argument");
    Phase ph(reinterpret_cast<cudaStream_t>(stream), "k5_cell_bwd", 4.0 * B * (D + H) * 4.0 * H);
    cell_bwd(B, D, H, x, h0, c0, W, R, saved, gh, gc, dx, dh0, dc0, dW, dR, db, accumulate,
             reinterpret_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"

#include "../../include/seqloom_cuda_internal.h"

extern "C" int sl_debug_gemm_bf16(int M, int N, int K, const void* A, int64_t lda, int a_mn,
                                  const void* B, int64_t ldb, int b_mn, float* C, int64_t ldc,
                                  float alpha, float beta, const float* bias, sl_stream_t stream) {
  return guarded([&] {
    TcGemm g{M, N, K, static_cast<const __nv_bfloat16*>(A), lda, a_mn != 0,
             static_cast<const __nv_bfloat16*>(B), ldb, b_mn != 0, C, ldc, alpha, beta, bias};
    gemm_bf16_tc(g, reinterpret_cast<cudaStream_t>(stream));
  });
}

extern "C" int sl_debug_gemm_bf16_split(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
                                        int64_t ldb, int b_mn, float* C, int64_t ldc, int ksplit,
                                        sl_stream_t stream) {
  return guarded([&] {
    TcGemm g{M, N, K, static_cast<const __nv_bfloat16*>(A), lda, a_mn != 0,
             static_cast<const __nv_bfloat16*>(B), ldb, b_mn != 0, C, ldc, 1.f, 0.f, nullptr};
    g.ksplit = ksplit;
    g.split_stride = (int64_t)M * ldc;
    gemm_bf16_tc(g, reinterpret_cast<cudaStream_t>(stream));
  });
}

extern "C" int sl_debug_small_gemm(int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb,
                                   int b_kn, float* C, int64_t ldc, const float* bias, sl_stream_t stream) {
  return guarded([&] {
    small_gemm_bf16(M, N, K, static_cast<const __nv_bfloat16*>(A), lda, static_cast<const __nv_bfloat16*>(B), ldb,
                    b_kn != 0, C, ldc, bias, reinterpret_cast<cudaStream_t>(stream));
  });
}

extern "C" size_t sl_debug_gemm_f32x3_ws(int transA, int transB, int M, int N, int K) {
  return gemm_f32x3_workspace_bytes(transA != 0, transB != 0, M, N, K, false);
}

extern "C" int sl_debug_gemm_f32x3(int transA, int transB, int M, int N, int K, const float* A, int64_t lda,
                                   const float* B, int64_t ldb, float beta, float* C, int64_t ldc, const float* bias,
                                   void* ws, sl_stream_t stream) {
  return guarded([&] {
    gemm_f32x3(transA != 0, transB != 0, M, N, K, A, lda, B, ldb, beta, C, ldc, bias, nullptr, 0, ws,
               reinterpret_cast<cudaStream_t>(stream));
  });
}

extern "C" int sl_debug_gemm_trace(unsigned long long* dev_buf) {
  return guarded([&] { gemm_tc2_set_trace(dev_buf); });
}

extern "C" int sl_debug_set_trace(unsigned long long* dev_buf, int cta) {
  g_rec_trace = dev_buf;
  g_rec_trace_cta = cta;
  return 0;
}

extern "C" int sl_debug_set_flags(int flags) {
  g_rec_debug_flags = flags;
  return 0;
}

extern "C" int sl_debug_gemm_bf16_out(int M, int N, int K, const void* A, int64_t lda,
                                      const void* B, int64_t ldb, void* Cb, int64_t ldc,
                                      const float* bias, sl_stream_t stream) {
  return guarded([&] {
    TcGemm g{M, N, K, static_cast<const __nv_bfloat16*>(A), lda, false,
             static_cast<const __nv_bfloat16*>(B), ldb, true, nullptr, ldc, 1.f, 0.f, bias};
    g.Cb = static_cast<__nv_bfloat16*>(Cb);
    gemm_bf16_tc(g, reinterpret_cast<cudaStream_t>(stream));
  });
}
