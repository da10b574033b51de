// Tensor-core persistent recurrence (rec_tc.cu) — arguments and entry points.
#pragma once
#include "common.cuh"

namespace sl {

// Saved activations of the bf16 path (written by K2, read only by K3), laid
// out step-major and batch-row-interleaved in 16-unit chunks:
//   gates (i,f,g,o)  [T][4][NC][B][16],   c_{s-1}  [T][NC][B][16],
// NC = ceil(H / 16), indexed by processing step s (not by time: the reversed
// direction and ragged lengths map steps to times per row).  The epilogue
// threads of both kernels own one batch row each (TMEM lane = row), so a warp
// touching a 16-unit chunk of 32 consecutive rows hits 1 KB of contiguous
// memory instead of 32 rows 8 KB apart.  A thread's unit slice must not cross
// a 16-unit chunk.
__host__ __device__ inline int save_hq(int H) { return (H + 15) / 16 * 16; }
__host__ __device__ inline size_t gate_save_off(int s, int g, int row, int B, int H, int u) {
  return ((((size_t)s * 4 + g) * (save_hq(H) / 16) + u / 16) * B + row) * 16 + u % 16;
}
__host__ __device__ inline size_t cprev_save_off(int s, int row, int B, int H, int u) {
  return (((size_t)s * (save_hq(H) / 16) + u / 16) * B + row) * 16 + u % 16;
}

// Step counters of the persistent recurrences: kBarPerChunk zeroed unsigned
// per 256-row batch chunk (one launch each), rec_bar_count(B) in total.
constexpr int kBarPerChunk = 512;  // fwd: [dir][tile][16 K groups]; bwd: [dir][tile][128 DZ boxes]
inline size_t rec_bar_count(int B) { return (size_t)kBarPerChunk * ((B + 255) / 256); }

struct TcRecFwdArgs {
  int B, T, H, nd, U, P;  // P = CTAs per direction (= ceil(H / U))
  int b0;                 // first batch row of this launch (set internally)
  int Kp;                 // K padded to 64 (= round_up(H, 64))
  int stages;             // h-tile ring depth (set internally)
  int kb;                 // 64-wide K chunks per TMA box (set internally)
  const int32_t* lens;
  int dirsign[2];
  const __nv_bfloat16* xw[2];  // hoisted x W + b, bf16 [B*T, xw_ld], dir d's gate blocks at col 0
  int64_t xw_ld;
  float* y;  // fp32 [B*T, y_ld] (dir d at col d*H) or null
  int64_t y_ld;
  __nv_bfloat16* ybf;  // bf16 copy of y (next layer's K1 operand) or null
  int64_t ybf_ld;
  float* h_last;  // [nd, B, H] or null
  float* c_last;
  __nv_bfloat16* gates[2];    // saved (i,f,g,o), step-major (gate_save_off; null = inference)
  __nv_bfloat16* cprev[2];    // saved c_{s-1}, step-major (cprev_save_off)
  __nv_bfloat16* hprev[2];    // saved h_{s-1} bf16 [B*T, hprev_ld] (dR GEMM operand)
  int64_t hprev_ld;
  __nv_bfloat16* hbuf[2];     // h ring, zeroed (tc_rec_hbuf_elems): [2][B][Kp] (rec_tc.cu kernels) or
                              // the interleaved dz_ring_off layout with K = Kp (pair kernel)
  unsigned* bar;              // zeroed step counters, 2 per batch chunk
  unsigned long long* trace;  // optional per-step phase timestamps (debug), [T][8] for trace_cta
  int trace_cta;
  int xw_tma;       // pair kernel: x W tiles may be TMA-loaded (set internally)
  // ---- fp32-class ("x3", split-bf16) pair kernel only: one direction per launch
  // (SL_LAYER_Y_X3) y written as its split image instead of fp32: hi rows at yimg (row
  // stride yimg_ld, position-major like y), lo rows yimg_lo elements further on
  __nv_bfloat16* yimg;
  int64_t yimg_ld, yimg_lo;
  int dir0;                      // global index of launch direction 0 (y columns, h_last / c_last rows)
  const float* xwf[2];           // hoisted x W + b, fp32 [B*T, xw_ld]
  __nv_bfloat16* hbuf_lo[2];     // lo halves of h (h - bf16(h)), same ring layout as hbuf (the hi halves)
  float* gatesf[2];              // saved (i,f,g,o) fp32, step-major (gate_save_off)
  float* cprevf[2];              // saved c_{s-1} fp32, step-major (cprev_save_off)
  __nv_bfloat16* hprevi[2];      // saved h_{s-1} as its split image (K4 dR operand): hi [B*T, hprev_ld],
  int64_t hprevi_lo;             // lo hprevi_lo elements further on
  int debug_flags;  // experiments only: 1 = skip MMAs, 2 = skip epilogue math/stores,
                    // 4 = no step-counter waits (wrong results)
};

// DZ ring of the BPTT kernel (written by its epilogues, TMA-read as the MMA A
// operand): [2 slots][Kz / 8][Bp][8] bf16, Bp = round_up(B, 8) — 16 B K-chunks
// of all rows back to back (the SWIZZLE_NONE K-major core-matrix layout), so a
// warp's 32 rows of one 8-unit slice are 512 contiguous bytes.  Gate g of unit
// u is column g * dz_ring_hq(H) + u.
__host__ __device__ inline int dz_ring_hq(int H) { return (H + 7) / 8 * 8; }
__host__ __device__ inline int dz_ring_bp(int B) { return (B + 7) / 8 * 8; }
__host__ __device__ inline size_t dz_ring_off(int slot, int row, int col, int Bp, int Kz) {
  return (((size_t)slot * (Kz / 8) + col / 8) * Bp + row) * 8 + col % 8;
}

struct TcRecBwdArgs {
  int B, T, H, nd, U, P;
  int b0;      // first batch row of this launch (set internally)
  int Kz;      // K of the per-step dh GEMM = gate columns padded to 64 (round_up(4H, 64))
  int stages;  // set internally
  int kb;      // 64-wide K chunks per TMA box (set internally)
  const int32_t* lens;
  int dirsign[2];
  const __nv_bfloat16* gates[2];  // saved by K2: (i,f,g,o), step-major (gate_save_off)
  const __nv_bfloat16* cprev[2];  // saved by K2: c_{s-1}, step-major (cprev_save_off)
  const float* dy;        // [B*T, dy_ld], dir d at col d*H
  int64_t dy_ld;
  const float* dh_last;  // [nd, B, H] or null
  const float* dc_last;
  __nv_bfloat16* dzring[2];  // dz_ring_off layout, 2 * dz_ring_bp(B) * Kz bf16, zeroed
  __nv_bfloat16* dzcat;      // out: DZ bf16 [B*T, dzcat_ld], dir d at col d*dz_dir_off
  int64_t dzcat_ld, dz_dir_off;
  unsigned* bar;  // zeroed step counters
  unsigned long long* trace;
  int trace_cta;
  int debug_flags;  // experiments only: 8 = skip the DZ copy for K4, 16 = skip dy / saved-activation
                    // loads (wrong results)
  // ---- fp32-class ("x3") kernel only: one direction per launch
  int dir0;                        // global index of launch direction 0 (dy columns, final-state rows)
  const float* gatesf[2];          // saved (i,f,g,o) fp32 (K2 x3), step-major
  const float* cprevf[2];          // saved c_{s-1} fp32, step-major
  __nv_bfloat16* dzring_lo[2];     // lo halves of DZ (DZ - bf16(DZ)), dzring layout, zeroed
  // out: DZ's split image (gemm.h x3_split_img layout): hi [B*T, dzcat_ld] at dzimg, lo
  // dzimg_rows * dzcat_ld elements further on; dir (dir0 + d) at col (dir0 + d)*dz_dir_off
  __nv_bfloat16* dzimg;
  int64_t dzimg_rows;
};

// K-split partition of the BPTT kernel: clusters of C CTAs, each finalizing U
// units, P CTAs per direction, Kz = gate columns padded to 64*C.
struct TcBwdShape {
  int C, U, P, Kz;
  int pair = 0;  // 1: CTA-pair kernel (rec_tc_bwd_pair.cu), clusters of 8 = 4 pairs x 128 units
};
TcBwdShape tc_rec_bwd_shape(int H, int nd, int sms);  // C == 0: unsupported
size_t tc_rec_bwd_pack_elems(const TcBwdShape& sh);
void tc_rec_bwd_pack(const float* R, int H, const TcBwdShape& sh, __nv_bfloat16* RB,
                     cudaStream_t stream);
void rec_bwd_tc(const TcRecBwdArgs& a, const TcBwdShape& sh, __nv_bfloat16* const* RB,
                cudaStream_t stream);
bool tc_rec_bwd_pair_fits(int H, int nd, int sms, int B, TcBwdShape* out);
size_t tc_rec_bwd_pair_pack_elems(const TcBwdShape& sh);
void tc_rec_bwd_pair_pack(const float* R, int H, const TcBwdShape& sh, __nv_bfloat16* RB, cudaStream_t stream);
void rec_bwd_pair(const TcRecBwdArgs& a, const TcBwdShape& sh, __nv_bfloat16* const* RB, cudaStream_t stream);

// fp32-class BPTT (split-bf16, "x3"): the K-split kernel with R resident as hi
// and lo bf16 slices, DZ exchanged as hi and lo rings, dh = DZ_hi R_hi^T +
// DZ_lo R_hi^T + DZ_hi R_lo^T in fp32 TMEM, fp32 partial exchange, saves and DZ.
// One direction per launch.
// nd == 2 and the grid fits: both directions in ONE launch (shape.pair == 2: R_hi
// resident, R_lo streamed with DZ in 32-K stages); otherwise one direction per
// launch (shape.pair == 1: R hi + lo resident).
TcBwdShape tc_rec_bwd_x3_shape(int H, int sms, int nd = 1);  // C == 0: unsupported
size_t tc_rec_bwd_x3_pack_elems(const TcBwdShape& sh);  // hi rows then lo rows
void tc_rec_bwd_x3_pack(const float* R, int H, const TcBwdShape& sh, __nv_bfloat16* RB, cudaStream_t stream);
void rec_bwd_x3(const TcRecBwdArgs& a, const TcBwdShape& sh, const __nv_bfloat16* const* RB, cudaStream_t stream);

// K-split partition of the forward kernel: clusters of C CTAs, each finalizing
// U units (the cluster owns C*U units, MMA N = 4*C*U), P CTAs per direction,
// Kp = H padded to 64*C.
struct TcFwdShape {
  int C, U, P, Kp;
  int pair = 0;  // 1: CTA-pair kernel (rec_tc_pair.cu): U = units per pair, P = pairs per direction
};
TcFwdShape tc_rec_fwd_shape(int H, int nd, int sms);  // C == 0: unsupported
size_t tc_rec_hbuf_elems(int B, const TcFwdShape& sh);  // one direction's h ring
size_t tc_rec_pack_elems(const TcFwdShape& sh);         // one direction's packed R^T
// Pack R [H, 4H] fp32 into the per-CTA K-major bf16 slices the kernel loads.
void tc_rec_pack(const float* R, int H, const TcFwdShape& sh, __nv_bfloat16* RT,
                 cudaStream_t stream);
void rec_fwd_tc(const TcRecFwdArgs& a, const TcFwdShape& sh, __nv_bfloat16* const* RT,
                cudaStream_t stream);
bool tc_rec_fwd_pair_fits(int H, int nd, int sms);
int tc_rec_fwd_pair_units(int H, int nd, int sms);  // units per pair of the bf16 pair kernel: 32 or 16
void rec_fwd_pair(const TcRecFwdArgs& a, const TcFwdShape& sh, __nv_bfloat16* const* RT,
                  cudaStream_t stream);

// fp32-class forward recurrence (split-bf16, "x3"): the pair kernel with 16
// units per pair, R^T resident as hi and lo bf16 slices, h exchanged as hi and
// lo bf16 rings, z = h_hi R_hi + h_lo R_hi + h_hi R_lo accumulated in fp32
// TMEM; fp32 x W, cell state, saves and outputs.  One direction per launch
// (both directions' hi+lo R do not fit in shared memory at once).
// nd == 2 and the grid fits: both directions in ONE launch (shape.pair == 2: 32 units
// per pair, R hi and lo streamed through the ring with h); otherwise one
// direction per launch (shape.pair == 1: 16 units per pair, R hi + lo resident).
TcFwdShape tc_rec_fwd_x3_shape(int H, int sms, int nd = 1);  // C == 0: unsupported
size_t tc_rec_x3_pack_elems(const TcFwdShape& sh);   // one direction's packed R^T (hi rows, then lo rows)
void tc_rec_x3_pack(const float* R, int H, const TcFwdShape& sh, __nv_bfloat16* RT, cudaStream_t stream);
void rec_fwd_pair_x3(const TcRecFwdArgs& a, const TcFwdShape& sh, const __nv_bfloat16* const* RT,
                     cudaStream_t stream);

}  // namespace sl
