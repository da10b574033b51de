"""Per-CTA timeline of the pair GEMM (sl_debug_gemm_trace) at the decoder's step shapes."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_05225_b200 import lstm

L = lstm.lib()
vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
L.sl_debug_gemm_bf16_split.argtypes = [ci] * 3 + [vp, i64, ci, vp, i64, ci, vp, i64, ci, vp]
L.sl_debug_gemm_trace.argtypes = [vp]
pad = lambda n: (n + 63) // 64 * 64
names = ["entry", "prologue", "1st TMA", "last MMA", "acc ready", "epi done", "final sync", "dealloc"]
CASES = [("s_tr", 256, 1000, 1000, 1, 4), ("cell_fwd", 256, 4000, 3000, 1, 4), ("g1", 256, 3000, 4000, 0, 6)]
if "--x3" in sys.argv:  # the fp32-class GEMMs' K-tripled operand images
    CASES = [("s_tr x3", 256, 1000, 3008, 1, 10), ("cell_fwd x3", 256, 4000, 9024, 1, 4),
             ("g1 x3", 256, 3000, 12000, 0, 6), ("cell_fwd x3 ks1", 256, 4000, 9024, 1, 1)]
for name, M, N, K, b_mn, ks in CASES:
    A = torch.randn(M, pad(K), device="cuda").bfloat16()
    B = (torch.randn(K, pad(N), device="cuda") if b_mn else torch.randn(N, pad(K), device="cuda")).bfloat16()
    C = torch.empty(ks, M, N, device="cuda")
    tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: L.sl_debug_gemm_bf16_split(M, N, K, A.data_ptr(), A.shape[1], 0, B.data_ptr(), B.shape[1], b_mn,
                                           C.data_ptr(), N, ks, st)
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    L.sl_debug_gemm_trace(tr.data_ptr())
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    f()
    e1.record()
    torch.cuda.synchronize()
    L.sl_debug_gemm_trace(None)
    t = tr.view(148, 8).cpu()
    used = t[:, 0] > 0
    t = t[used].double()
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    print(f"{name}: event {e0.elapsed_time(e1) * 1e3:.1f} us, CTAs {int(used.sum())}")
    for i, n in enumerate(names):
        col = rel[:, i]
        ok = t[:, i] > 0
        if ok.any():
            c = col[ok]
            print(f"   {n:10s} min {c.min():7.2f} mean {c.mean():7.2f} max {c.max():7.2f} us")
