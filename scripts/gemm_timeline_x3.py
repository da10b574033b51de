"""Per-CTA timeline of the pair GEMM in x3 mode (sl_debug_gemm_trace) at the decoder's
per-step shapes, through sl_debug_gemm_f32x3 (operand split + GEMM + split-K reduce;
the trace covers the GEMM kernel)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm
L = lstm.lib()
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L.sl_debug_gemm_f32x3_ws.restype = ctypes.c_size_t
L.sl_debug_gemm_f32x3_ws.argtypes = [ctypes.c_int] * 5
L.sl_debug_gemm_f32x3.argtypes = [ctypes.c_int] * 5 + [vp, i64, vp, i64, ctypes.c_float, vp, i64, vp, vp, vp]
L.sl_debug_gemm_trace.argtypes = [vp]
names = ["entry", "prologue", "1st TMA", "last MMA", "acc ready", "epi done", "final sync", "dealloc"]
for name, tB, M, N, K in [("cell z", 0, 256, 4000, 3000), ("g1 dxa", 1, 256, 3000, 4000), ("s_tr", 0, 256, 1000, 1000)]:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda") if tB else torch.randn(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    ws = torch.empty(L.sl_debug_gemm_f32x3_ws(0, tB, M, N, K), dtype=torch.uint8, device="cuda")
    tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    f = lambda: L.sl_debug_gemm_f32x3(0, tB, M, N, K, A.data_ptr(), K, B.data_ptr(), B.stride(0), 0.0, C.data_ptr(),
                                      N, None, ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    L.sl_debug_gemm_trace(tr.data_ptr())
    f()
    torch.cuda.synchronize()
    L.sl_debug_gemm_trace(None)
    t = tr.view(148, 8).cpu()
    used = t[:, 0] > 0
    t = t[used].double()
    rel = (t - t[:, 0].min()) / 1e3
    print(f"{name}: CTAs {int(used.sum())}")
    for i, n in enumerate(names):
        c = rel[:, i][t[:, i] > 0]
        if len(c):
            print(f"   {n:10s} min {c.min():7.2f} mean {c.mean():7.2f} max {c.max():7.2f} us")
