"""Accuracy of the split-bf16 ("x3") GEMM vs fp64 at long K, on dZ-like operands
(one large entry per row + many tiny ones: the output layer's dX = dZ W^T)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm
L = lstm.lib()
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L.sl_debug_gemm_f32x3_ws.restype = ctypes.c_size_t
L.sl_debug_gemm_f32x3_ws.argtypes = [ctypes.c_int] * 5
L.sl_debug_gemm_f32x3.argtypes = [ctypes.c_int] * 5 + [vp, i64, vp, i64, ctypes.c_float, vp, i64, vp, vp, vp]
s = torch.cuda.current_stream().cuda_stream
def x3(A, B, transB):
    M, K = A.shape
    N = B.shape[0] if transB else B.shape[1]
    C = torch.empty(M, N, device="cuda")
    ws = torch.empty(L.sl_debug_gemm_f32x3_ws(0, int(transB), M, N, K), dtype=torch.uint8, device="cuda")
    assert L.sl_debug_gemm_f32x3(0, int(transB), M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), 0.0,
                                 C.data_ptr(), N, None, ws.data_ptr(), s) == 0
    return C
g = torch.Generator(device="cuda").manual_seed(0)
def rel(a, b):
    return float((a.double() - b).abs().max() / b.abs().max())
for (M, K, N, kind) in [(15360, 20000, 1000, "dz"), (15360, 4096, 1000, "dz"), (2048, 20000, 1000, "uniform"),
                        (2048, 60000, 1000, "dz"), (2048, 60000, 1000, "uniform")]:
    if kind == "dz":
        A = torch.rand(M, K, device="cuda", generator=g) * 4e-9
        A[torch.arange(M), torch.randint(0, K, (M,), device="cuda", generator=g)] = -7e-5
    else:
        A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    W = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1) * 0.095
    ref = A.double() @ W.double().T
    C = x3(A, W, True)
    print(f"M={M} K={K} N={N} {kind}: x3 rel {rel(C, ref):.3e}; fp32 torch rel {rel(A @ W.T, ref):.3e}", flush=True)
