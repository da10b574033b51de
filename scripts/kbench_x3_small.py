"""Timing of the fp32-class (x3) GEMM at the decoder's per-step shapes (M = batch)."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm
L = lstm.lib()
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L.sl_debug_gemm_f32x3_ws.restype = ctypes.c_size_t
L.sl_debug_gemm_f32x3_ws.argtypes = [ctypes.c_int] * 5
L.sl_debug_gemm_f32x3.argtypes = [ctypes.c_int] * 5 + [vp, i64, vp, i64, ctypes.c_float, vp, i64, vp, vp, vp]
L.sl_profile_enable.argtypes = [ctypes.c_int]
s = torch.cuda.current_stream().cuda_stream
for (name, M, N, K, tB) in [("cell z = xa W", 256, 4000, 3000, 0), ("g1 dxa = dz W^T", 256, 3000, 4000, 1),
                            ("s_tr", 256, 1000, 1000, 0), ("d s", 256, 1000, 1000, 1)]:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda") if tB else torch.randn(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    ws = torch.empty(L.sl_debug_gemm_f32x3_ws(0, tB, M, N, K), dtype=torch.uint8, device="cuda")
    f = lambda: L.sl_debug_gemm_f32x3(0, tB, M, N, K, A.data_ptr(), K, B.data_ptr(), B.stride(0), 0.0, C.data_ptr(),
                                      N, None, ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    for _ in range(5): f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20): f()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "us": us, "exec_tflops": 3 * 2 * M * N * K / us / 1e6}))
