"""Graph-timed microbenchmark of the small-M mma.sync GEMM (sl_debug_small_gemm) at the
decoder's per-step shapes."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_05225_b200 import lstm

L = lstm.lib()
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L.sl_debug_small_gemm.argtypes = [ctypes.c_int] * 3 + [vp, i64, vp, i64, ctypes.c_int, vp, i64, vp, vp]


def timed(f, n=50):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            f()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            f()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for name, M, N, K, b_kn in [("s_tr", 256, 1000, 1000, 1), ("g2", 256, 1000, 1000, 0),
                            ("cell_fwd", 256, 4000, 3000, 1), ("g1", 256, 3000, 4000, 0)]:
    A = torch.randn(M, K + 8, device="cuda").bfloat16()
    B = (torch.randn(K, N + 8, device="cuda") if b_kn else torch.randn(N, K + 8, device="cuda")).bfloat16()
    C = torch.empty(M, N, device="cuda")
    f = lambda: L.sl_debug_small_gemm(M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], b_kn,
                                      C.data_ptr(), N, None, torch.cuda.current_stream().cuda_stream)
    us = timed(f)
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "us": round(us, 2), "tflops": round(2 * M * N * K / us / 1e6, 1)}))
