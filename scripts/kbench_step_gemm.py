"""Microbenchmark of the attention decoder's per-step GEMMs (M = batch rows) at
several split-K counts, back to back (CUDA events), with cuBLAS for context."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_05225_b200 import lstm

L = lstm.lib()
vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
L.sl_debug_gemm_bf16_split.argtypes = [ci] * 3 + [vp, i64, ci, vp, i64, ci, vp, i64, ci, vp]
pad = lambda n: (n + 63) // 64 * 64


def timed(f, n=50):
    """Device time per call: n calls captured in one CUDA graph, replayed (no host gaps)."""
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
for name, M, N, K, b_mn in [("cell_fwd", 256, 4000, 3000, 1), ("s_tr", 256, 1000, 1000, 1),
                            ("g1", 256, 3000, 4000, 0), ("g2", 256, 1000, 1000, 0)]:
    A = torch.randn(M, pad(K), device="cuda").bfloat16()
    B = (torch.randn(K, pad(N), device="cuda") if b_mn else torch.randn(N, pad(K), device="cuda")).bfloat16()
    nk = (K + 63) // 64
    seen = set()
    for want in (1, 2, 3, 4, 6, 8, 12, 16):
        ks = -(-nk // -(-nk // want))
        if ks in seen:
            continue
        seen.add(ks)
        C = torch.empty(ks, M, N, device="cuda")
        f = lambda: L.sl_debug_gemm_bf16_split(M, N, K, A.data_ptr(), A.shape[1], 0, B.data_ptr(), B.shape[1], b_mn,
                                               C.data_ptr(), N, ks, torch.cuda.current_stream().cuda_stream)
        us = timed(f)
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "ksplit": ks, "us": round(us, 2),
                          "tflops": round(2 * M * N * K / us / 1e6, 1)}), flush=True)
    opB = B[:, :N] if b_mn else B[:, :K].t()
    Ak = A[:, :K]
    us = timed(lambda: torch.matmul(Ak, opB))
    print(json.dumps({"gemm": name, "cublas_us": round(us, 2)}), flush=True)
