"""Microbenchmark of the BF16 tcgen05 GEMM at the encoder's K1/K4 shapes (CUDA events)."""
import ctypes, json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm

L = lstm.lib()
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L.sl_debug_gemm_bf16.argtypes = [ctypes.c_int] * 3 + [vp, i64, ctypes.c_int, vp, i64, ctypes.c_int, vp, i64, ctypes.c_float, ctypes.c_float, vp, vp]
res = []
for (name, M, N, K, a_mn, b_mn) in [("k1_xw", 15360, 8000, 2000, 0, 1), ("k1_xw_k620", 15360, 8000, 620, 0, 1),
                                    ("k1_xw_k620_nmajorB", 15360, 8000, 640, 0, 0), ("k4_dx", 15360, 2000, 8000, 0, 0),
                                    ("k4_dw", 2000, 8000, 15360, 1, 1), ("k4_dr", 1000, 4000, 15360, 1, 1),
                                    ("sq8192", 8192, 8192, 8192, 0, 0)]:
    # MN-major operands padded to 64-multiples like the layer's buffers
    pad = lambda n: (n + 63) // 64 * 64
    A = torch.randn((K, pad(M)) if a_mn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, pad(N)) if b_mn else (N, K), device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: L.sl_debug_gemm_bf16(M, N, K, A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn, C.data_ptr(), N, 1.0, 0.0, None, s)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 10
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    # torch/cuBLAS on the same shape for context
    opA = A[:, :M].t() if a_mn else A
    opB = B[:, :N] if b_mn else B.t()
    for _ in range(3): torch.matmul(opA, opB)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n): torch.matmul(opA, opB)
    e1.record(); torch.cuda.synchronize()
    ms_cublas = e0.elapsed_time(e1) / n
    res.append({"gemm": name, "M": M, "N": N, "K": K, "ms": ms, "tflops": 2*M*N*K/ms/1e9, "cublas_bf16out_ms": ms_cublas, "cublas_tflops": 2*M*N*K/ms_cublas/1e9})
    print(json.dumps(res[-1]), flush=True)

# K1 as the layer runs it: bf16 output [M, Gc] with the fused bias (A = x K-major, B = [W_fw|W_bw] N-major)
L.sl_debug_gemm_bf16_out.argtypes = [ctypes.c_int] * 3 + [vp, i64, vp, i64, vp, i64, vp, vp]
for (name, M, N, K, nb) in [("k1_layer0", 15360, 8064, 620, 1), ("k1_layer0_nobias", 15360, 8064, 620, 0),
                           ("k1_layerN", 15360, 8064, 2000, 1), ("k1_dec", 15360, 4032, 2620, 1)]:
    Kp = (K + 1 + 63) // 64 * 64
    A = torch.randn(M, Kp, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda")
    Cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: L.sl_debug_gemm_bf16_out(M, N, K, A.data_ptr(), Kp, B.data_ptr(), N, Cb.data_ptr(), N,
                                         bias.data_ptr() if nb else None, s)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 10
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9}), flush=True)
