"""Timing of the fp32-class (x3) GEMM (operand splits included) at the decoder's
shapes: the per-step ones (M = batch) and, with --hoisted, the hoisted ones over
all B*T rows (config 4: B=256, T=Ts=60, H=1000, E=2000, K=1000, Emb=620, Rd=1000)."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm
L = lstm.lib()
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L.sl_debug_gemm_f32x3_ws.restype = ctypes.c_size_t
L.sl_debug_gemm_f32x3_ws.argtypes = [ctypes.c_int] * 5
L.sl_debug_gemm_f32x3.argtypes = [ctypes.c_int] * 5 + [vp, i64, vp, i64, ctypes.c_float, vp, i64, vp, vp, vp]
SMALL = [("cell z = xa W", 0, 0, 256, 4000, 3000), ("g1 dxa = dz W^T", 0, 1, 256, 3000, 4000),
         ("s_tr", 0, 0, 256, 1000, 1000), ("d s", 0, 1, 256, 1000, 1000)]
BT = 15360
HOISTED = [("enc_ctx", 0, 0, BT, 1000, 2000), ("xw trg", 0, 0, BT, 4000, 620), ("readout", 0, 0, BT, 1000, 3620),
           ("d ro", 0, 1, BT, 3620, 1000), ("dW_ro", 1, 0, 3620, 1000, BT), ("dW_att", 1, 0, 2000, 4000, BT),
           ("dR", 1, 0, 1000, 4000, BT), ("dW_trg", 1, 0, 620, 4000, BT), ("d trg", 0, 1, BT, 620, 4000),
           ("dW_str", 1, 0, 1000, 1000, BT), ("dW_ctx", 1, 0, 2000, 1000, BT), ("d enc", 0, 1, BT, 2000, 1000)]
shapes = HOISTED if "--hoisted" in sys.argv else SMALL
reps = 3 if "--hoisted" in sys.argv else 20
for (name, tA, tB, M, N, K) in shapes:
    A = torch.randn(K, M, device="cuda") if tA else torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda") if tB else torch.randn(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    ws = torch.empty(L.sl_debug_gemm_f32x3_ws(tA, tB, M, N, K), dtype=torch.uint8, device="cuda")
    f = lambda: L.sl_debug_gemm_f32x3(tA, tB, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), 0.0,
                                      C.data_ptr(), N, None, ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    for _ in range(3): f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): f()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(json.dumps({"gemm": name, "tA": tA, "tB": tB, "M": M, "N": N, "K": K, "us": round(us, 2),
                      "exec_tflops": round(3 * 2 * M * N * K / us / 1e6, 1)}))
    del A, B, C, ws
