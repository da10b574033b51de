"""The fp32 output layer's logits GEMM ([B*T, D] x [D, V], x3) in isolation:
plain fp32 output, with bias, and the output layer's own phases (the GEMM with
the softmax-statistics epilogue, the CE pass, dX, dW) — config 4 shapes."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm
from paper_1805_05225_b200.output import OutputCE
L = lstm.lib()
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L.sl_debug_gemm_f32x3_ws.restype = ctypes.c_size_t
L.sl_debug_gemm_f32x3_ws.argtypes = [ctypes.c_int] * 5
L.sl_debug_gemm_f32x3.argtypes = [ctypes.c_int] * 5 + [vp, i64, vp, i64, ctypes.c_float, vp, i64, vp, vp, vp]
B, T, D, V = 256, 60, 1000, int(os.environ.get("V", 20000))
M = B * T


def timed(f, reps=5):
    for _ in range(2): f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): f()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


A = torch.randn(M, D, device="cuda") * 0.1
W = torch.randn(D, V, device="cuda") * 0.03
bias = torch.randn(V, device="cuda") * 0.1
C = torch.empty(M, V, device="cuda")
ws = torch.empty(L.sl_debug_gemm_f32x3_ws(0, 0, M, V, D), dtype=torch.uint8, device="cuda")
st = lambda: torch.cuda.current_stream().cuda_stream
for name, bp in (("plain", None), ("bias", bias.data_ptr())):
    us = timed(lambda: L.sl_debug_gemm_f32x3(0, 0, M, V, D, A.data_ptr(), D, W.data_ptr(), V, 0.0, C.data_ptr(), V,
                                              bp, ws.data_ptr(), st()))
    print(json.dumps({"gemm": "logits " + name + " (splits included)", "us": round(us, 1),
                      "exec_tflops": round(3 * 2 * M * V * D / us / 1e6, 1)}))
del C, ws
out = OutputCE(B, T, D, V, precision=os.environ.get("PREC", "fp32"))
x = A.view(B, T, D)
tg = torch.randint(0, V, (B, T), device="cuda", dtype=torch.int32)
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
dx = torch.empty(B, T, D, device="cuda"); dW = torch.empty(D, V, device="cuda"); db = torch.empty(V, device="cuda")
us = timed(lambda: out.forward_backward(x, tg, lens, W, bias, dx, dW, db))
print(json.dumps({"output_ce_f32 fwd+bwd": round(us, 1)}))


class Entry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("calls", ctypes.c_int32), ("ms", ctypes.c_double),
                ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]


L.sl_profile_enable.argtypes = [ctypes.c_int]
L.sl_profile_read(None, 0, 1)
L.sl_profile_enable(1)
for _ in range(3):
    out.forward_backward(x, tg, lens, W, bias, dx, dW, db)
torch.cuda.synchronize()
L.sl_profile_enable(0)
es = (Entry * 64)()
n = L.sl_profile_read(es, 64, 1)
for e in es[:n]:
    print(json.dumps({"phase": e.name.decode(), "us_per_call": round(e.ms / e.calls * 1e3, 1)}))
