"""One bidirectional LSTM layer fwd+bwd at the config-4 encoder shape, for ncu.

    python scripts/prof_layer.py [--prec bf16] [--D 2000] [--B 256] [--iters 2]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1805_05225_b200 import lstm

ap = argparse.ArgumentParser()
ap.add_argument("--prec", default="bf16")
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--T", type=int, default=60)
ap.add_argument("--D", type=int, default=2000)
ap.add_argument("--H", type=int, default=1000)
ap.add_argument("--nd", type=int, default=2)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--fwd-only", action="store_true")
ap.add_argument("--infer", action="store_true")
a = ap.parse_args()
B, T, D, H, nd = a.B, a.T, a.D, a.H, a.nd
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(B, T, D, device="cuda", generator=g) * 2 - 1
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
s = H ** -0.5
W = [(torch.rand(D, 4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
R = [(torch.rand(H, 4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
b = [(torch.rand(4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(nd)]
dy = torch.rand(B, T, nd * H, device="cuda", generator=g) * 2 - 1
layer = lstm.LSTMLayer(B, T, D, H, nd, 1, a.prec)
for _ in range(a.iters):
    layer.forward(x, lens, W, R, b)
    if not a.fwd_only:
        layer.backward(dy)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
layer.forward(x, lens, W, R, b)
e1.record()
torch.cuda.synchronize()
print(f"fwd layer ms {e0.elapsed_time(e1):.3f}")
from trace_report import report
if os.environ.get("SL_TRACE"):
    import ctypes
    L = lstm.lib()
    L.sl_debug_set_flags(int(os.environ.get("SL_FLAGS", "0")))
    for cta in [int(c) for c in os.environ["SL_TRACE"].split(",")]:
        buf = torch.zeros(T * 16, dtype=torch.int64, device="cuda")
        L.sl_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), cta)
        layer.forward(x, lens, W, R, b, train=not a.infer)
        torch.cuda.synchronize()
        L.sl_debug_set_trace(None, 0)
        report(buf, T, f"fwd cta {cta}{' (inference)' if a.infer else ''}")
if os.environ.get("SL_TRACE_BWD"):
    import ctypes
    L = lstm.lib()
    L.sl_debug_set_flags(int(os.environ.get("SL_FLAGS", "0")))
    for cta in [int(c) for c in os.environ["SL_TRACE_BWD"].split(",")]:
        buf = torch.zeros(T * 16, dtype=torch.int64, device="cuda")
        layer.forward(x, lens, W, R, b)
        L.sl_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), cta)
        layer.backward(dy)
        torch.cuda.synchronize()
        L.sl_debug_set_trace(None, 0)
        report(buf, T, f"bwd cta {cta}")
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    layer.forward(x, lens, W, R, b)
    e0.record(); layer.backward(dy); e1.record(); torch.cuda.synchronize()
    print(f"bwd layer ms {e0.elapsed_time(e1):.3f}")
