"""Per-phase device times (sl_profile, CUDA events on the launching stream) of one
bidirectional LSTM layer fwd+bwd at the config-4 encoder shape, per precision.

    python scripts/phase_layer.py [--D 2000] [--B 256] [--prec fp32,bf16]
"""
import argparse, ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200 import lstm

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--T", type=int, default=60)
ap.add_argument("--D", type=int, default=2000)
ap.add_argument("--H", type=int, default=1000)
ap.add_argument("--prec", default="fp32,bf16")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
L = lstm.lib()
L.sl_profile_enable.argtypes = [ctypes.c_int]
if os.environ.get("SL_DEBUG_FLAGS"):  # experiments builds: timing switches (capi.cu sl_debug_set_flags)
    L.sl_debug_set_flags.argtypes = [ctypes.c_int]
    L.sl_debug_set_flags(int(os.environ["SL_DEBUG_FLAGS"]))


class Entry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("calls", ctypes.c_int32), ("ms", ctypes.c_double),
                ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]


B, T, D, H = a.B, a.T, a.D, a.H
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(B, T, D, device="cuda", generator=g) * 2 - 1
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
s = H ** -0.5
W = [(torch.rand(D, 4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(2)]
R = [(torch.rand(H, 4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(2)]
b = [(torch.rand(4 * H, device="cuda", generator=g) * 2 - 1) * s for _ in range(2)]
dy = torch.rand(B, T, 2 * H, device="cuda", generator=g) * 2 - 1
for prec in a.prec.split(","):
    layer = lstm.LSTMLayer(B, T, D, H, 2, 1, prec)
    for _ in range(2):
        layer.forward(x, lens, W, R, b)
        layer.backward(dy)
    torch.cuda.synchronize()
    L.sl_profile_read(None, 0, 1)
    L.sl_profile_enable(1)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(a.iters):
        layer.forward(x, lens, W, R, b)
        layer.backward(dy)
    e1.record()
    torch.cuda.synchronize()
    L.sl_profile_enable(0)
    ents = (Entry * 64)()
    n = L.sl_profile_read(ents, 64, 1)
    out = {"prec": prec, "B": B, "T": T, "D": D, "H": H,
           "layer_fwd_bwd_ms": e0.elapsed_time(e1) / a.iters,
           "phases": {e.name.decode(): {"ms_per_call": e.ms / e.calls, "calls_per_iter": e.calls / a.iters,
                                        "tflops_alg": e.flops / max(e.ms, 1e-9) / 1e9}
                      for e in ents[:n]}}
    for k in ("k2_rec_fwd", "k3_rec_bwd"):
        if k in out["phases"]:
            ph = out["phases"][k]
            out["phases"][k]["us_per_step"] = ph["ms_per_call"] * 1e3 / T
    print(json.dumps(out), flush=True)
    del layer
    torch.cuda.empty_cache()
