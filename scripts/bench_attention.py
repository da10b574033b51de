"""Microbenchmark of the decoder's MLP attention step at the
config-4 shape: B=256 target sequences, Ts=60 source positions, key K=1000,
encoder states E=2000, decoder state H=1000.  Times fwd and bwd with CUDA
events (inputs resident; enc_ctx + enc = 184 MB stay L2/HBM across steps as
in the decoder loop) and reports the achieved bytes/s against the measured
HBM copy bandwidth (the step is bandwidth-bound).  The times include the
step's three small projection GEMMs (fp32-accurate split-bf16 on the tensor
cores, gemm_f32x3.cu), which the algorithmic byte count leaves out.

    python scripts/bench_attention.py [--B 256] [--iters 50]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_05225_b200.attention import Attention

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=256)
ap.add_argument("--Ts", type=int, default=60)
ap.add_argument("--K", type=int, default=1000)
ap.add_argument("--E", type=int, default=2000)
ap.add_argument("--H", type=int, default=1000)
ap.add_argument("--iters", type=int, default=50)
a = ap.parse_args()
B, Ts, K, E, H = a.B, a.Ts, a.K, a.E, a.H
g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: torch.rand(*s, device="cuda", generator=g) * 2 - 1
inp = dict(src_lens=torch.full((B,), Ts, dtype=torch.int32, device="cuda"), enc_ctx=r(B, Ts, K), enc=r(B, Ts, E),
           s=r(B, H), accum=torch.rand(B, Ts, device="cuda", generator=g), W_s=r(H, K) / H ** 0.5, b_s=r(K),
           W_fb=r(1, K), b_fb=r(K), v=r(K, 1) / K ** 0.5)
b_v = torch.zeros(1, device="cuda")
at = Attention(B, Ts, K, E, H)
d_att, d_acc = r(B, E), r(B, Ts)
att, aw, _ = at.forward(**inp, b_v=b_v)


def timeit(f):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(a.iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters


fwd_ms = timeit(lambda: at.forward(**inp, b_v=b_v))
bwd_ms = timeit(lambda: at.backward(**inp, a=aw, d_att=d_att, d_accum_out=d_acc))
fwd_bytes = 4.0 * B * Ts * (K + E)          # enc_ctx + enc read once
bwd_bytes = 4.0 * B * Ts * (2 * K + 2 * E)  # enc_ctx read + d_enc_ctx written, enc read + d_enc written
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = peaks["hbm_gbs"]
out = {"op": "attention_step", "B": B, "Ts": Ts, "K": K, "E": E, "H": H,
       "fwd_us": fwd_ms * 1e3, "bwd_us": bwd_ms * 1e3,
       "fwd_gbs": fwd_bytes / fwd_ms / 1e6, "bwd_gbs": bwd_bytes / bwd_ms / 1e6, "hbm_peak_gbs": hbm,
       "fwd_frac": fwd_bytes / fwd_ms / 1e6 / hbm, "bwd_frac": bwd_bytes / bwd_ms / 1e6 / hbm,
       "per_decoder_step_us": (fwd_ms + bwd_ms) * 1e3,
       "per_training_step_ms_T60": (fwd_ms + bwd_ms) * Ts}
print(json.dumps(out))
