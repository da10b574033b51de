"""Time the attention decoder (sl_attn_decoder_fwd/bwd) alone at the config-4 shape.

    python scripts/bench_decoder.py [--batch 256] [--iters 5]

Prints per-call fwd / bwd ms (CUDA events on the launching stream) and the
library's per-phase split (sl_profile_*)."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_05225_b200 import lstm
from paper_1805_05225_b200.decoder import NAMES, AttnDecoder, param_shapes

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--time", type=int, default=60)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
B, T, Emb, H = a.batch, a.time, 620, 1000
E, K, Rd, V = 2 * H, H, H, 20000
dec = AttnDecoder(B, T, T, Emb, E, H, K, Rd, V)
g = torch.Generator(device="cuda").manual_seed(0)
P = {n: (torch.rand(s, device="cuda", generator=g) * 2 - 1) * 0.03 for n, s in param_shapes(Emb, E, H, K, Rd, V).items()}
G = {n: torch.empty_like(P[n]) for n in P}
enc = torch.zeros(B, T, lstm.bf16_pitch(E), dtype=torch.bfloat16, device="cuda")
enc[:, :, :E] = (torch.rand(B, T, E, device="cuda", generator=g) * 2 - 1).bfloat16()
enc[:, :, E] = 1
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
ids = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
ids[:, 0] = -1
dro = torch.rand(B, T, Rd, device="cuda", generator=g) * 2 - 1
ro = dec.forward(enc, lens, ids, P)
dec.backward(enc, lens, ids, P, ro, dro, G)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
fw, bw = [], []
for _ in range(a.iters):
    e[0].record()
    dec.forward(enc, lens, ids, P, readout=ro)
    e[1].record()
    dec.backward(enc, lens, ids, P, ro, dro, G)
    e[2].record()
    torch.cuda.synchronize()
    fw.append(e[0].elapsed_time(e[1]))
    bw.append(e[1].elapsed_time(e[2]))
print(json.dumps({"batch": B, "time": T, "fwd_ms": min(fw), "bwd_ms": min(bw),
                  "fwd_us_per_step": min(fw) * 1e3 / T, "bwd_us_per_step": min(bw) * 1e3 / T}))
