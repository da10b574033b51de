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
# the same two calls captured as CUDA graphs (as the bench step runs them): no host launch gaps
graphs = []
for fn in (lambda: dec.forward(enc, lens, ids, P, readout=ro), lambda: dec.backward(enc, lens, ids, P, ro, dro, G)):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    graphs.append(gr)
gt = []
for gr in graphs:
    gr.replay()
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(a.iters):
        gr.replay()
    e[1].record()
    torch.cuda.synchronize()
    gt.append(e[0].elapsed_time(e[1]) / a.iters)
print(json.dumps({"batch": B, "time": T, "eager_fwd_ms": min(fw), "eager_bwd_ms": min(bw),
                  "graph_fwd_ms": gt[0], "graph_bwd_ms": gt[1],
                  "graph_fwd_us_per_step": gt[0] * 1e3 / T, "graph_bwd_us_per_step": gt[1] * 1e3 / T}))
