"""BASELINE config 5: 6-layer BLSTM n=1024 encoder, inference only, batch 1-1024,
T = 60-500 (Switchboard-length frames).  One GPU runs its batch shard; across
the 8 GPUs of a box the batch shards with no communication, so
the box-level number is 8x the per-GPU one at B_total = 8 x B.

For every (B, T) point: the inference-only encoder (no reserves, one shared
workspace, ping-pong activations; encoder.py train=False) is run with inputs
resident in HBM, timed with CUDA events after warm-up, and reported as
frames/s (one frame = one valid (sequence, time) position) and as the average
per-step recurrence latency implied by the K2 phase (sl_profile_*).

The reference CPU path (oracle/_ref: lstm_sequence forward, grad-disabled
Tape) is timed beside it on a bounded sample: one sequence per thread at T=60
through one layer-direction of each input width, scaled to the 6-layer stack.

    python scripts/bench_inference.py [--layers 6] [--hidden 1024] [--feat 40]
        [--batches 1,16,64,256,1024] [--times 60,500] [--iters 3] [--no-cpu]
"""
import argparse
import ctypes
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_05225_b200 import lstm
from paper_1805_05225_b200.encoder import BLSTMEncoder

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=6)
ap.add_argument("--hidden", type=int, default=1024)
ap.add_argument("--feat", type=int, default=40)
ap.add_argument("--batches", default="1,16,64,256,1024")
ap.add_argument("--times", default="60,500")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--precision", default="bf16")
ap.add_argument("--no-cpu", action="store_true")
a = ap.parse_args()

L = lstm.lib()


L.sl_profile_enable.argtypes = [ctypes.c_int]


class Entry(ctypes.Structure):  # sl_profile_entry (include/seqloom_cuda.h)
    _fields_ = [("name", ctypes.c_char * 32), ("calls", ctypes.c_int32), ("ms", ctypes.c_double),
                ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]


def phases():
    entries = (Entry * 32)()
    n = L.sl_profile_read(entries, 32, 1)
    return {entries[i].name.decode(): (entries[i].ms, entries[i].calls) for i in range(n)}


H, D0, NL = a.hidden, a.feat, a.layers
results = []
for T in [int(t) for t in a.times.split(",")]:
    for B in [int(b) for b in a.batches.split(",")]:
        enc = BLSTMEncoder(NL, B, T, D0, H, precision=a.precision, train=False)
        enc.init_uniform(0)
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand(B, T, D0, device="cuda", generator=g) * 2 - 1
        lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
        for _ in range(2):
            enc.forward(x, lens)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.iters):
            enc.forward(x, lens)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        # one more pass with per-phase events for the recurrence share
        L.sl_profile_read(None, 0, 1)
        L.sl_profile_enable(1)
        enc.forward(x, lens)
        torch.cuda.synchronize()
        L.sl_profile_enable(0)
        ph = phases()
        rec_ms = ph.get("k2_rec_fwd", (0.0, 0))[0]
        flops = 2.0 * B * T * sum(2 * 4 * H * (D + H) for D in [D0] + [2 * H] * (NL - 1))
        row = {"B": B, "T": T, "ms": round(ms, 3), "frames_per_s": B * T / ms * 1e3,
               "tflops": flops / ms / 1e9, "k2_rec_ms": round(rec_ms, 3),
               "k2_us_per_step": round(rec_ms * 1e3 / (NL * T * max(1, -(-B // 256))), 2),
               "box8_frames_per_s_at_8xB": 8 * B * T / ms * 1e3}
        results.append(row)
        print(json.dumps(row), flush=True)
        del enc, x
        torch.cuda.empty_cache()


def cpu_reference(T=60):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    import oracle
    ref = oracle.Reference(32)
    rng = np.random.default_rng(0)
    s = 1 / np.sqrt(H)
    shapes = [D0, 2 * H]
    prm = {D: tuple(rng.uniform(-s, s, shp) for shp in ((D, 4 * H), (H, 4 * H), (4 * H,))) for D in shapes}
    xs = {D: rng.uniform(-1, 1, (1, T, D)) for D in shapes}
    lens = np.full(1, T, np.int32)
    threads = max(1, min(os.cpu_count() or 1, 64))
    res = []

    def one():
        tt = {}
        for D in shapes:
            t0 = time.perf_counter()
            ref.sequence(xs[D], lens, *prm[D], 1)
            tt[D] = time.perf_counter() - t0
        res.append(tt)

    ths = [threading.Thread(target=one) for _ in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    per_seq = max(2 * r[D0] + 2 * (NL - 1) * r[2 * H] for r in res)
    return {"kind": "reference", "cores": threads, "value": threads * T / per_seq, "unit": "frames/s",
            "sample": f"{threads} threads x 1 sequence (T={T}) through one layer-direction of each input "
                      f"width (D={D0}, D={2 * H}; H={H}), forward only, step = 2 t(D0) + {2 * (NL - 1)} t(2H)"}


summary = {"config": "BASELINE configs[4]: 6xBLSTM n=%d, F=%d, inference, %s" % (H, D0, a.precision),
           "points": results}
if not a.no_cpu:
    try:
        summary["cpu_baseline"] = cpu_reference()
    except FileNotFoundError as e:
        summary["cpu_baseline"] = {"unavailable": str(e)}
print(json.dumps(summary))
