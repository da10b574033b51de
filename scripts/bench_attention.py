"""Microbenchmark of the decoder's MLP attention step at the
config-4 shape: B=256 target sequences, Ts=60 source positions, key K=1000,
encoder states E=2000, decoder state H=1000.  Times fwd and bwd with CUDA
events (inputs resident; enc_ctx + enc = 184 MB stay L2/HBM across steps as
in the decoder loop) and reports the achieved bytes/s against the measured
HBM copy bandwidth (the step is bandwidth-bound).  The times include the
step's three small projection GEMMs (fp32-accurate split-bf16 on the tensor
cores, gemm_f32x3.cu), which the algorithmic byte count leaves out.

The reference's own CPU implementation of the same step (oracle/_ref: the
attention subnet built from its Tape ops, fwd + bwd) is timed beside it on a
bounded sample (--cpu-rows batch rows, one thread per row up to the host's
cores) and reported as steps/s scaled to the full batch.

    python scripts/bench_attention.py [--B 256] [--iters 50] [--cpu-rows 16]
"""
import argparse, json, os, sys, threading, time
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
ap.add_argument("--cpu-rows", type=int, default=16, help="batch rows in the CPU reference sample (0 = skip)")
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


def cpu_reference(rows):
    """The reference attention step (fwd + bwd through its Tape) on `rows`
    one-row batches in parallel threads; returns full-batch steps/s."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    import oracle
    ref = oracle.Reference(32)
    rng = np.random.default_rng(0)
    args = dict(enc_ctx=rng.uniform(-1, 1, (1, Ts, K)), enc=rng.uniform(-1, 1, (1, Ts, E)),
                s=rng.uniform(-1, 1, (1, H)), accum=rng.uniform(0, 1, (1, Ts)),
                Ws=rng.uniform(-1, 1, (H, K)) / H ** 0.5, bs=rng.uniform(-.5, .5, K),
                Wfb=rng.uniform(-.5, .5, (1, K)), bfb=rng.uniform(-.5, .5, K),
                v=rng.uniform(-1, 1, (K, 1)) / K ** 0.5, bv=0.0,
                d_att=rng.uniform(-1, 1, (1, E)), d_accum=rng.uniform(-1, 1, (1, Ts)))
    lens = np.full(1, Ts, np.int32)
    threads = max(1, min(rows, os.cpu_count() or 1))
    secs = []

    def one():
        t0 = time.perf_counter()
        for _ in range(rows // threads):
            ref.attention_step(lens, **args)
        secs.append(time.perf_counter() - t0)

    ths = [threading.Thread(target=one) for _ in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    per_row = max(secs) / (rows // threads)  # seconds per batch row per thread
    return {"kind": "reference", "cores": threads, "value": threads / (per_row * B), "unit": "steps/s",
            "sample": f"{threads} threads x {rows // threads} one-row steps (Ts={Ts}, K={K}, E={E}, H={H}), "
                      f"fwd+bwd through the reference Tape (fp32 build), scaled to B={B}"}


if a.cpu_rows:
    try:
        out["cpu_baseline"] = cpu_reference(a.cpu_rows)
        out["gpu_steps_per_s"] = 1e3 / (fwd_ms + bwd_ms)
    except FileNotFoundError as e:
        out["cpu_baseline"] = {"unavailable": str(e)}
print(json.dumps(out))
