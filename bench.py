"""Benchmark of the BASELINE.json metric on B200.

Metric: "LSTM fwd+bwd target tokens/sec (6xBLSTM n=1000, T=60) at 1/2/4/8 B200
vs CPU" (BASELINE.json), on configs[3] — the Listing-1 attention model's
training step (make_attention_model, models.cpp:26-184): source / target
embedding lookups (V = 20K each; width 620, models.hpp:14) from
token ids, forward + backward of the 6-layer bidirectional LSTM encoder
(H = 1000), enc_ctx, the `output` subnetwork run step by step with teacher
forcing (the LSTM decoder cell with input feeding of the previous attention,
the MLP attention with weight feedback, the relu readout; decoder.py), the
output softmax layer (V = 20K) with the label-smoothed CE loss, T_src = T_tgt
= 60, then the fused global-norm clip + Adam step over all parameters, plus at
N > 1 the data-parallel NCCL gradient all-reduce overlapped with BPTT.
--no-attention runs the earlier step without attention (decoder context = the
encoder output at the same position).  tokens = target (sequence, time)
positions.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (see DESIGN.md §Measurement for every key).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LSTM fwd+bwd target tokens/sec (6×BLSTM n=1000, T=60) at 1/2/4/8 B200 vs CPU"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["fp32", "bf16"], default=os.environ.get("SL_BENCH_PREC", "fp32"),
                    help="fp32 (default, the reference's precision: split-bf16 x3 tensor cores, rel. 1e-4) or bf16")
    ap.add_argument("--config", type=int, choices=[1, 2, 3, 4, 5], default=4,
                    help="BASELINE.json configs[i-1]: 4 (default) = the headline training step; 1-3 = LSTM "
                         "layer / stack fwd+bwd; 5 = the inference sweep")
    ap.add_argument("--no-bf16-line", action="store_true",
                    help="skip the bf16-mode companion measurement reported beside the fp32 headline")
    ap.add_argument("--batch", type=int, default=256, help="sequences per GPU (weak scaling)")
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--hidden", type=int, default=1000)
    ap.add_argument("--input", type=int, default=620)
    ap.add_argument("--time", type=int, default=60)
    ap.add_argument("--vocab", type=int, default=20000, help="target vocabulary (output softmax); 0 = none")
    ap.add_argument("--src-vocab", type=int, default=20000, help="source embedding table rows; 0 = feed embeddings")
    ap.add_argument("--trg-vocab", type=int, default=20000,
                    help="target embedding table rows (needs --vocab); 0 = feed embeddings")
    ap.add_argument("--no-attention", action="store_true",
                    help="the pre-attention step (decoder context = encoder output at t) instead of Listing 1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--dp-selftest", action="store_true",
                    help="(test) issue the gradient all-reduces even at one rank (NCCL, graph-captured), "
                         "to exercise the N>1 step's capture on a single GPU")
    a = ap.parse_args()
    a.attention = not a.no_attention
    if a.attention and not (a.vocab and a.src_vocab and a.trg_vocab):
        ap.error("the attention step needs --vocab, --src-vocab, --trg-vocab > 0 (or --no-attention)")
    return a


def flops_per_token(L, D0, H, V=0, attention=False, Ts=60):
    """Algorithmic GEMM flops per target token, fwd+bwd: 24 H (D + H)
    per layer-direction — the encoder's 2L layer-directions plus the decoder
    cell (D = D0 + 2H); T_src = T_tgt — plus 6 H V for the output layer.  With
    attention (key = readout = H, enc = 2H): + 6 E K (enc_ctx) + 6 H K (s_tr)
    + 6 (H + D0 + E) H (readout) + 6 Ts (K + E) (energies and context, fwd + bwd)."""
    enc = sum(2 * 24 * H * ((D0 if l == 0 else 2 * H) + H) for l in range(L))
    f = enc + 24 * H * (D0 + 2 * H + H) + 6 * H * V
    if attention:
        E, K = 2 * H, H
        f += 6 * E * K + 6 * H * K + 6 * (H + D0 + E) * H + 6 * Ts * (K + E)
    return f


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.skip = 0

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi can take longer to start than a short timed region lasts: wait for its
            # first line (up to 5 s), so the 100 ms samples cover the region; that line itself
            # is taken before the region and is not counted
            t0 = time.time()
            while not self.lines and self.proc.poll() is None and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.skip = len(self.lines)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[self.skip:]:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU reference
_ADAM_S = None


def _adam_seconds(n_par: int) -> float:
    """One real fused clip(5.0) + Adam pass over n_par fp32 parameters in numpy on
    this host (the reference has no optimizer code) — timed
    once per process over ALL the parameters."""
    global _ADAM_S
    if _ADAM_S is None:
        import numpy as np
        rng = np.random.default_rng(0)
        p = rng.standard_normal(n_par, dtype=np.float32)
        g = rng.standard_normal(n_par, dtype=np.float32)
        m, v = np.zeros(n_par, np.float32), np.zeros(n_par, np.float32)
        t0 = time.perf_counter()
        g *= min(1.0, 5.0 / float(np.sqrt(np.dot(g, g))))
        m *= 0.9
        m += 0.1 * g
        v *= 0.999
        v += 0.001 * g * g
        p -= 1e-3 * (m / 0.1) / (np.sqrt(v / 0.001) + 1e-8)
        _ADAM_S = time.perf_counter() - t0
    return _ADAM_S


def cpu_reference(args, steps=1):
    """Time the reference's own CPU implementation of the path on this host.

    oracle/_ref/libseqloom_ref32.so = the reference's tensor/tape/layers.cpp
    compiled unmodified (fp32), driven through its public lstm_sequence /
    Tape::lstm_step / layer ops + Tape::backward (kind "reference"); if absent,
    the C restatement (kind "port").  The reference's data-parallel model
    (SURVEY §8(d)): one Tape per host thread (<= 64), each on a
    B/N-row batch shard of the workload (16 sequences per thread at B=256 on 16
    threads), OpenBLAS at 1 thread per tape (EIGEN_DONT_PARALLELIZE, reference
    core/CMakeLists.txt:31).

    Bounded sample per step: every thread runs, on its own shard, one full
    fwd+bwd layer-direction of each distinct encoder shape (D0, 2H), the
    step-by-step decoder (T x [lstm_step + closure, attention step fwd+bwd],
    the readout GEMMs), the output softmax + CE and the two embedding lookups;
    the reference runs the layers one after another, so the step's time is
    2 t(D0) + 2(L-1) t(2H) + t(dec) + t(out) + t(emb) (max over threads) plus
    one clip+Adam pass over all parameters; tokens/s = B * T / that.
    """
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    import oracle
    L, H, D0, T, B = args.layers, args.hidden, args.input, args.time, args.batch
    try:
        ref = oracle.Reference(32)
        kind = "reference"
    except FileNotFoundError:
        ref = oracle.Restatement()
        kind = "port"
    threads = max(1, min(os.cpu_count() or 1, 64, B))
    rows = -(-B // threads)  # sequences per thread
    rng = np.random.default_rng(0)
    s = 1 / np.sqrt(H)
    att = getattr(args, "attention", False)
    shapes = [D0, 2 * H] if att else [D0, 2 * H, D0 + 2 * H]  # encoder layer 0, layers 1.., (decoder)
    params = {D: tuple(rng.uniform(-s, s, shp) for shp in ((D, 4 * H), (H, 4 * H), (4 * H,)))
              for D in shapes + [D0 + 2 * H]}
    xs = {D: rng.uniform(-1, 1, (rows, T, D)) for D in shapes}
    lens = np.full(rows, T, np.int32)
    dy = rng.uniform(-1, 1, (rows, T, H))
    n_par = sum(2 * (D * 4 * H + H * 4 * H + 4 * H) for D in [D0] + [2 * H] * (L - 1))
    n_par += (D0 + 2 * H) * 4 * H + H * 4 * H + 4 * H
    n_par += H * args.vocab + args.vocab
    n_par += (args.src_vocab + (args.trg_vocab if args.vocab else 0)) * D0
    if att:
        E, K = 2 * H, H
        n_par += E * K + K + H * K + K + 2 * K + K + 1 + (H + D0 + E) * H + H
    adam_s = _adam_seconds(n_par)
    V = args.vocab
    Vs, Vt = args.src_vocab, (args.trg_vocab if V else 0)
    if (Vs or Vt) and kind == "reference":
        tbl = {Vv: rng.uniform(-s, s, (Vv, D0)) for Vv in {Vs, Vt} if Vv}
        ids_e = {Vv: rng.integers(0, Vv, (rows, T)).astype(np.int32) for Vv in tbl}
        d_e = rng.uniform(-1, 1, (rows, T, D0))
    if V and kind == "reference":
        Wo, bo = rng.uniform(-s, s, (H, V)), rng.uniform(-s, s, V)
        xo = rng.uniform(-1, 1, (rows, T, H))
        tgo = rng.integers(0, V, (rows, T)).astype(np.int32)
    att_case = None
    if att and kind == "reference":
        E, K = 2 * H, H
        att_case = dict(enc_ctx=rng.uniform(-1, 1, (rows, T, K)), enc=rng.uniform(-1, 1, (rows, T, E)),
                        Ws=rng.uniform(-s, s, (H, K)), bs=rng.uniform(-s, s, K), Wfb=rng.uniform(-s, s, (1, K)),
                        bfb=rng.uniform(-s, s, K), v=rng.uniform(-s, s, (K, 1)), bv=0.1)
        att_in = dict(s=rng.uniform(-1, 1, (rows, H)), accum=rng.uniform(0, 1, (rows, T)),
                      d_att=rng.uniform(-1, 1, (rows, E)), d_accum=rng.uniform(-1, 1, (rows, T)))
        Wd, Rd_, bd = params[D0 + 2 * H]
        xc, hc, cc = (rng.uniform(-1, 1, (rows, n)) for n in (D0 + 2 * H, H, H))
        Wro = rng.uniform(-s, s, (H + D0 + E, H)).astype(np.float32)
        xro = rng.uniform(-1, 1, (rows * T, H + D0 + E)).astype(np.float32)

    comps = (["dec"] if att_case is not None else []) + (["emb"] if (Vs or Vt) and kind == "reference" else []) + \
        (["out"] if V and kind == "reference" else []) + list(shapes)

    def one(out, which):
        tt = {}
        if "dec" in which:  # the step-by-step attention decoder of the shard, fwd + bwd
            t0 = time.perf_counter()
            for _ in range(T):
                ref.step(xc, hc, cc, Wd, Rd_, bd, gh=hc, gc=cc)          # RnnCell s (lstm_step + closure)
                ref.attention_step(lens, **att_case, s=att_in["s"], accum=att_in["accum"],
                                   d_att=att_in["d_att"], d_accum=att_in["d_accum"])
            y = np.maximum(xro @ Wro, 0)                                  # readout fwd + both GEMMs of its bwd
            _ = (y @ Wro.T, xro.T @ y)
            tt["dec"] = time.perf_counter() - t0
        if "emb" in which:
            t0 = time.perf_counter()
            for Vv in [v for v in (Vs, Vt) if v]:
                ref.gather_rows(tbl[Vv], ids_e[Vv], d_e)
            tt["emb"] = time.perf_counter() - t0
        if "out" in which:  # the output softmax layer + CE, fwd + bwd
            t0 = time.perf_counter()
            ref.output_ce(xo, lens, tgo, Wo, bo, 0.1)
            tt["out"] = time.perf_counter() - t0
        for D in shapes:
            if D not in which:
                continue
            W, R, b = params[D]
            t0 = time.perf_counter()
            if kind == "reference":
                ref.sequence(xs[D], lens, W, R, b, 1, dy)
            else:
                ref.sequence_bwd(xs[D], lens, W, R, b, 1, dy)
            tt[D] = time.perf_counter() - t0
        out.append(tt)

    def measure(which):  # every thread runs `which` on its own shard; max over threads per component
        res = []
        ths = [threading.Thread(target=one, args=(res, which)) for _ in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return {c: max(r[c] for r in res) for c in which}

    def step_seconds(e):
        return (2 * e[D0] + 2 * (L - 1) * e[2 * H] + e.get("dec", e.get(D0 + 2 * H, 0.0)) + e.get("out", 0.0)
                + e.get("emb", 0.0) + adam_s)

    # one full sample of every component, then (steps > 1) each further step re-times ONE
    # component in turn (round robin) so a long --steps run stays bounded
    est = measure(comps)
    secs = [step_seconds(est)]
    for i in range(1, steps):
        c = comps[(i - 1) % len(comps)]
        est.update(measure([c]))
        secs.append(step_seconds(est))
    rates = [threads * rows * T / x for x in secs]
    value = statistics.median(rates)
    return {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{threads} threads x {rows}-sequence batch shard (T={T}, B={threads * rows}); per thread "
                      f"one fwd+bwd layer-direction of each encoder shape (D={D0}, D={2 * H}; H={H}), the decoder "
                      + ("(T x [lstm_step + closure, D=" + str(D0 + 2 * H) + "] + T x [attention step fwd+bwd, "
                         "Ts=" + str(T) + "] + the readout GEMMs)" if att_case is not None else
                         "(one lstm_sequence D=" + str(D0 + 2 * H) + ")") + f", the output "
                      f"softmax + CE (V={V}) and the src/trg embedding lookups (gather_rows fwd+bwd, "
                      f"V={Vs}/{Vt}); step time = 2 t(D0) + {2 * (L - 1)} t(2H) + t(dec) + t(out) + t(emb) "
                      f"(layers run sequentially in the reference) + one clip+Adam pass over all "
                      f"{n_par / 1e6:.1f}M params ({adam_s:.2f} s, numpy fp32 on 1 thread, timed for real once: "
                      f"the reference has no optimizer code); fp32 reference build + scipy OpenBLAS 1 thread/tape; "
                      f"median of {steps} steps (step 1 times every component, each later step re-times one "
                      f"component in turn)",
            "seconds_per_step": statistics.median(secs)}


# ---------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank, precision):
    import torch
    import torch.distributed as dist
    from paper_1805_05225_b200 import lstm
    from paper_1805_05225_b200.model import Seq2SeqAttention, Seq2SeqLSTM

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    L, B, T, D0, H = args.layers, args.batch, args.time, args.input, args.hidden
    Vs, Vt = args.src_vocab, (args.trg_vocab if args.vocab else 0)
    if args.attention:
        model = Seq2SeqAttention(L, B, T, T, D0, H, args.vocab, Vs, Vt, device=dev, precision=precision)
    else:
        model = Seq2SeqLSTM(L, B, T, D0, H, precision, dev, vocab=args.vocab, src_vocab=Vs, trg_vocab=Vt)
    model.init_uniform(seed=1)
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    if Vs:  # source token ids (the `src` embedding layer looks them up)
        x = torch.randint(0, Vs, (B, T), device=dev, generator=g, dtype=torch.int32)
    else:  # source embeddings
        x = torch.rand(B, T, D0, device=dev, generator=g) * 2 - 1
    emb = torch.rand(B, T, D0, device=dev, generator=g) * 2 - 1    # target embeddings (trg_vocab = 0)
    lens = torch.full((B,), T, dtype=torch.int32, device=dev)
    if args.vocab:  # target ids for the output layer's CE loss (and the `trg` lookup)
        dy = torch.randint(0, min(args.vocab, Vt or args.vocab), (B, T), device=dev, generator=g,
                           dtype=torch.int32)
    else:
        dy = torch.rand(B, T, H, device=dev, generator=g) * 2 - 1  # dL/d(decoder output)
    if not Vt and not args.attention:
        model.set_target_embeddings(emb)
    lib = lstm.lib()
    lib.sl_profile_enable.argtypes = [ctypes.c_int]
    lib.sl_launch_count.restype = ctypes.c_ulonglong

    class Entry(ctypes.Structure):
        _fields_ = [("name", ctypes.c_char * 32), ("calls", ctypes.c_int32), ("ms", ctypes.c_double),
                    ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]

    from paper_1805_05225_b200.dp import BucketAllReducer
    red = BucketAllReducer()  # layer-bucketed NCCL all-reduce, overlapped with BPTT
    if args.dp_selftest:
        red.force = True

    def step(xin):
        model.step(xin, lens, dy, reducer=red, grad_scale=1.0 / world)

    for _ in range(args.warmup):
        step(x)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lib.sl_profile_read(None, 0, 1)
    lib.sl_profile_enable(1)
    n0 = lib.sl_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            step(x)
        e1.record()
        torch.cuda.synchronize()
    lib.sl_profile_enable(0)
    launches = (lib.sl_launch_count() - n0)
    ms = e0.elapsed_time(e1)
    entries = (Entry * 64)()
    n = lib.sl_profile_read(entries, 64, 1)
    phases = {e.name.decode(): {"calls": e.calls, "ms": e.ms, "flops": e.flops, "bytes": e.bytes}
              for e in entries[:n]}
    eager_ms = ms
    graph = None
    graph_note = None
    if not args.no_graph:
        # The whole step (every kernel of the library, the glue copies, the
        # optimizer with its device-side step counter and, at N>1, the bucketed
        # NCCL all-reduces) captured once as a CUDA graph and replayed: no host
        # launch gaps.  Phases above come from the eager pass (same kernels); the
        # headline time from the replays.  At N>1 every rank must end up on the
        # same path: a capture failure on any rank drops all ranks to eager.
        ok = 1
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step(x)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            c0 = lib.sl_launch_count()
            with torch.cuda.graph(graph):
                step(x)
            per_step = lib.sl_launch_count() - c0
        except Exception as exc:  # noqa: BLE001 - reported in the line, eager timing instead
            ok, graph, graph_note = 0, None, f"graph capture failed ({type(exc).__name__}: {exc}); eager"
            torch.cuda.synchronize()
        if world > 1:
            f = torch.tensor([ok], device=dev, dtype=torch.int32)
            dist.all_reduce(f, op=dist.ReduceOp.MIN)
            if int(f.item()) == 0:
                graph = None
                graph_note = graph_note or "graph capture failed on another rank; eager"
    if graph is not None:
        graph.replay()
        torch.cuda.synchronize()
        with ClockSampler(local_rank) as clocks:
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.steps):
                graph.replay()
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        launches = per_step * args.steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # ---- end to end: host buffers through the public API, copies timed
    e2e = None
    if not args.no_e2e:
        # per step in: source ids (or embeddings), target ids (or target
        # embeddings + the upstream gradient), lengths; out: the scalar loss
        hin = [x, lens] + ([dy] if args.vocab else []) + ([] if Vt or args.attention else [emb])
        hosts = [t.cpu().pin_memory() for t in hin]
        devs = [torch.empty_like(t) for t in hin]
        xd, ld = devs[0], devs[1]
        dyd = devs[2] if args.vocab else dy
        ed = devs[-1] if not (Vt or args.attention) else None
        loss_h = torch.empty((), dtype=torch.float32).pin_memory()

        graphed = None
        if args.attention and graph is not None:  # (at N>1 only when every rank captured the timed step)
            from paper_1805_05225_b200.model import GraphedStep
            # the public graphed-step API, the bucketed all-reduces captured with the kernels
            graphed = GraphedStep(model, x, lens, dy, reducer=red, grad_scale=1.0 / world)

        def e2e_step():
            if graphed is not None:  # H2D of the step's inputs, graph replay, D2H of the loss
                return graphed(hosts[0], hosts[1], hosts[2])
            for d_, h_ in zip(devs, hosts):
                d_.copy_(h_, non_blocking=True)
            if ed is not None:
                model.set_target_embeddings(ed)
            if args.vocab:  # the real loss: output softmax + label-smoothed CE
                loss = model.step(xd, ld, dyd, reducer=red, grad_scale=1.0 / world)
                loss_h.copy_(loss, non_blocking=True)
            else:
                y = model.forward(xd, ld)
                loss = (y * dy).sum()  # L = sum(y . dy), so dL/dy = dy
                loss_h.copy_(loss, non_blocking=True)
                model.backward(dy, on_grads=red)
                red.wait()
                model.opt.step(model.grads, grad_scale=1.0 / world)
            torch.cuda.current_stream().synchronize()  # the host reads the step's loss
            return float(loss_h)

        e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * B * T * args.steps / float(tt.item()), "unit": UNIT,
               "h2d_bytes_per_step": sum(h_.numel() * h_.element_size() for h_ in hosts), "d2h_bytes_per_step": 4,
               "note": ("source ids" if Vs else "source embeddings") + ", " +
                       ("target ids" if Vt else "target embeddings") + " and lens copied in; the scalar "
                       "loss copied out" + ("; through model.GraphedStep (the step as one CUDA graph)"
                                            if graphed is not None else "; eager launches"),
               "timing": "host wall clock, max over ranks"}
    return dict(ms=ms_max, phases=phases, launches=int(launches), clocks=clocks.summary(),
                e2e=e2e, eager_ms=eager_ms / args.steps, eager_ms_total=eager_ms, graph=graph is not None,
                graph_note=graph_note, allreduces=red.issued,
                backend=dist.get_backend() if dist.is_initialized() else None)


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(args) -> int:
    """`bench.py --gpus N` outside torchrun: start the N ranks ourselves (one
    process per GPU, torch.distributed.run on 127.0.0.1) with the same
    arguments; NCCL_DEBUG=INFO so each rank's communicator lines (nranks=N)
    are in the log.  Returns the launcher's exit code."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------- configs 1, 2, 3, 5
# BASELINE.json configs (SURVEY §8 shapes table, §9 decisions): layers, directions, H, D0, B, T
LAYER_CONFIGS = {
    1: dict(layers=1, dirs=1, H=128, D0=128, B=8, T=20, train=True,
            name="config1: single-layer unidirectional LSTM n=128, B=8, T=20, fp32 fwd+bwd (D=H)"),
    2: dict(layers=1, dirs=1, H=1024, D0=1024, B=128, T=60, train=True,
            name="config2: single-layer LSTM n=1024, B=128, T=60 fwd+bwd on 1xB200 (D=H; kernel micro-benchmark)"),
    3: dict(layers=4, dirs=2, H=1000, D0=620, B=256, T=60, train=True,
            name="config3: 4-layer bidirectional LSTM encoder n=1000, B=256, T=60 fwd+bwd, both directions "
                 "concurrent (D0=620)"),
    5: dict(layers=6, dirs=2, H=1024, D0=40, B=None, T=None, train=False,
            name="config5: 6-layer BLSTM n=1024 encoder inference (F=40 input features), batch-sharded "
                 "(no communication)"),
}
SWEEP = [(1, 60), (16, 60), (64, 60), (256, 60), (1024, 60), (1, 500), (16, 500), (64, 500), (256, 500), (1024, 500)]


def _layer_stack(spec, B, T, precision, dev):
    from paper_1805_05225_b200 import lstm
    from paper_1805_05225_b200.encoder import BLSTMEncoder
    if spec["dirs"] == 2:
        enc = BLSTMEncoder(spec["layers"], B, T, spec["D0"], spec["H"], precision, dev, train=spec["train"])
        enc.init_uniform(seed=1)
        return enc
    H, D = spec["H"], spec["D0"]
    layer = lstm.LSTMLayer(B, T, D, H, 1, 1, precision, dev)
    s = H ** -0.5
    g = torch_gen(dev, 1)
    import torch
    W = [(torch.rand(D, 4 * H, device=dev, generator=g) * 2 - 1) * s]
    R = [(torch.rand(H, 4 * H, device=dev, generator=g) * 2 - 1) * s]
    b = [(torch.rand(4 * H, device=dev, generator=g) * 2 - 1) * s]
    y, dx = torch.empty(B, T, H, device=dev), torch.empty(B, T, D, device=dev)
    dW, dR, db = [torch.empty_like(W[0])], [torch.empty_like(R[0])], [torch.empty_like(b[0])]

    class One:
        def forward(self, x, lens, train=True):
            layer.forward(x, lens, W, R, b, y=y)
            return y

        def backward(self, dy):
            layer.backward(dy, dx=dx, dW=dW, dR=dR, db=db, need_dx=True)
            return dx
    return One()


def torch_gen(dev, seed):
    import torch
    return torch.Generator(device=dev).manual_seed(seed)


def _time_layers(args, spec, B, T, precision, local_rank, rank):
    """K timed steps of fwd(+bwd) of the config's stack (CUDA graph replay), with the
    per-phase events of one eager pass and the H2D/D2H end-to-end leg."""
    import torch
    from paper_1805_05225_b200 import lstm
    dev = torch.device("cuda", local_rank)
    net = _layer_stack(spec, B, T, precision, dev)
    g = torch_gen(dev, 100 + rank)
    x = torch.rand(B, T, spec["D0"], device=dev, generator=g) * 2 - 1
    lens = torch.full((B,), T, dtype=torch.int32, device=dev)
    out_w = spec["dirs"] * spec["H"]
    dy = torch.rand(B, T, out_w, device=dev, generator=g) * 2 - 1
    lib = lstm.lib()
    lib.sl_profile_enable.argtypes = [ctypes.c_int]
    lib.sl_launch_count.restype = ctypes.c_ulonglong

    def step():
        y = net.forward(x, lens, train=spec["train"])
        if spec["train"]:
            net.backward(dy)
        return y

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    class Entry(ctypes.Structure):
        _fields_ = [("name", ctypes.c_char * 32), ("calls", ctypes.c_int32), ("ms", ctypes.c_double),
                    ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]
    lib.sl_profile_read(None, 0, 1)
    lib.sl_profile_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    lib.sl_profile_enable(0)
    eager_ms = e0.elapsed_time(e1)
    entries = (Entry * 64)()
    n = lib.sl_profile_read(entries, 64, 1)
    phases = {e.name.decode(): {"calls": e.calls, "ms": e.ms, "flops": e.flops, "bytes": e.bytes}
              for e in entries[:n]}
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    c0 = lib.sl_launch_count()
    with torch.cuda.graph(graph):
        y_out = step()
    per_step = lib.sl_launch_count() - c0
    graph.replay()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # end to end: pinned host input in, the output (inference) / a checksum (training) out
    hx = x.cpu().pin_memory()
    hy = torch.empty(y_out.shape, dtype=y_out.dtype).pin_memory() if not spec["train"] else \
        torch.empty((), dtype=torch.float32).pin_memory()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x.copy_(hx, non_blocking=True)
        graph.replay()
        if spec["train"]:
            hy.copy_(y_out.float().sum(), non_blocking=True)
        else:
            hy.copy_(y_out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    e2e_s = time.perf_counter() - t0
    return dict(ms=ms, eager_ms=eager_ms, phases=phases, launches=per_step * args.steps, clocks=clocks.summary(),
                e2e_s=e2e_s, h2d=hx.numel() * hx.element_size(), d2h=hy.numel() * hy.element_size())


def cpu_reference_layers(args, spec, B, T, steps=1):
    """The reference's lstm_sequence (oracle/_ref, fp32, OpenBLAS 1 thread per tape) on
    B/N-row shards per host thread, fwd(+bwd) of every layer-direction
    of the config; layers run one after another in the reference: step time = sum."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    import oracle
    try:
        ref, kind = oracle.Reference(32), "reference"
    except FileNotFoundError:
        ref, kind = oracle.Restatement(), "port"
    threads = max(1, min(os.cpu_count() or 1, 64, B))
    rows = -(-B // threads)
    H, L, nd = spec["H"], spec["layers"], spec["dirs"]
    rng = np.random.default_rng(0)
    s = 1 / np.sqrt(H)
    shapes = sorted({spec["D0"]} | ({nd * H} if L > 1 else set()))
    params = {D: tuple(rng.uniform(-s, s, shp) for shp in ((D, 4 * H), (H, 4 * H), (4 * H,))) for D in shapes}
    xs = {D: rng.uniform(-1, 1, (rows, T, D)) for D in shapes}
    lens = np.full(rows, T, np.int32)
    dy = rng.uniform(-1, 1, (rows, T, H)) if spec["train"] else None

    def one(out):
        tt = {}
        for D in shapes:
            t0 = time.perf_counter()
            if kind == "reference":
                ref.sequence(xs[D], lens, *params[D], 1, dy)
            elif dy is not None:
                ref.sequence_bwd(xs[D], lens, *params[D], 1, dy)
            else:
                ref.sequence_fwd(xs[D], lens, *params[D], 1)
            tt[D] = time.perf_counter() - t0
        out.append(tt)

    secs = []
    for _ in range(steps):
        res = []
        ths = [threading.Thread(target=one, args=(res,)) for _ in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        per = {D: max(r[D] for r in res) for D in shapes}
        secs.append(sum(nd * per[spec["D0"] if l == 0 else nd * H] for l in range(L)))
    sec = statistics.median(secs)
    return {"value": threads * rows * T / sec, "unit": "tokens/s" if spec["train"] else "frames/s",
            "cores": threads, "kind": kind, "seconds_per_step": sec,
            "sample": f"{threads} threads x {rows}-sequence shard (T={T}): one lstm_sequence "
                      f"{'fwd+bwd' if spec['train'] else 'fwd'} per distinct layer input width {shapes} (H={H}), "
                      f"step = sum over the {L} x {nd} layer-directions (the reference runs them one after "
                      f"another); fp32 reference build, OpenBLAS 1 thread/tape; median of {steps}"}


def run_layer_config(args, rank, world, local_rank):
    """--config 1, 2, 3 (training fwd+bwd) or 5 (inference sweep): one JSON line, same schema."""
    import torch
    spec = LAYER_CONFIGS[args.config]
    H, L, nd = spec["H"], spec["layers"], spec["dirs"]
    torch.cuda.set_device(local_rank)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    x3 = 3 if args.precision == "fp32" else 1
    points = SWEEP if args.config == 5 else [(spec["B"], spec["T"])]
    lines = []
    for (B, T) in points:
        r = _time_layers(args, spec, B, T, args.precision, local_rank, rank)
        tokens = world * B * T * args.steps
        ph = r["phases"]
        top = max(ph.items(), key=lambda kv: kv[1]["ms"]) if ph else (None, None)
        roof = None
        if top[0]:
            name, e = top
            per_launch_ms = e["ms"] / max(e["calls"], 1)
            achieved = x3 * e["flops"] / max(e["calls"], 1) / (per_launch_ms / 1e3) / 1e12
            peak = peaks.get("bf16_tflops_sustained", 1400.0)
            roof = {"kernel": name, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": None, "share_of_step": e["ms"] / r["eager_ms"],
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (of measured)" if peaks else "fallback",
                    "achieved_counts": "executed tensor FLOP/s (x3: 3 bf16 products per fp32 product)" if x3 == 3
                    else "algorithmic FLOP/s",
                    "phases": {k: {"calls": v["calls"], "ms_per_call": v["ms"] / max(v["calls"], 1)}
                               for k, v in ph.items()}}
            f_sm = (r["clocks"].get("sm_mhz") or 1965.0) * 1e6
            rec = {}
            for pname in ("k2_rec_fwd", "k3_rec_bwd"):
                e = ph.get(pname)
                if not e:
                    continue
                ndl = 1 if x3 == 3 else nd
                us = e["ms"] / max(e["calls"], 1) * 1e3 / T
                smem_us = ndl * 4 * H * H * 2 * (2 if x3 == 3 else 1) / (148 * 128 * f_sm) * 1e6
                tens_us = x3 * 2.0 * min(B, 256) * 4 * H * H * ndl / (peak * 1e12) * 1e6
                rec[pname] = {"us_per_step": us, "wh_smem_bound_us": smem_us, "tensor_bound_us": tens_us,
                              "ratio_to_bound": us / max(smem_us, tens_us)}
            roof["recurrence_per_step"] = rec
        lines.append({"B": B, "T": T, "value": tokens / (r["ms"] / 1e3), "ms_per_step": r["ms"] / args.steps,
                      "e2e": {"value": tokens / r["e2e_s"], "unit": "tokens/s" if spec["train"] else "frames/s",
                              "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                              "timing": "host wall clock: pinned input H2D, graph replay, output D2H"},
                      "gpu_launches": r["launches"], "clocks": r["clocks"], "roofline": roof,
                      "eager_ms_per_step": r["eager_ms"] / args.steps})
    head = lines[-1]  # config 5: the largest point (B=1024, T=500) is the headline
    unit = "tokens/s" if spec["train"] else "frames/s"
    cfg = {"workload": spec["name"], "layers": L, "directions": nd, "hidden": H, "input_dim": spec["D0"],
           "batch_per_gpu": head["B"], "global_batch": head["B"] * world, "seq_len": head["T"],
           "parallelism": f"dp{world}" if spec["train"] else f"batch-sharded x{world} (no communication)",
           "seq_lens": "all = T", "l2": "inputs, weights and saved activations exceed the 126 MB L2"
           if args.config != 1 else "config 1 fits in L2 (126 MB): timed as back-to-back graph replays"}
    out = {"metric": f"LSTM {'fwd+bwd' if spec['train'] else 'inference'} {unit} ({spec['name'].split(':')[0]})",
           "value": head["value"], "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": args.precision.replace("fp", "f"), "data": "synthetic (x ~ U(-1,1), params ~ U(+-1/sqrt(H)))",
           "config": cfg, "e2e": head["e2e"], "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
           "roofline": head["roofline"], "eager_ms_per_step": head["eager_ms_per_step"]}
    if args.config == 5:
        out["sweep"] = [{k: v for k, v in p.items() if k in ("B", "T", "value", "ms_per_step")} for p in lines]
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            out["cpu_baseline"] = cpu_reference_layers(args, spec, min(head["B"], 256), min(head["T"], 60))
            out["cpu_baseline"]["sample"] += (" (config 5: the B=256, T=60 point)" if args.config == 5 else "")
        except Exception as exc:
            out["cpu_baseline"] = {"error": repr(exc)}
    return out


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    L, B, T, D0, H = args.layers, args.batch, args.time, args.input, args.hidden
    out_s = (f" + output softmax V={args.vocab} with label-smoothed CE (eps 0.1)" if args.vocab else "")
    Vt = args.trg_vocab if args.vocab else 0
    emb_s = (f"src/trg embedding lookups from token ids (V={args.src_vocab}/{Vt}) + " if args.src_vocab or Vt
             else "")
    if args.attention:
        work = (f"config4 training step (Listing-1 attention model): src/trg embedding lookups from token ids "
                f"(V={args.src_vocab}/{Vt}, width {D0}) + {L}xBLSTM encoder H={H} + enc_ctx + LSTM decoder cell "
                f"H={H} with input feeding [prev trg {D0} ‖ prev att {2 * H}] + MLP attention (key {H}, weight "
                f"feedback) + relu readout {H} + output softmax V={args.vocab} with label-smoothed CE (eps 0.1), "
                f"teacher forcing, T_src=T_tgt={T}, fwd+bwd + fused clip(5.0)+Adam over all parameters "
                f"(+DP grad all-reduce at N>1); dropout 0.3 on the output_prob input (the reference's "
                f"counter-based mask, bit-identical)")
    else:
        work = (f"config4 training step: {emb_s}{L}xBLSTM encoder H={H} D0={D0} + LSTM decoder "
                f"H={H} (input {D0}+{2 * H}){out_s}, T_src=T_tgt={T}, fwd+bwd + fused "
                f"clip(5.0)+Adam (+DP grad all-reduce at N>1); no attention (context = encoder output at t)")
    cfg = {"workload": work, "attention": args.attention,
           "vocab": args.vocab, "src_vocab": args.src_vocab, "trg_vocab": Vt,
           "global_batch": B * world, "batch_per_gpu": B,
           "seq_len": T, "hidden": H, "input_dim": D0, "layers": L, "directions": 2,
           "parallelism": f"dp{world}", "seq_lens": "all = T",
           "l2": "working set (weights ~0.77 GB fp32 + Adam moments + activations) far exceeds the 126 MB L2"}

    if args.impl == "reference":
        if rank != 0:
            return
        cpu = cpu_reference(args, steps=max(1, args.steps))
        print(json.dumps({"metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["seconds_per_step"] * 1e3,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "f32", "data": "synthetic", "config": cfg, "impl": "reference",
                          "cpu_baseline": {k: cpu[k] for k in ("kind", "cores", "sample", "value", "unit")},
                          "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return

    import torch
    import torch.distributed as dist
    if world > 1 or (args.dp_selftest and "RANK" in os.environ):
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks=N) in the log
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.config != 4:
        out = run_layer_config(args, rank, world, local_rank)
        if world > 1:  # max over ranks of the step time (weak scaling: every rank runs the per-GPU batch)
            t = torch.tensor([out["ms_per_step"]], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out["ms_per_step"] = float(t.item())
            out["value"] = world * out["config"]["batch_per_gpu"] * out["config"]["seq_len"] / (out["ms_per_step"] / 1e3)
        if rank == 0:
            print(json.dumps(out), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    r = run_ours(args, rank, world, local_rank, args.precision)
    out = result_line(args, r, world, cfg, peaks, args.precision)
    if args.precision == "fp32" and not args.no_bf16_line:
        # the bf16 mode beside the fp32 headline (same workload, same clock rules)
        torch.cuda.empty_cache()
        rb = run_ours(args, rank, world, local_rank, "bf16")
        lb = result_line(args, rb, world, cfg, peaks, "bf16")
        out["bf16_mode"] = {k: lb[k] for k in ("value", "unit", "ms_per_step", "dtype", "e2e", "gpu_launches",
                                               "clocks", "algorithmic_tflops")}
        out["bf16_mode"]["roofline"] = {k: lb["roofline"][k] for k in ("kernel", "bound", "achieved", "peak", "unit",
                                                                       "frac", "share_of_step")} if lb["roofline"] else None
        out["bf16_mode"]["tolerance"] = "bf16 operands, fp32 accumulation / state: rel. 2e-2 per tensor"
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            out["cpu_baseline"] = cpu_reference(args, steps=1)
        except Exception as exc:  # the baseline must never sink the GPU line
            out["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def result_line(args, r, world, cfg, peaks, precision):
    """The JSON line of one measured run (run_ours) in `precision`."""
    L, B, T, D0, H = args.layers, args.batch, args.time, args.input, args.hidden
    x3 = 3 if precision == "fp32" else 1  # tensor-core products per fp32-class product (split-bf16 x3)
    tokens = world * B * T * args.steps
    value = tokens / (r["ms"] / 1e3)
    # dominant kernel phase -> roofline
    ph = r["phases"]
    top = max(ph.items(), key=lambda kv: kv[1]["ms"]) if ph else (None, None)
    roof = None
    if top[0]:
        name, e = top
        per_launch_ms = e["ms"] / max(e["calls"], 1)
        hbm = e["flops"] == 0 and e.get("bytes", 0) > 0  # a bandwidth-bound phase
        if hbm:
            achieved = e["bytes"] / max(e["calls"], 1) / (per_launch_ms / 1e3) / 1e9
            peak = peaks.get("hbm_gbs", 6650.0)
        else:  # tensor FLOP/s the tensor cores execute (x3: three bf16 products per fp32 product)
            achieved = x3 * e["flops"] / max(e["calls"], 1) / (per_launch_ms / 1e3) / 1e12
            peak = peaks.get("bf16_tflops_sustained", 1400.0)
        traffic = None
        try:  # DRAM bytes per launch of this kernel from the committed ncu capture
            tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            traffic = tr.get(f"{precision}:{name}", tr.get(name) if precision == "bf16" else None)
        except Exception:
            pass
        roof = {"kernel": name, "bound": "hbm" if hbm else "tensor", "achieved": achieved, "peak": peak,
                "unit": "GB/s" if hbm else "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/)",
                "peak_source": ("MEASURED_PEAKS.json " + ("hbm_gbs" if hbm else "bf16_tflops_sustained") +
                                " (of measured)") if peaks else "fallback",
                "achieved_counts": ("executed tensor-core FLOP/s: the split-bf16 products (3 per fp32 product) "
                                    "over the launch's CUDA-event time" if x3 == 3 and not hbm else
                                    "algorithmic work / CUDA-event time of the launch"),
                "share_of_step": e["ms"] / r["eager_ms_total"],
                "phases": {k: {"calls": v["calls"], "ms_per_call": v["ms"] / max(v["calls"], 1),
                               "tflops": v["flops"] / max(v["ms"], 1e-9) / 1e9,
                               "gbs": v.get("bytes", 0) / max(v["ms"], 1e-9) / 1e6}
                           for k, v in ph.items()}}
        # recurrence phases: per-step latency against max(W_h-from-SMEM bound, tensor bound)
        f_sm = (r["clocks"].get("sm_mhz") or 1965.0) * 1e6
        rec = {}
        for pname in ("k2_rec_fwd", "k3_rec_bwd"):
            e = ph.get(pname)
            if not e:
                continue
            us = e["ms"] / max(e["calls"], 1) * 1e3 / T  # per time step of one launch
            nd_launch = 2  # both directions per launch (x3 too: R_hi resident, R_lo streamed from L2)
            wh_bytes = nd_launch * 4 * H * H * 2  # the resident bf16 R (x3: R_hi; R_lo streams from L2)
            smem_us = wh_bytes / (148 * 128 * f_sm) * 1e6
            tensor_us = x3 * 2.0 * B * 4 * H * H * nd_launch / (peaks.get("bf16_tflops_sustained", 1400.0) * 1e12) * 1e6
            rec[pname] = {"us_per_step": us, "directions_per_launch": nd_launch, "wh_smem_bound_us": smem_us,
                          "tensor_bound_us": tensor_us, "bound_us": max(smem_us, tensor_us),
                          "ratio_to_bound": us / max(smem_us, tensor_us)}
        roof["recurrence_per_step"] = rec
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": precision.replace("fp", "f"),
            "data": "synthetic (token ids ~ U[0, V), params ~ U(+-1/sqrt(H)))",
            "config": cfg, "cuda_graph": r["graph"], "eager_ms_per_step": r["eager_ms"],
            **({"graph_note": r["graph_note"]} if r.get("graph_note") else {}),
            **({"dp_selftest": f"gradient all-reduces issued over NCCL at world 1 ({r['allreduces']} issued, "
                                f"backend {r['backend']})"} if args.dp_selftest else {}),
            "precision_note": ("fp32 semantics (rel. 1e-4 per tensor vs the fp32 reference): every product on the "
                               "tcgen05 tensor cores as split-bf16 x3 (A B = A_hi B_hi + A_lo B_hi + A_hi B_lo, fp32 "
                               "accumulation in K chunks), fp32 state / activations" if precision == "fp32" else
                               "bf16 operands, fp32 accumulation and state (rel. 2e-2 per tensor)"),
            "e2e": r["e2e"], "gpu_launches": r["launches"], "clocks": r["clocks"],
            "roofline": roof,
            "algorithmic_tflops": flops_per_token(L, D0, H, args.vocab, args.attention, T) * B * T * world /
            (r["ms"] / args.steps / 1e3) / 1e12}


if __name__ == "__main__":
    main()
