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
    ap.add_argument("--precision", choices=["fp32", "bf16"], default=os.environ.get("SL_BENCH_PREC", "bf16"))
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
    a = ap.parse_args()
    a.attention = not a.no_attention
    if a.attention and not (a.vocab and a.src_vocab and a.trg_vocab and a.precision == "bf16"):
        ap.error("the attention step needs --vocab, --src-vocab, --trg-vocab > 0 and bf16 (or --no-attention)")
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

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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
        for ln in self.lines:
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
def cpu_reference(args, steps=1):
    """Time the reference's own CPU implementation of the path on this host.

    oracle/_ref/libseqloom_ref32.so = the reference's tensor/tape/layers.cpp
    compiled unmodified, driven through its public lstm_sequence + Tape::backward
    (kind "reference"); if absent, the C restatement (kind "port").  Threads =
    host cores (<= 64), each with its own Tape on a one-sequence batch shard (the
    reference's data-parallel model); OpenBLAS at 1 thread per tape
    (EIGEN_DONT_PARALLELIZE, reference core/CMakeLists.txt:31).

    Bounded sample: the reference runs layers one after another, so one
    sequence through the full 6xBLSTM stack costs 2 t(D0) + 2(L-1) t(2H), where
    t(D) is one layer-direction fwd+bwd with input width D.  Each step times
    one layer-direction of each distinct shape per thread (~10 s) and reports
    threads * T / (2 t(D0) + 2 (L-1) t(2H)).
    """
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    import oracle
    L, H, D0, T = args.layers, args.hidden, args.input, args.time
    try:
        ref = oracle.Reference(32)
        kind = "reference"
    except FileNotFoundError:
        ref = oracle.Restatement()
        kind = "port"
    threads = max(1, min(os.cpu_count() or 1, 64))
    rng = np.random.default_rng(0)
    s = 1 / np.sqrt(H)
    shapes = [D0, 2 * H, D0 + 2 * H]  # encoder layer 0, encoder layers 1.., decoder
    params = {D: tuple(rng.uniform(-s, s, shp) for shp in ((D, 4 * H), (H, 4 * H), (4 * H,)))
              for D in shapes}
    xs = {D: rng.uniform(-1, 1, (1, T, D)) for D in shapes}
    lens = np.full(1, T, np.int32)
    dy = rng.uniform(-1, 1, (1, T, H))
    times = []
    # optimizer step on the host: all LSTM parameters, timed on a slice
    n_par = sum(2 * (D * 4 * H + H * 4 * H + 4 * H) for D in [D0] + [2 * H] * (L - 1))
    n_par += (D0 + 2 * H) * 4 * H + H * 4 * H + 4 * H
    n_par += H * args.vocab + args.vocab  # output softmax layer
    n_par += (args.src_vocab + (args.trg_vocab if args.vocab else 0)) * D0  # embedding tables
    k = 4_000_000
    pa, ga = rng.standard_normal(k).astype(np.float32), rng.standard_normal(k).astype(np.float32)
    ma, va = np.zeros(k, np.float32), np.zeros(k, np.float32)
    t0 = time.perf_counter()
    nrm = np.sqrt(np.dot(ga, ga))
    ga *= min(1.0, 5.0 / nrm)
    ma *= 0.9
    ma += 0.1 * ga
    va *= 0.999
    va += 0.001 * ga * ga
    pa -= 1e-3 * (ma / 0.1) / (np.sqrt(va / 0.001) + 1e-8)
    adam_s = (time.perf_counter() - t0) * n_par / k

    V = args.vocab
    Vs, Vt = args.src_vocab, (args.trg_vocab if V else 0)
    if (Vs or Vt) and kind == "reference":  # embedding lookups of one sequence, fwd + bwd
        tbl = {Vv: rng.uniform(-s, s, (Vv, D0)) for Vv in {Vs, Vt} if Vv}
        ids_e = {Vv: rng.integers(0, Vv, (1, T)).astype(np.int32) for Vv in tbl}
        d_e = rng.uniform(-1, 1, (1, T, D0))
    if V and kind == "reference":
        Wo = rng.uniform(-s, s, (H, V))
        bo = rng.uniform(-s, s, V)
        xo = rng.uniform(-1, 1, (1, T, H))
        tgo = rng.integers(0, V, (1, T)).astype(np.int32)

    att_case = None
    if getattr(args, "attention", False) and kind == "reference":
        E, K = 2 * H, H
        att_case = dict(enc_ctx=rng.uniform(-1, 1, (1, T, K)), enc=rng.uniform(-1, 1, (1, T, E)),
                        Ws=rng.uniform(-s, s, (H, K)), bs=rng.uniform(-s, s, K), Wfb=rng.uniform(-s, s, (1, K)),
                        bfb=rng.uniform(-s, s, K), v=rng.uniform(-s, s, (K, 1)), bv=0.1)
        att_in = dict(s=rng.uniform(-1, 1, (1, H)), accum=rng.uniform(0, 1, (1, T)),
                      d_att=rng.uniform(-1, 1, (1, E)), d_accum=rng.uniform(-1, 1, (1, T)))
        Wd, Rd_, bd = params[D0 + 2 * H]
        xc, hc, cc = rng.uniform(-1, 1, (1, D0 + 2 * H)), rng.uniform(-1, 1, (1, H)), rng.uniform(-1, 1, (1, H))
        Wro = rng.uniform(-s, s, (H + D0 + E, H)).astype(np.float32)
        xro = rng.uniform(-1, 1, (T, H + D0 + E)).astype(np.float32)

    def one(out):
        tt = {}
        if att_case is not None:  # the step-by-step attention decoder of one sequence, fwd + bwd
            t0 = time.perf_counter()
            for _ in range(T):
                ref.step(xc, hc, cc, Wd, Rd_, bd, gh=hc, gc=cc)          # RnnCell s (lstm_step + closure)
                ref.attention_step(lens, **att_case, s=att_in["s"], accum=att_in["accum"],
                                   d_att=att_in["d_att"], d_accum=att_in["d_accum"])
            y = np.maximum(xro @ Wro, 0)                                  # readout fwd + both GEMMs of its bwd
            _ = (y @ Wro.T, xro.T @ y)
            tt["dec"] = time.perf_counter() - t0
        if (Vs or Vt) and kind == "reference":
            t0 = time.perf_counter()
            for Vv in [v for v in (Vs, Vt) if v]:
                ref.gather_rows(tbl[Vv], ids_e[Vv], d_e)
            tt["emb"] = time.perf_counter() - t0
        if V and kind == "reference":  # the output softmax layer + CE, fwd + bwd
            t0 = time.perf_counter()
            ref.output_ce(xo, lens, tgo, Wo, bo, 0.1)
            tt["out"] = time.perf_counter() - t0
        for D in (shapes[:2] if att_case is not None else shapes):
            W, R, b = params[D]
            t0 = time.perf_counter()
            if kind == "reference":
                ref.sequence(xs[D], lens, W, R, b, 1, dy)
            else:
                ref.sequence_bwd(xs[D], lens, W, R, b, 1, dy)
            tt[D] = time.perf_counter() - t0
        out.append(tt)

    rates = []
    for _ in range(steps):
        res = []
        ths = [threading.Thread(target=one, args=(res,)) for _ in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        per_seq = [2 * r[D0] + 2 * (L - 1) * r[2 * H] + r.get("dec", r.get(D0 + 2 * H, 0.0)) + r.get("out", 0.0)
                   + r.get("emb", 0.0) for r in res]
        rates.append(threads * T / (max(per_seq) + adam_s))
    value = statistics.median(rates)
    return {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{threads} threads x 1 sequence (T={T}); per thread one fwd+bwd layer-direction "
                      f"of each shape (D={D0}, D={2 * H}; H={H}), the decoder "
                      + ("(T x [lstm_step + closure, D=" + str(D0 + 2 * H) + "] + T x [attention step fwd+bwd, "
                         "Ts=" + str(T) + "] + the readout GEMMs)" if att_case is not None else
                         "(one lstm_sequence D=" + str(D0 + 2 * H) + ")") + f", the output "
                      f"softmax + CE (V={V}) and the src/trg embedding lookups (gather_rows fwd+bwd, "
                      f"V={Vs}/{Vt}), step time = 2 t(D0) + {2 * (L - 1)} t(2H) + t(dec) + t(out) + t(emb) "
                      f"(layers run sequentially in the reference) "
                      f"+ one clip+Adam step over {n_par / 1e6:.1f}M params ({adam_s:.2f} s, fp32 numpy "
                      f"restatement timed on a 4M-element slice and scaled: the reference has no optimizer "
                      f"code); fp32 reference build + scipy OpenBLAS 1 thread/tape; median of {steps}",
            "seconds_per_step": max(per_seq) + adam_s}


# ---------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1805_05225_b200 import lstm
    from paper_1805_05225_b200.model import Seq2SeqAttention, Seq2SeqLSTM

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    L, B, T, D0, H = args.layers, args.batch, args.time, args.input, args.hidden
    Vs, Vt = args.src_vocab, (args.trg_vocab if args.vocab else 0)
    if args.attention:
        model = Seq2SeqAttention(L, B, T, T, D0, H, args.vocab, Vs, Vt, device=dev)
    else:
        model = Seq2SeqLSTM(L, B, T, D0, H, args.precision, dev, vocab=args.vocab, src_vocab=Vs, trg_vocab=Vt)
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
    if world == 1 and not args.no_graph:
        # The whole step (every kernel of the library, the glue copies, the
        # optimizer with its device-side step counter) captured once as a CUDA
        # graph and replayed: no host launch gaps.  Phases above come from the
        # eager pass (same kernels); the headline time from the replays.
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
        if args.attention and world == 1 and not args.no_graph:
            from paper_1805_05225_b200.model import GraphedStep
            graphed = GraphedStep(model, x, lens, dy)  # the public graphed-step API

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
                e2e=e2e, eager_ms=eager_ms / args.steps, graph=graph is not None)


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
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "f32", "data": "synthetic", "config": cfg, "impl": "reference",
                          "cpu_baseline": {k: cpu[k] for k in ("kind", "cores", "sample", "value", "unit")},
                          "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks=N) in the log
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    r = run_ours(args, rank, world, local_rank)
    tokens = world * B * T * args.steps
    value = tokens / (r["ms"] / 1e3)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
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
            peak = peaks.get("hbm_gbs", 7700.0)
        else:
            achieved = e["flops"] / max(e["calls"], 1) / (per_launch_ms / 1e3) / 1e12
            peak = peaks.get("bf16_tflops_sustained", 1400.0)
        traffic = None
        try:  # DRAM bytes per launch of this kernel from the committed ncu capture
            traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(name)
        except Exception:
            pass
        roof = {"kernel": name, "bound": "hbm" if hbm else "tensor", "achieved": achieved, "peak": peak,
                "unit": "GB/s" if hbm else "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/)",
                "peak_source": ("MEASURED_PEAKS.json " + ("hbm_gbs" if hbm else "bf16_tflops_sustained"))
                if peaks else "fallback",
                "share_of_step": e["ms"] / r["ms"],
                "phases": {k: {"calls": v["calls"], "ms_per_call": v["ms"] / max(v["calls"], 1),
                               "tflops": v["flops"] / max(v["ms"], 1e-9) / 1e9,
                               "gbs": v.get("bytes", 0) / max(v["ms"], 1e-9) / 1e6}
                           for k, v in ph.items()}}
    # recurrence phases: per-step latency against the W_h-from-SMEM bound the
    # north star names (bytes of W_h resident across the SMs / (SMs x 128 B/clk x f_SM))
    if roof is not None:
        f_sm = (r["clocks"].get("sm_mhz") or 1965.0) * 1e6
        rec = {}
        for name, nd_, hid in (("k2_rec_fwd", 2, H), ("k3_rec_bwd", 2, H)):
            e = ph.get(name)
            if not e:
                continue
            us = e["ms"] / max(e["calls"], 1) * 1e3 / T
            wh_bytes = nd_ * 4 * hid * hid * (2 if args.precision == "bf16" else 4)
            bound = wh_bytes / (148 * 128 * f_sm) * 1e6
            rec[name] = {"us_per_step": us, "wh_smem_bound_us": bound, "ratio_to_bound": us / bound}
        roof["recurrence_per_step"] = rec
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": r["ms"] / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": args.precision.replace("fp", "f"),
           "data": "synthetic (x ~ U(-1,1), params ~ U(+-1/sqrt(H)), dy ~ U(-1,1))",
           "config": cfg, "cuda_graph": r["graph"], "eager_ms_per_step": r["eager_ms"],
           "e2e": r["e2e"], "gpu_launches": r["launches"], "clocks": r["clocks"],
           "roofline": roof,
           "algorithmic_tflops": flops_per_token(L, D0, H, args.vocab, args.attention, T) * B * T * world / (r["ms"] / args.steps / 1e3) / 1e12}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            out["cpu_baseline"] = cpu_reference(args, steps=1)
        except Exception as exc:  # the baseline must never sink the GPU line
            out["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
