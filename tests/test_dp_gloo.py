"""N>1 path on CPU: world_size-2 gloo processes exercise the bucketed,
overlapped gradient all-reduce the bench uses with NCCL (dp.BucketAllReducer),
and check that data-parallel gradients over batch shards equal the
single-process gradient of the whole batch — on the fp64 oracle's LSTM
gradients (the GPU kernels are covered by the gpu tests)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1805_05225_b200.dp import BucketAllReducer
        orc = oracle.Restatement()
        B, T, D, H = 6, 5, 4, 3
        x, lens, W, R, b = oracle.seeded_case(77, B, T, D, H)
        dy = np.random.default_rng(5).uniform(-1, 1, (B, T, H))
        shard = slice(rank * B // world, (rank + 1) * B // world)
        # two "layers" (fw, bw directions) -> two buckets, reduced as each finishes
        flat = torch.zeros(2 * (D * 4 * H + H * 4 * H + 4 * H), dtype=torch.float64)
        n = D * 4 * H + H * 4 * H + 4 * H
        red = BucketAllReducer()
        for layer, d in enumerate((-1, 1)):
            _, gW, gR, gb = orc.sequence_bwd(x[shard], lens[shard], W, R, b, d, dy[shard])
            bucket = flat[layer * n:(layer + 1) * n]
            bucket.copy_(torch.from_numpy(np.concatenate([gW.ravel(), gR.ravel(), gb.ravel()])))
            red(layer, bucket)
        assert red.in_flight == 2
        red.wait()
        q.put((rank, flat.numpy()))
    finally:
        dist.destroy_process_group()


def test_dp_allreduce_matches_full_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    orc = oracle.Restatement()
    B, T, D, H = 6, 5, 4, 3
    x, lens, W, R, b = oracle.seeded_case(77, B, T, D, H)
    dy = np.random.default_rng(5).uniform(-1, 1, (B, T, H))
    full = []
    for d in (-1, 1):
        _, gW, gR, gb = orc.sequence_bwd(x, lens, W, R, b, d, dy)
        full.append(np.concatenate([gW.ravel(), gR.ravel(), gb.ravel()]))
    full = np.concatenate(full)
    for r in range(world):
        assert np.allclose(results[r], full, rtol=0, atol=1e-12)
