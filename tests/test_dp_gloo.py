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


def test_shard_rows_cover_the_batch_once():
    from paper_1805_05225_b200.dp import length_balanced_order, shard_rows
    for B, world in [(256, 8), (10, 3), (5, 8), (1024, 4)]:
        got = []
        for r in range(world):
            got.extend(range(B)[shard_rows(B, r, world)])
        assert got == list(range(B))
        sizes = [len(range(B)[shard_rows(B, r, world)]) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1
    lens = [60, 3, 59, 60, 10, 31, 2, 45]
    perm, inv = length_balanced_order(lens, 2)
    assert sorted(perm) == list(range(8)) and [perm[inv[i]] for i in range(8)] == list(range(8))
    shards = [[lens[i] for i in perm[shard_rows(8, r, 2)]] for r in range(2)]
    assert abs(sum(shards[0]) - sum(shards[1])) <= max(lens)  # balanced work
    assert max(shards[0]) == max(shards[1]) == 60


def _infer_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1805_05225_b200.dp import ShardedInference
        orc = oracle.Restatement()
        B, T, D, H = 7, 5, 4, 3
        x, lens, W, R, b = oracle.seeded_case(13, B, T, D, H)

        class Enc:  # the per-rank encoder (here the fp64 oracle layer; on a GPU box BLSTMEncoder)
            def __init__(self, rows):
                self.rows = rows

            def forward(self, xs, ls, train=False):
                y, _, _ = orc.sequence_fwd(xs.numpy(), ls.numpy(), W, R, b, 1)
                return torch.as_tensor(y)

        inf = ShardedInference(Enc, B, lens)
        rows, y = inf(torch.as_tensor(x), torch.as_tensor(lens))
        q.put((rank, rows, y.numpy()))  # no collective on the data path
    finally:
        dist.destroy_process_group()


def test_sharded_inference_equals_whole_batch():
    """Config-5 style inference over world-2 gloo ranks: the union of the ranks'
    rows equals the whole-batch forward, with no communication on the data path."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_infer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    orc = oracle.Restatement()
    B, T, D, H = 7, 5, 4, 3
    x, lens, W, R, b = oracle.seeded_case(13, B, T, D, H)
    full, _, _ = orc.sequence_fwd(x, lens, W, R, b, 1)
    seen = []
    for _, rows, y in res:
        seen.extend(rows)
        assert np.allclose(y, full[rows], rtol=0, atol=1e-12)
    assert sorted(seen) == list(range(B))
