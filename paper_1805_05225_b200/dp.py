"""Data-parallel gradient exchange for the batch-sharded LSTM stack (SURVEY §8 e).

Training shards the batch across ranks; the one exchange per step is a sum
(optionally mean) all-reduce of every parameter gradient.  Gradients live in
one flat buffer with one contiguous bucket per layer (BLSTMEncoder), and the
bucket of layer l is reduced as soon as its BPTT finishes — while the BPTT of
layers l-1..0 still runs — so the collective overlaps compute.  With the NCCL
backend the reduction runs on NCCL's stream over NVLink/NVSwitch; the same
object works with gloo for the CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class BucketAllReducer:
    def __init__(self, group=None, average: bool = False):
        self.group = group
        self.average = average
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.force = False  # (test) issue the collective even at world 1
        self.issued = 0     # collectives issued (eager calls and graph captures)
        self._pending = []

    def __call__(self, layer: int, bucket: torch.Tensor) -> None:
        """on_layer_grads hook: start reducing this layer's bucket now."""
        if self.world == 1 and not (self.force and dist.is_initialized()):
            if self.average:
                bucket.div_(1)
            return
        self.issued += 1
        self._pending.append((bucket, dist.all_reduce(bucket, group=self.group, async_op=True)))

    def wait(self) -> None:
        while self._pending:
            bucket, h = self._pending.pop(0)
            h.wait()
            if self.average:
                bucket.div_(self.world)

    @property
    def in_flight(self) -> int:
        return len(self._pending)


def shard_rows(global_batch: int, rank: int, world: int) -> slice:
    """Rows of a global batch that rank `rank` of `world` owns: contiguous, sizes
    differing by at most one (SPEC.md:116 — independent tapes per batch shard)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return slice(start, start + base + (1 if rank < extra else 0))


def length_balanced_order(seq_lens, world: int):
    """A permutation of the global batch that deals the sequences, longest first,
    round-robin over the ranks: every shard gets a similar length mix, so no rank's
    recurrence runs many more steps than another's (the per-step latency, not the
    batch, bounds the recurrence).  Returns (order, inverse) index lists."""
    order = sorted(range(len(seq_lens)), key=lambda i: (-int(seq_lens[i]), i))
    dealt = [order[r::world] for r in range(world)]
    perm = [i for shard in dealt for i in shard]
    inv = [0] * len(perm)
    for pos, i in enumerate(perm):
        inv[i] = pos
    return perm, inv


class ShardedInference:
    """Config-5 inference sharded over the ranks with no communication: each rank
    encodes its rows of the global batch (length-balanced) and returns them with
    their global row indices; a caller that needs the whole output on one host
    concatenates the ranks' pieces by those indices (or each rank writes its rows
    to its own output file)."""

    def __init__(self, encoder_factory, global_batch: int, seq_lens, rank: int = None, world: int = None):
        self.rank = dist.get_rank() if rank is None and dist.is_initialized() else (rank or 0)
        self.world = dist.get_world_size() if world is None and dist.is_initialized() else (world or 1)
        perm, _ = length_balanced_order(list(seq_lens), self.world)
        sl = shard_rows(global_batch, self.rank, self.world)
        self.rows = perm[sl]                       # global row indices of this rank's shard
        self.encoder = encoder_factory(len(self.rows))

    def __call__(self, x, seq_lens):
        """x [B_global, T, F], seq_lens [B_global] (device) -> (global rows, y of those rows)."""
        idx = torch.as_tensor(self.rows, device=x.device, dtype=torch.long)
        return self.rows, self.encoder.forward(x.index_select(0, idx).contiguous(),
                                               seq_lens.index_select(0, idx).contiguous(), train=False)
