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
        self._pending = []

    def __call__(self, layer: int, bucket: torch.Tensor) -> None:
        """on_layer_grads hook: start reducing this layer's bucket now."""
        if self.world == 1:
            if self.average:
                bucket.div_(1)
            return
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
