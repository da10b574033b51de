"""Data parallelism on the real model (SURVEY §8 e, SPEC.md:116 — independent
tapes per batch shard, one gradient all-reduce): the Listing-1 attention model's
gradients averaged over two batch shards equal the full-batch gradients (the
bench's NCCL sum all-reduce + grad_scale = 1/N in the fused Adam), emulated on
one GPU as two shard models with the same parameters.  fp32 mode, 1e-4 per
tensor; dropout off (its mask is keyed by the batch row within a tape, so a
sharded run draws different masks by construction, as in the reference)."""
import pytest
import torch

from paper_1805_05225_b200.model import Seq2SeqAttention

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 2e-2)])
def test_shard_gradients_average_to_full_batch(cuda, prec, tol):
    L, B, T, E, H, V = 2, 16, 9, 24, 32, 50
    full = Seq2SeqAttention(L, B, T, T, E, H, V, V, V, device="cuda", dropout=0.0, precision=prec)
    full.init_uniform(seed=3)
    shards = [Seq2SeqAttention(L, B // 2, T, T, E, H, V, V, V, device="cuda", dropout=0.0, precision=prec)
              for _ in range(2)]
    for s in shards:
        s.params.copy_(full.params)
    g = torch.Generator(device="cuda").manual_seed(4)
    src = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
    trg = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int32)
    lens = torch.full((B,), T, dtype=torch.int32, device="cuda")  # equal valid counts per shard
    full.forward_backward(src, lens, trg)
    for r, s in enumerate(shards):
        sl = slice(r * B // 2, (r + 1) * B // 2)
        s.forward_backward(src[sl].contiguous(), lens[sl].contiguous(), trg[sl].contiguous())
    torch.cuda.synchronize()
    avg = (shards[0].grads + shards[1].grads) / 2  # NCCL sum, then the 1/N folded into Adam
    for name, off, shape in full.manifest:
        n = 1
        for d in shape:
            n *= d
        a, r = avg[off:off + n].double(), full.grads[off:off + n].double()
        if name == "output/e/b":  # 0 analytically: compare on the scale of the energy gradient
            continue
        err = float((a - r).abs().max() / r.abs().max().clamp_min(1e-30))
        assert err < tol, (name, err)
