"""torchrun worker for tests/test_dp_graph_gpu.py: at world 1 over NCCL, the
data-parallel training step captured as one CUDA graph WITH its bucketed
gradient all-reduces (dp.BucketAllReducer forced to issue them) replays exactly
what the eager step without collectives computes (a 1-rank sum is the identity)."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1805_05225_b200.dp import BucketAllReducer  # noqa: E402
from paper_1805_05225_b200.model import GraphedStep, Seq2SeqAttention  # noqa: E402

DIMS = dict(enc_layers=2, batch=8, src_time=7, trg_time=6, emb=24, hidden=32, vocab=50, src_vocab=40, trg_vocab=50)


def make(prec):
    m = Seq2SeqAttention(**DIMS, device="cuda", lr=3e-3, dropout=0.3, precision=prec)
    m.init_uniform(5)
    return m


def main():
    prec = sys.argv[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    g = torch.Generator(device="cuda").manual_seed(6)
    B, Ts, T = DIMS["batch"], DIMS["src_time"], DIMS["trg_time"]
    src = torch.randint(0, DIMS["src_vocab"], (B, Ts), device="cuda", generator=g, dtype=torch.int32)
    trg = torch.randint(0, DIMS["vocab"], (B, T), device="cuda", generator=g, dtype=torch.int32)
    lens = torch.full((B,), Ts, dtype=torch.int32, device="cuda")
    lens[2:5] = torch.tensor([3, 5, 6], dtype=torch.int32)
    m1, m2 = make(prec), make(prec)
    red = BucketAllReducer()
    red.force = True
    gs = GraphedStep(m2, src, lens, trg, reducer=red, grad_scale=1.0)  # warm-up step + capture
    n_capture = red.issued
    m1.step(src, lens, trg)
    l1 = [float(m1.step(src, lens, trg)) for _ in range(3)]
    hs = [t.cpu().pin_memory() for t in (src, lens, trg)]
    l2 = [gs(*hs) for _ in range(3)]
    assert n_capture > 0 and red.issued == n_capture, (n_capture, red.issued)  # replays issue nothing new
    assert l1 == l2, (l1, l2)
    assert torch.equal(m1.params, m2.params)
    dist.destroy_process_group()
    print(f"DP_GRAPH_OK {prec} allreduces_per_step={n_capture // 2}")


if __name__ == "__main__":
    main()
