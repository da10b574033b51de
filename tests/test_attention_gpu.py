"""The decoder's MLP attention step on the GPU against the fp64
restatement pinned to the reference's own layer ops (tests/test_oracle.py)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1805_05225_b200.attention import Attention

pytestmark = pytest.mark.gpu
TOL = 1e-4  # fp32 step vs fp64


def rel(a, b):
    a = torch.as_tensor(a).double().cpu()
    b = torch.as_tensor(np.asarray(b)).double().reshape(a.shape)
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("B,Ts,K,E,H", [(3, 6, 9, 8, 5), (17, 23, 130, 70, 40), (64, 60, 1000, 2000, 1000)])
def test_attention_step_matches_reference_restatement(cuda, B, Ts, K, E, H):
    rng = np.random.default_rng(B + Ts)
    lens = rng.integers(max(1, Ts // 2), Ts + 1, B).astype(np.int32)
    lens[0] = Ts
    args = dict(enc_ctx=rng.uniform(-1, 1, (B, Ts, K)), enc=rng.uniform(-1, 1, (B, Ts, E)),
                s=rng.uniform(-1, 1, (B, H)), accum=rng.uniform(0, 1, (B, Ts)),
                Ws=rng.uniform(-1, 1, (H, K)) / np.sqrt(H), bs=rng.uniform(-.5, .5, K),
                Wfb=rng.uniform(-.5, .5, (1, K)), bfb=rng.uniform(-.5, .5, K),
                v=rng.uniform(-1, 1, (K, 1)) / np.sqrt(K), bv=0.3)
    d_att, d_acc = rng.uniform(-1, 1, (B, E)), rng.uniform(-1, 1, (B, Ts))
    att, a, acc2, g = oracle.attention_step_np(lens, **args, d_att=d_att, d_accum=d_acc)
    cu = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.float32).cuda().contiguous()
    at = Attention(B, Ts, K, E, H)
    gi = dict(src_lens=torch.as_tensor(lens).cuda(), enc_ctx=cu(args["enc_ctx"]), enc=cu(args["enc"]),
              s=cu(args["s"]), accum=cu(args["accum"]), W_s=cu(args["Ws"]), b_s=cu(args["bs"]),
              W_fb=cu(args["Wfb"]), b_fb=cu(args["bfb"]), v=cu(args["v"]), b_v=cu([args["bv"]]))
    gatt, ga, gacc = at.forward(**gi)
    assert rel(gatt, att) < TOL and rel(ga, a) < TOL and rel(gacc, acc2) < TOL
    gi.pop("b_v")
    gg = at.backward(**gi, a=ga, d_att=cu(d_att), d_accum_out=cu(d_acc))
    torch.cuda.synchronize()
    for mine, ref in (("enc_ctx", "enc_ctx"), ("enc", "enc"), ("s", "s"), ("accum", "accum"), ("W_s", "Ws"),
                      ("b_s", "bs"), ("W_fb", "Wfb"), ("b_fb", "bfb"), ("v", "v")):
        assert rel(gg[mine], g[ref]) < TOL, mine
    # d b_v = sum of a softmax adjoint = 0 analytically: absolute check against the scale of d_e
    assert abs(float(gg["b_v"]) - float(g["bv"][0])) < 1e-5 * np.abs(g["enc_ctx"]).max() * B * Ts
    # padded source positions: no weight, no gradient into their encoder states
    for b in range(B):
        if lens[b] < Ts:
            assert float(ga[b, lens[b]:].abs().max()) == 0.0
            assert float(gg["enc"][b, lens[b]:].abs().max()) == 0.0
