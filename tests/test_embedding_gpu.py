"""Embedding lookup on the GPU against the restatement of
Tape::gather_rows pinned to the reference (tests/test_oracle.py): the lookup is
a copy and the adjoint keeps the reference's fp32 summation order, so both
are compared bit-exactly."""
import numpy as np
import pytest
import torch

import oracle
from paper_1805_05225_b200 import lstm
from paper_1805_05225_b200.embedding import Embedding

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("V,D,B,T", [(2, 2, 1, 2), (13, 7, 5, 9), (20000, 620, 256, 60)])
def test_embedding_bitexact_vs_reference_restatement(cuda, V, D, B, T):
    rng = np.random.default_rng(V + D)
    tbl = rng.uniform(-1, 1, (V, D)).astype(np.float32)
    ids = rng.integers(0, V, (B, T)).astype(np.int32)
    ids[0, : T // 2 + 1] = V - 1  # a duplicate run: the order of the fp32 adds matters
    d_out = rng.uniform(-1, 1, (B, T, D)).astype(np.float32)
    out_o, g_o = oracle.gather_rows_np(tbl, ids, d_out)
    emb = Embedding(V, D, B * T)
    t_ids = torch.from_numpy(ids).cuda()
    t_tbl = torch.from_numpy(tbl).cuda()
    out = emb.forward(t_ids, t_tbl)
    emb.check_ids()
    assert np.array_equal(out.cpu().numpy(), out_o)
    g = torch.full((V, D), 7.0, device="cuda")
    emb.backward(t_ids, torch.from_numpy(d_out).cuda(), g)
    assert np.array_equal(g.cpu().numpy(), g_o)
    # accumulate: old + (the reference's per-call table gradient), GradBuffer::accumulate
    old = torch.from_numpy(rng.uniform(-1, 1, (V, D)).astype(np.float32)).cuda()
    g2 = old.clone()
    emb.backward(t_ids, torch.from_numpy(d_out).cuda(), g2, accumulate=True)
    assert np.array_equal(g2.cpu().numpy(), old.cpu().numpy() + g_o)


def test_embedding_bf16_layer0_input(cuda):
    V, D, B, T = 50, 37, 3, 4
    rng = np.random.default_rng(2)
    tbl = torch.from_numpy(rng.uniform(-1, 1, (V, D)).astype(np.float32)).cuda()
    ids = torch.from_numpy(rng.integers(0, V, (B, T)).astype(np.int32)).cuda()
    pitch = lstm.bf16_pitch(D)
    out = Embedding(V, D, B * T).forward(ids, tbl, bf16_pitch=pitch)
    ref = torch.zeros(B, T, pitch, dtype=torch.bfloat16, device="cuda")
    ref[..., :D] = tbl[ids.long()].to(torch.bfloat16)
    ref[..., D] = 1.0
    assert torch.equal(out, ref)


def test_embedding_bad_id_raises_index_error_naming_layer(cuda):
    emb = Embedding(4, 3, 8, layer="source_embed")
    tbl = torch.zeros(4, 3, device="cuda")
    ids = torch.tensor([[0, 1, 9, 2]], dtype=torch.int32, device="cuda")
    emb.forward(ids, tbl)
    with pytest.raises(IndexError, match=r"id 9 out of range \[0, 4\) in layer 'source_embed'"):
        emb.check_ids()
    emb.forward(torch.tensor([[3, 0]], dtype=torch.int32, device="cuda"), tbl)
    emb.check_ids()  # a clean call resets the flag


def test_embedding_strided_rows_and_negative_zero(cuda):
    # the decoder's previous-target embedding: rows land in the first E columns of
    # the wider [embedding ‖ context] input; id -1 (t = 0) gives the zero row
    # (initial_output = 0, models.cpp:96) without an error and adds no gradient
    V, E, W, B, T = 9, 5, 12, 2, 4
    rng = np.random.default_rng(4)
    tbl = torch.from_numpy(rng.uniform(-1, 1, (V, E)).astype(np.float32)).cuda()
    ids = torch.tensor([[-1, 3, 3, 8], [-1, 0, 7, 3]], dtype=torch.int32, device="cuda")
    buf = torch.full((B, T, W), 5.0, device="cuda")
    emb = Embedding(V, E, B * T)
    emb.forward(ids, tbl, out=buf[:, :, :E], negative_zero=True)
    emb.check_ids()
    ref = tbl[ids.clamp_min(0).long()] * (ids >= 0).unsqueeze(-1)
    assert torch.equal(buf[:, :, :E], ref) and bool((buf[:, :, E:] == 5.0).all())
    bufb = torch.full((B, T, W), 5.0, dtype=torch.bfloat16, device="cuda")
    emb.forward(ids, tbl, out=bufb[:, :, :E], negative_zero=True)
    assert torch.equal(bufb[:, :, :E], ref.to(torch.bfloat16)) and bool((bufb[:, :, E:] == 5.0).all())
    d = torch.from_numpy(rng.uniform(-1, 1, (B, T, W)).astype(np.float32)).cuda()
    g = torch.zeros(V, E, device="cuda")
    emb.backward(ids, d[:, :, :E], g)
    idn = ids.cpu().numpy().reshape(-1)
    dn = d[:, :, :E].cpu().numpy().reshape(-1, E)
    gr = np.zeros((V, E), np.float32)
    for r, v in enumerate(idn):
        if v >= 0:
            gr[v] += dn[r]
    assert np.array_equal(g.cpu().numpy(), gr)
    with pytest.raises(IndexError):  # without the flag a negative id is the reference's IndexError
        emb.forward(ids, tbl)
        emb.check_ids()
