"""The attention decoder at the reference's precision (sl_attn_decoder_fwd_f32 /
bwd_f32: split-bf16 tcgen05 GEMMs, fp32 attention and cell state) against the
fp64 restatement pinned to the reference build (tests/test_decoder_oracle.py),
per tensor within the FP32 tolerance 1e-4 — up to the config-4 widths."""
import numpy as np
import pytest
import torch

import oracle
from paper_1805_05225_b200.decoder import NAMES, AttnDecoder
from test_decoder_gpu import make_case, rel

pytestmark = pytest.mark.gpu
TOL = 1e-4


def run_f32(dims, P, enc_x, lens, ids, d_ro, dec=None):
    B, Ts, T, emb, enc, hidden, key, readout, V = dims
    dec = dec or AttnDecoder(B, Ts, T, emb, enc, hidden, key, readout, V, precision="fp32")
    e = torch.as_tensor(enc_x).cuda().contiguous()
    params = {n: torch.as_tensor(P[n]).cuda().contiguous() for n, _ in NAMES}
    grads = {n: torch.full_like(params[n], float("nan")) for n, _ in NAMES}
    src_lens = torch.as_tensor(lens).cuda()
    prev = torch.as_tensor(ids).cuda()
    ro = dec.forward(e, src_lens, prev, params)
    d_enc = dec.backward(e, src_lens, prev, params, ro, torch.as_tensor(d_ro).cuda(), grads)
    torch.cuda.synchronize()
    dec.check_ids(prev)
    return ro, grads, d_enc


def check(dims, lens_override=None):
    P, enc_b, lens, ids, d_ro = make_case(sum(dims), *dims)
    enc_x = np.random.default_rng(sum(dims) + 1).uniform(-1, 1, enc_b.shape).astype(np.float32)
    if lens_override is not None:
        lens = np.asarray(lens_override, dtype=np.int32)
    ro, grads, d_enc = run_f32(dims, P, enc_x, lens, ids, d_ro)
    mask = (ro > 0).cpu().numpy()
    r_ro, g, r_denc = oracle.attn_decoder_np(lens, enc_x.astype(np.float64), ids, P, d_readout=d_ro, relu_mask=mask)
    pre = oracle.attn_decoder_np.pre
    flips = mask != (pre > 0)  # only pre-activations within fp32-class error of 0 may flip
    assert np.abs(pre[flips]).max(initial=0.0) < 2 * TOL * np.abs(pre).max()
    assert rel(ro, r_ro) < TOL, rel(ro, r_ro)
    assert rel(d_enc, r_denc) < TOL, rel(d_enc, r_denc)
    for n, _ in NAMES:
        if n == "e_b":  # sum of softmax adjoints: 0 analytically — compare on the scale of d e
            assert abs(float(grads[n]) - float(g[n][0])) < 1e-5 * max(1.0, np.abs(g["e_W"]).max()), n
            continue
        assert rel(grads[n], g[n]) < TOL, (n, rel(grads[n], g[n]))


CASES = [(4, 7, 5, 12, 16, 8, 16, 8, 11), (16, 23, 9, 20, 64, 32, 48, 24, 50), (5, 129, 2, 8, 24, 16, 8, 16, 9),
         (4, 7, 5, 16, 32, 128, 32, 16, 11), (8, 60, 60, 620, 2000, 1000, 1000, 1000, 300)]


@pytest.mark.parametrize("dims", CASES)
def test_decoder_f32_matches_restatement(cuda, dims):
    check(dims)


def test_decoder_f32_ragged_and_length_one_sources(cuda):
    check((3, 300, 6, 12, 16, 8, 16, 8, 11), [300, 1, 137])


def test_decoder_f32_padded_sources_do_not_matter(cuda):
    dims = CASES[1]
    P, enc_b, lens, ids, d_ro = make_case(7, *dims)
    enc_x = np.random.default_rng(3).uniform(-1, 1, enc_b.shape).astype(np.float32)
    lens[1] = 5
    dec = AttnDecoder(*dims, precision="fp32")
    ro1, g1, d1 = run_f32(dims, P, enc_x, lens, ids, d_ro, dec)
    enc2 = enc_x.copy()
    enc2[1, 5:] = 3.0
    ro2, g2, d2 = run_f32(dims, P, enc2, lens, ids, d_ro, dec)
    assert torch.equal(ro1, ro2)
    assert float(d1[1, 5:].abs().max()) == 0.0
