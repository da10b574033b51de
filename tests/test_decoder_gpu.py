"""The attention decoder (sl_attn_decoder_fwd/bwd) on the GPU against the fp64
restatement pinned to the reference build (tests/test_decoder_oracle.py).
bf16 tensor-core operands: the SL_PREC_BF16 tolerance (norm-wise 2e-2)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1805_05225_b200 import lstm
from paper_1805_05225_b200.decoder import NAMES, AttnDecoder, param_shapes

pytestmark = pytest.mark.gpu
TOL = 2e-2


def rel(a, b):
    a = torch.as_tensor(a).double().cpu()
    b = torch.as_tensor(np.asarray(b)).double().reshape(a.shape)
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def make_case(seed, B, Ts, T, emb, enc, hidden, key, readout, trg_vocab):
    rng = np.random.default_rng(seed)
    shapes = param_shapes(emb, enc, hidden, key, readout, trg_vocab)
    fan = {"enc_ctx_W": enc, "s_W": emb + enc + hidden, "s_R": emb + enc + hidden, "s_tr_W": hidden,
           "e_W": key, "readout_W": hidden + emb + enc}
    P = {}
    for n, s in shapes.items():
        sc = 1.0 / np.sqrt(fan[n]) if n in fan else 0.5
        P[n] = rng.uniform(-sc, sc, s).astype(np.float32)
    P["trg_W"] = rng.uniform(-1, 1, shapes["trg_W"]).astype(np.float32)
    enc_x = torch.as_tensor(rng.uniform(-1, 1, (B, Ts, enc)), dtype=torch.float32).bfloat16()
    lens = rng.integers(max(1, Ts // 2), Ts + 1, B).astype(np.int32)
    lens[0] = Ts
    ids = rng.integers(0, trg_vocab, (B, T)).astype(np.int32)
    ids[:, 0] = -1
    d_ro = rng.uniform(-1, 1, (B, T, readout)).astype(np.float32)
    return P, enc_x, lens, ids, d_ro


def run_gpu(dims, P, enc_x, lens, ids, d_ro, dec=None):
    B, Ts, T, emb, enc, hidden, key, readout, V = dims
    dec = dec or AttnDecoder(B, Ts, T, emb, enc, hidden, key, readout, V)
    pitch = lstm.bf16_pitch(enc)
    e = torch.zeros(B, Ts, pitch, dtype=torch.bfloat16, device="cuda")
    e[:, :, :enc] = enc_x.cuda()
    e[:, :, enc] = 1.0
    params = {n: torch.as_tensor(P[n]).cuda().contiguous() for n, _ in NAMES}
    grads = {n: torch.full_like(params[n], float("nan")) for n, _ in NAMES}
    src_lens = torch.as_tensor(lens).cuda()
    prev = torch.as_tensor(ids).cuda()
    ro = dec.forward(e, src_lens, prev, params)
    d_enc = dec.backward(e, src_lens, prev, params, ro, torch.as_tensor(d_ro).cuda(), grads)
    torch.cuda.synchronize()
    dec.check_ids(prev)
    return ro, grads, d_enc


CASES = [(4, 7, 5, 12, 16, 8, 16, 8, 11), (16, 23, 9, 20, 64, 32, 48, 24, 50),
         (8, 60, 60, 620, 2000, 1000, 1000, 1000, 300)]


# edge cases: long sources (Ts > 128: the softmax's looped tail, several energy / context
# tiles per row) with a length-1 source row; the largest batch one call takes (256); one target step
EDGE = [((3, 300, 6, 12, 16, 8, 16, 8, 11), [300, 1, 137]), ((256, 5, 3, 8, 8, 8, 8, 8, 7), None),
        ((5, 129, 2, 8, 24, 16, 8, 16, 9), [129, 128, 1, 64, 2]), ((4, 7, 1, 8, 8, 8, 8, 8, 5), None),
        # key_dim well below hidden: the d s = d s_tr W_s^T partials have their own row pitch
        ((4, 7, 5, 16, 32, 128, 32, 16, 11), None), ((6, 9, 4, 8, 16, 1000, 64, 16, 7), None)]


def check_against_restatement(dims, lens_override=None):
    P, enc_x, lens, ids, d_ro = make_case(sum(dims), *dims)
    if lens_override is not None:
        lens = np.asarray(lens_override, dtype=np.int32)
    ro, grads, d_enc = run_gpu(dims, P, enc_x, lens, ids, d_ro)
    # the relu derivative as the GPU saw it: bf16 operands may round a pre-activation
    # within its error of 0 to the other side (each such flip moves a whole readout_W
    # column), so the gradients are compared under the same mask, and the masks may
    # differ only where the fp64 pre-activation is within that error of 0
    mask = (ro > 0).cpu().numpy()
    r_ro, g, r_denc = oracle.attn_decoder_np(lens, enc_x.float().numpy(), ids, P, d_readout=d_ro, relu_mask=mask)
    pre = oracle.attn_decoder_np.pre
    flips = mask != (pre > 0)
    assert np.abs(pre[flips]).max(initial=0.0) < 2 * TOL * np.abs(pre).max()
    assert rel(ro, r_ro) < TOL
    assert rel(d_enc, r_denc) < TOL
    for n, _ in NAMES:
        if n == "e_b":  # sum of softmax adjoints: 0 analytically — compare on the scale of d e
            assert abs(float(grads[n]) - float(g[n][0])) < 1e-3 * max(1.0, np.abs(g["e_W"]).max()), n
            continue
        assert rel(grads[n], g[n]) < TOL, (n, rel(grads[n], g[n]))


@pytest.mark.parametrize("dims", CASES)
def test_decoder_matches_restatement(cuda, dims):
    check_against_restatement(dims)


@pytest.mark.parametrize("dims,lens", EDGE)
def test_decoder_edge_cases_match_restatement(cuda, dims, lens):
    check_against_restatement(dims, lens)


def test_decoder_deterministic_and_masked(cuda):
    dims = CASES[1]
    P, enc_x, lens, ids, d_ro = make_case(7, *dims)
    lens[1] = 5
    dec = AttnDecoder(*dims)
    ro1, g1, d1 = run_gpu(dims, P, enc_x, lens, ids, d_ro, dec)
    enc2 = enc_x.clone()
    enc2[1, 5:] = 3.0  # padded source positions must not matter
    ro2, g2, d2 = run_gpu(dims, P, enc2, lens, ids, d_ro, dec)
    assert torch.equal(ro1, ro2)
    assert float(d1[1, 5:].abs().max()) == 0.0
    for n, _ in NAMES:
        if n in ("enc_ctx_W", "enc_ctx_b"):
            continue
        assert torch.equal(g1[n], g2[n]), n
    ro3, g3, d3 = run_gpu(dims, P, enc_x, lens, ids, d_ro, dec)
    assert torch.equal(ro1, ro3) and torch.equal(d1, d3)
    for n, _ in NAMES:
        assert torch.equal(g1[n], g3[n]), n


def test_decoder_bad_id_raises(cuda):
    dims = CASES[0]
    P, enc_x, lens, ids, d_ro = make_case(1, *dims)
    ids[2, 3] = dims[-1]
    with pytest.raises(IndexError, match="output/trg"):
        run_gpu(dims, P, enc_x, lens, ids, d_ro)


def test_decoder_shape_errors(cuda):
    with pytest.raises(lstm.ShapeError):
        AttnDecoder(4, 7, 5, 12, 16, 8, 2000, 8, 11)  # key_dim > 1024



def test_dropout_matches_reference_mask_bitwise(cuda):
    """sl_dropout_fwd/bwd: the reference's counter-based mask (oracle.dropout_np, pinned
    to Tape::dropout), bit-identical values and gradients; the device-side counter
    path equals the host-value path."""
    from paper_1805_05225_b200.dropout import Dropout
    rng = np.random.default_rng(3)
    for (B, T, F), seed, counter, rate in (((16, 60, 1000), 1, 0, 0.3), ((16, 60, 1000), 77, 12, 0.5),
                                           ((4, 5, 999), 5, 3, 0.1), ((3, 7, 1000), 9, 1, 0.0)):
        x = rng.uniform(-1, 1, (B, T, F)).astype(np.float32)
        d = rng.uniform(-1, 1, (B, T, F)).astype(np.float32)
        dr = Dropout(rate, seed, "output/output_prob", 0)
        xg, dg = torch.as_tensor(x).cuda(), torch.as_tensor(d).cuda()
        y, dx = torch.empty_like(xg), torch.empty_like(xg)
        dr.forward(xg, y, counter_value=counter)
        dr.backward(dg, dx, counter_value=counter)
        key = oracle.dropout_key(seed, "output/output_prob", 0, counter)
        ry, rdx = oracle.dropout_np(x, key, rate, d_out=d)
        assert np.array_equal(y.cpu().numpy(), ry) and np.array_equal(dx.cpu().numpy(), rdx)
        ctr = torch.tensor([counter], dtype=torch.int32, device="cuda")
        y2 = torch.empty_like(xg)
        dr.forward(xg, y2, counter=ctr)
        assert torch.equal(y, y2)
    with pytest.raises(ValueError):
        Dropout(1.0, 1, "x")
