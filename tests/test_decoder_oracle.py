"""Pinning the attention-decoder oracle (oracle.attn_decoder_np) on CPU.

The decoder restatement chains two per-step restatements; each is pinned to
the REFERENCE build (oracle/_ref), and the chaining (the reverse replay of the
per-step closures) is pinned by finite differences of the whole sequence."""
import numpy as np
import pytest

import oracle
from paper_1805_05225_b200.decoder import param_shapes

DIMS = dict(emb=5, enc=6, hidden=4, key=7, readout=3, trg_vocab=9)


def _ref():
    try:
        return oracle.Reference(64)
    except FileNotFoundError as e:
        pytest.skip(str(e))


def decoder_case(seed, B, Ts, T, emb, enc, hidden, key, readout, trg_vocab, scale=0.6):
    rng = np.random.default_rng(seed)
    P = {n: rng.uniform(-scale, scale, s) for n, s in param_shapes(emb, enc, hidden, key, readout, trg_vocab).items()}
    enc_x = rng.uniform(-1, 1, (B, Ts, enc))
    lens = rng.integers(max(1, Ts // 2), Ts + 1, B).astype(np.int32)
    lens[0] = Ts
    ids = rng.integers(0, trg_vocab, (B, T)).astype(np.int32)
    ids[:, 0] = -1  # the zero initial output of prev:trg
    return P, enc_x, lens, ids


def test_lstm_step_restatement_pinned_to_reference():
    ref = _ref()
    rng = np.random.default_rng(3)
    B, D, H = 3, 5, 4
    x, h, c = rng.uniform(-1, 1, (B, D)), rng.uniform(-1, 1, (B, H)), rng.uniform(-1, 1, (B, H))
    W, R, b = rng.uniform(-1, 1, (D, 4 * H)), rng.uniform(-1, 1, (H, 4 * H)), rng.uniform(-1, 1, 4 * H)
    gh, gc = rng.uniform(-1, 1, (B, H)), rng.uniform(-1, 1, (B, H))
    h2, c2 = oracle.lstm_step_np(x, h, c, W, R, b)
    rh, rc, rg = ref.step(x, h, c, W, R, b, gh=gh, gc=gc)
    assert np.abs(h2 - rh).max() < 1e-13 and np.abs(c2 - rc).max() < 1e-13
    mine = oracle.lstm_step_np(x, h, c, W, R, b, gh=gh, gc=gc)
    for m, r in zip(mine, rg):
        assert np.abs(m - r).max() < 1e-12


def test_decoder_restatement_finite_differences():
    B, Ts, T = 2, 4, 3
    P, enc_x, lens, ids = decoder_case(0, B, Ts, T, **DIMS)
    rng = np.random.default_rng(1)
    w = rng.uniform(-1, 1, (B, T, DIMS["readout"]))
    loss = lambda P_, e_: float((oracle.attn_decoder_np(lens, e_, ids, P_) * w).sum())
    _, g, d_enc = oracle.attn_decoder_np(lens, enc_x, ids, P, d_readout=w)
    eps = 1e-6
    for name in P:
        flat = P[name].reshape(-1)
        for idx in rng.choice(flat.size, size=min(4, flat.size), replace=False):
            old = flat[idx]
            flat[idx] = old + eps
            lp = loss(P, enc_x)
            flat[idx] = old - eps
            lm = loss(P, enc_x)
            flat[idx] = old
            fd = (lp - lm) / (2 * eps)
            an = g[name].reshape(-1)[idx]
            assert abs(fd - an) <= 1e-6 + 1e-5 * abs(fd), (name, idx, fd, an)
    flat = enc_x.reshape(-1)
    for idx in rng.choice(flat.size, size=8, replace=False):
        old = flat[idx]
        flat[idx] = old + eps
        lp = loss(P, enc_x)
        flat[idx] = old - eps
        lm = loss(P, enc_x)
        flat[idx] = old
        fd = (lp - lm) / (2 * eps)
        assert abs(fd - d_enc.reshape(-1)[idx]) <= 1e-6 + 1e-5 * abs(fd), idx


def test_decoder_restatement_masks_padded_sources():
    """Padded source positions get no attention weight, so neither the outputs
    nor any gradient depend on their encoder states (tape.cpp:952-960)."""
    P, enc_x, lens, ids = decoder_case(2, 3, 5, 3, **DIMS)
    lens[:] = [5, 3, 2]
    w = np.random.default_rng(4).uniform(-1, 1, (3, 3, DIMS["readout"]))
    r1, g1, d1 = oracle.attn_decoder_np(lens, enc_x, ids, P, d_readout=w)
    enc2 = enc_x.copy()
    enc2[1, 3:] = 7.0
    enc2[2, 2:] = -3.0
    r2, g2, d2 = oracle.attn_decoder_np(lens, enc2, ids, P, d_readout=w)
    assert np.array_equal(r1, r2)
    assert np.abs(d1[1, 3:]).max() == 0 and np.abs(d1[2, 2:]).max() == 0
    for n in g1:
        if n not in ("enc_ctx_W", "enc_ctx_b"):
            assert np.allclose(g1[n], g2[n], rtol=0, atol=1e-14), n


def test_dropout_restatement_pinned_to_reference():
    """The output_prob input dropout: the numpy restatement of the reference's
    counter-based mask (rng.hpp splitmix64/mix64/fnv1a, tape.cpp:540-600) equals the
    reference's own Tape::dropout bit for bit (values and gradient)."""
    ref = _ref()
    rng = np.random.default_rng(0)
    B, T, F = 3, 5, 7
    x, d = rng.uniform(-1, 1, (B, T, F)), rng.uniform(-1, 1, (B, T, F))
    for seed, counter, rate in ((1, 0, 0.3), (12345, 7, 0.5), (2**63 + 5, 3, 0.1)):
        out, dx = ref.dropout(x, rate, seed, "output/output_prob", 0, counter, d_out=d)
        key = oracle.dropout_key(seed, "output/output_prob", 0, counter)
        o2, d2 = oracle.dropout_np(x, key, rate, d_out=d, real=np.float64)
        assert np.array_equal(out, o2) and np.array_equal(dx, d2)
        keep = oracle.dropout_mask_np(key, B, T, F, rate)
        assert 0 < keep.sum() < keep.size
