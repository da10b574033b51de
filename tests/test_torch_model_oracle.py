"""Pins oracle/torch_model.py (the fp64 torch restatement of the whole Listing-1
training step, used by the full-size GPU parity tests) to the reference-pinned
compositions at small sizes: the reference build's own BLSTM stack
(oracle.Reference.blstm_stack), attn_decoder_np, dropout_np (the reference's
mask) and output_ce_np, chained exactly as the reference's graph chains them."""
import numpy as np
import pytest
import torch

import oracle
from oracle import torch_model

try:
    REF = oracle.Reference(64)
except FileNotFoundError:  # the reference build is only produced where /root/reference exists
    REF = None


def make_params(rng, L, D0, H, K, Rd, E, V, Vs, Vt):
    from paper_1805_05225_b200.decoder import param_shapes
    P = {}
    for l in range(L):
        D = D0 if l == 0 else 2 * H
        for d in ("fw", "bw"):
            P[f"enc{l}_{d}/W"] = rng.uniform(-0.4, 0.4, (D, 4 * H))
            P[f"enc{l}_{d}/R"] = rng.uniform(-0.4, 0.4, (H, 4 * H))
            P[f"enc{l}_{d}/b"] = rng.uniform(-0.4, 0.4, 4 * H)
    for n, s in param_shapes(D0, E, H, K, Rd, Vt).items():
        P[n] = rng.uniform(-0.4, 0.4, s)
    P["out_W"] = rng.uniform(-0.4, 0.4, (Rd, V))
    P["out_b"] = rng.uniform(-0.4, 0.4, V)
    P["src_W"] = rng.uniform(-1, 1, (Vs, D0))
    return P


@pytest.mark.skipif(REF is None, reason="reference build absent")
def test_torch_model_matches_reference_composition():
    rng = np.random.default_rng(3)
    L, B, Ts, T, D0, H, K, Rd, V, Vs, Vt = 2, 4, 6, 5, 7, 5, 6, 4, 9, 11, 9
    E = 2 * H
    P = make_params(rng, L, D0, H, K, Rd, E, V, Vs, Vt)
    src = rng.integers(0, Vs, (B, Ts)).astype(np.int32)
    trg = rng.integers(0, V, (B, T)).astype(np.int32)
    lens = np.array([6, 3, 5, 1], np.int32)
    tl = np.array([5, 5, 2, 4], np.int32)
    key = oracle.dropout_key(1, "output/output_prob", 0, 3)
    keep = oracle.dropout_mask_np(key, B, T, Rd, 0.3)
    # the reference-pinned composition
    x0 = P["src_W"][src]
    params = [tuple(P[f"enc{l}_{d}/{n}"] for d in ("fw", "bw") for n in ("W", "R", "b")) for l in range(L)]
    y, _, _ = REF.blstm_stack(x0, lens, params)
    prev = np.full_like(trg, -1)
    prev[:, 1:] = trg[:, :-1]
    readout = oracle.attn_decoder_np(lens, y, prev, P)
    drop = oracle.dropout_np(readout, key, 0.3, real=np.float64)
    r_loss, d_drop, r_dW, r_db = oracle.output_ce_np(drop, tl, trg, P["out_W"], P["out_b"], 0.1)
    _, d_ro = oracle.dropout_np(readout, key, 0.3, d_out=d_drop, real=np.float64)
    _, g, d_enc = oracle.attn_decoder_np(lens, y, prev, P, d_readout=d_ro)
    _, dx, eg = REF.blstm_stack(x0, lens, params, dy=d_enc)
    d_src = np.zeros_like(P["src_W"])
    np.add.at(d_src, src.reshape(-1), dx.reshape(-1, D0))
    # the torch restatement
    tP = {k: torch.as_tensor(v, dtype=torch.float64) for k, v in P.items()}
    t = lambda a: torch.as_tensor(a)
    loss, ro, tg = torch_model.loss_and_grads(tP, t(src), t(lens), t(trg), t(tl), L, keep=t(keep))
    def close(a, b):
        a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
        # 1e-7: the dropout scale is the reference's fp32 Real(1) / (Real(1) - rate) here,
        # 1 / 0.7 in fp64 in dropout_np(real=float64) — a 2.4e-8 relative difference
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)) < 1e-7
    assert close(float(loss), r_loss) and close(ro.numpy(), readout)
    assert close(tg["out_W"], r_dW) and close(tg["out_b"], r_db) and close(tg["src_W"], d_src)
    from paper_1805_05225_b200.decoder import NAMES
    for n, _ in NAMES:
        if n == "e_b":  # sum of softmax adjoints: 0 analytically (rounding noise ~1e-18 both sides)
            assert abs(float(tg[n][0]) - float(g[n][0])) < 1e-12
            continue
        assert close(tg[n], g[n]), n
    for l in range(L):
        for i, (d, n) in enumerate([(d, n) for d in ("fw", "bw") for n in ("W", "R", "b")]):
            assert close(tg[f"enc{l}_{d}/{n}"], eg[l][i]), (l, d, n)
