"""ORACLE — test infrastructure only (tests/ may import it; the product never does).

The whole Listing-1 training step (BASELINE configs[3]) restated in fp64 torch
with autograd, so GPU parity tests can check the bench workload at its full
size (6 x BLSTM H=1000, B=256, T=60, V=20000) in seconds on the GPU box:

  src lookup (gather_rows, tape.cpp:448-492) -> L BLSTM layers (lstm_sequence
  fw / bw + concat, layers.cpp:8-37, compiler.cpp:600-608; torch_ref.sequence's
  step math, tape.cpp:1103-1135) -> enc_ctx (models.cpp:60) -> the `output`
  subnetwork step by step with teacher forcing (models.cpp:83-166,
  compiler.cpp:770-905: lstm_step on [trg_{t-1} ‖ att_{t-1}], s_tr, the MLP
  energies with weight feedback, softmax_over_spatial tape.cpp:926-985,
  generic_attention tape.cpp:987-1072) -> relu readout -> dropout (the
  reference's keep mask, oracle.dropout_mask_np) -> output_prob + label-smoothed
  CE (compiler.cpp:651-663, tape.cpp:879-924, 1224-1298).

The gradients are autograd's adjoints of exactly this forward.  The module is
pinned at small sizes to the reference-pinned compositions
(oracle.Reference.blstm_stack, attn_decoder_np, output_ce_np, dropout_np) by
tests/test_torch_model_oracle.py.
"""
from __future__ import annotations

import torch


def _lstm_seq(x, lens, W, R, b, direction):
    """lstm_sequence forward (layers.cpp:22-36): per-sequence prefix reversal for
    direction -1 (tape.cpp:846), zero state, masked output (tape.cpp:797)."""
    B, T, D = x.shape
    H = R.shape[0]
    dev = x.device
    s = torch.arange(T, device=dev).unsqueeze(0).expand(B, T)
    L = lens.long().unsqueeze(1)
    src = s if direction > 0 else torch.where(s < L, L - 1 - s, s)
    rows = torch.arange(B, device=dev).unsqueeze(1)
    xs = x[rows, src]
    h = x.new_zeros(B, H)
    c = x.new_zeros(B, H)
    hs = []
    for t in range(T):
        z = xs[:, t] @ W + h @ R + b
        i, f = torch.sigmoid(z[:, :H]), torch.sigmoid(z[:, H:2 * H])
        g, o = torch.tanh(z[:, 2 * H:3 * H]), torch.sigmoid(z[:, 3 * H:])
        c = f * c + i * g
        h = o * torch.tanh(c)
        hs.append(h)
    Hs = torch.stack(hs, 1)
    valid = (s < L).unsqueeze(-1)
    y = torch.zeros_like(Hs).index_put((rows.expand(B, T), src), Hs * valid)
    return y


def _lstm_step(x, h, c, W, R, b):
    H = h.shape[1]
    z = x @ W + h @ R + b
    i, f = torch.sigmoid(z[:, :H]), torch.sigmoid(z[:, H:2 * H])
    g, o = torch.tanh(z[:, 2 * H:3 * H]), torch.sigmoid(z[:, 3 * H:])
    c2 = f * c + i * g
    return o * torch.tanh(c2), c2


def forward_loss(P, src_ids, src_lens, trg_ids, trg_lens, L, keep=None, rate=0.3, eps=0.1, relu_mask=None):
    """P: dict of fp64 leaf tensors named like the model's manifest
    (enc{l}_{fw,bw}/{W,R,b}, the decoder.NAMES fields, out_W, out_b, src_W).
    keep: the dropout keep mask [B, T, Rd] (bool) or None (no dropout).
    relu_mask: optional [B, T, Rd] bool used as the readout relu's derivative
    (the forward value is always relu(pre)).  Returns (loss, readout)."""
    dev = src_ids.device
    B, Ts = src_ids.shape
    T = trg_ids.shape[1]
    x = P["src_W"][src_ids.long()]
    for l in range(L):
        ys = [_lstm_seq(x, src_lens, P[f"enc{l}_{d}/W"], P[f"enc{l}_{d}/R"], P[f"enc{l}_{d}/b"], sgn)
              for d, sgn in (("fw", 1), ("bw", -1))]
        x = torch.cat(ys, 2)
    enc = x
    E = enc.shape[2]
    H = P["s_R"].shape[0]
    enc_ctx = enc @ P["enc_ctx_W"] + P["enc_ctx_b"]
    prev = torch.full_like(trg_ids, -1)
    prev[:, 1:] = trg_ids[:, :-1]
    trg = torch.where((prev >= 0).unsqueeze(-1), P["trg_W"][prev.clamp_min(0).long()], 0.0)
    valid_src = torch.arange(Ts, device=dev).unsqueeze(0) < src_lens.long().unsqueeze(1)
    s = enc.new_zeros(B, H)
    c = enc.new_zeros(B, H)
    att = enc.new_zeros(B, E)
    acc = enc.new_zeros(B, Ts)
    S, ATT = [], []
    for t in range(T):
        s, c = _lstm_step(torch.cat([trg[:, t], att], 1), s, c, P["s_W"], P["s_R"], P["s_b"])
        s_tr = s @ P["s_tr_W"] + P["s_tr_b"]
        u = torch.tanh(enc_ctx + acc.unsqueeze(-1) * P["fb_W"][0] + P["fb_b"] + s_tr.unsqueeze(1))
        e = u @ P["e_W"][:, 0] + P["e_b"][0]
        e = torch.where(valid_src, e, float("-inf"))
        a = torch.softmax(e, 1)
        a = torch.where(valid_src, a, 0.0)
        acc = acc + a
        att = torch.einsum("bj,bje->be", a, enc)
        S.append(s)
        ATT.append(att)
    RO = torch.cat([torch.stack(S, 1), trg, torch.stack(ATT, 1)], 2)
    pre = RO @ P["readout_W"] + P["readout_b"]
    if relu_mask is None:
        readout = torch.relu(pre)
    else:  # relu(pre) in value, the given mask as its derivative
        m = relu_mask.to(pre.dtype)
        readout = pre * m + (torch.relu(pre) - pre * m).detach()
    h = readout
    if keep is not None:
        inv = float(torch.tensor(1.0, dtype=torch.float32) / (1.0 - torch.tensor(rate, dtype=torch.float32)))
        h = torch.where(keep, h * inv, 0.0)
    z = h @ P["out_W"] + P["out_b"]
    lp = torch.log_softmax(z, 2)
    V = z.shape[2]
    valid_t = torch.arange(T, device=dev).unsqueeze(0) < trg_lens.long().unsqueeze(1)
    rowloss = -(1 - eps) * lp.gather(2, trg_ids.long().unsqueeze(-1))[..., 0] - eps / V * lp.sum(2)
    loss = (rowloss * valid_t).sum() / valid_t.sum()
    return loss, readout


def loss_and_grads(P, *args, **kw):
    """(loss, readout, {name: grad}) with fresh leaf copies of P (fp64)."""
    leaves = {k: v.detach().double().clone().requires_grad_(True) for k, v in P.items()}
    loss, readout = forward_loss(leaves, *args, **kw)
    names = list(leaves)
    grads = torch.autograd.grad(loss, [leaves[n] for n in names], allow_unused=True)
    return loss.detach(), readout.detach(), {n: (g if g is not None else torch.zeros_like(leaves[n]))
                                             for n, g in zip(names, grads)}
