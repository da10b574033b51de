"""ORACLE — test infrastructure only (tests/ may import it; the product never does).

The same restatement as lstm_oracle.c, written with torch fp64 tensor ops so
the GPU parity tests can check full BASELINE-sized layers (config 2:
B=128, T=60, H=1024) in seconds, on the GPU box, without /root/reference.
It is pinned to lstm_oracle.c at small sizes by tests/test_oracle.py, which is
in turn pinned to the reference build and the golden fixtures.

Follows reference layers.cpp:22-36 (sequence, direction, mask),
tape.cpp:1103-1135 (step forward), tape.cpp:1152-1215 (step backward),
tape.cpp:846 (per-sequence prefix reversal).
"""
from __future__ import annotations

import torch


def _src_index(lens: torch.Tensor, T: int, direction: int) -> torch.Tensor:
    """[B, T] long: source time of processing step s per row (tape.cpp:846)."""
    s = torch.arange(T, device=lens.device).unsqueeze(0).expand(lens.numel(), T)
    if direction > 0:
        return s
    L = lens.long().unsqueeze(1)
    return torch.where(s < L, L - 1 - s, s)


def sequence(x, lens, W, R, b, direction, dy=None, dh_last=None, dc_last=None):
    """fp64 forward (+ backward when dy is given) of lstm_sequence.

    Returns dict with y, h_last, c_last and (if dy) dx, dW, dR, db.
    """
    x, W, R, b = (t.double() for t in (x, W, R, b))
    B, T, D = x.shape
    H = R.shape[0]
    dev = x.device
    lens = lens.to(dev)
    src = _src_index(lens, T, direction)                     # [B, T]
    rows = torch.arange(B, device=dev)
    xs = x[rows.unsqueeze(1), src]                            # [B, T, D] processing order
    h = torch.zeros(B, H, dtype=torch.float64, device=dev)
    c = torch.zeros_like(h)
    hs, cs, acts = [h], [c], []
    for s in range(T):
        z = xs[:, s] @ W + h @ R + b
        i, f = torch.sigmoid(z[:, :H]), torch.sigmoid(z[:, H:2 * H])
        g, o = torch.tanh(z[:, 2 * H:3 * H]), torch.sigmoid(z[:, 3 * H:])
        c = f * c + i * g
        tc = torch.tanh(c)
        h = o * tc
        hs.append(h)
        cs.append(c)
        if dy is not None:  # forward-only calls keep no per-step activations
            acts.append((i, f, g, o, tc))
    Hs = torch.stack(hs[1:], 1)                               # [B, T, H] processing order
    valid = torch.arange(T, device=dev).unsqueeze(0) < lens.long().unsqueeze(1)
    y = torch.zeros(B, T, H, dtype=torch.float64, device=dev)
    y[rows.unsqueeze(1), src] = Hs * valid.unsqueeze(-1)
    last = (lens.long() - 1)
    out = {"y": y, "h_last": Hs[rows, last], "c_last": torch.stack(cs[1:], 1)[rows, last]}
    if dy is None:
        return out
    dy = dy.double()
    gext = dy[rows.unsqueeze(1), src] * valid.unsqueeze(-1)   # [B, T, H] processing order
    gh = torch.zeros(B, H, dtype=torch.float64, device=dev)
    gc = torch.zeros_like(gh)
    dxs = torch.zeros(B, T, D, dtype=torch.float64, device=dev)
    dW, dR = torch.zeros_like(W), torch.zeros_like(R)
    db = torch.zeros_like(b)
    for s in range(T - 1, -1, -1):
        gh = gh + gext[:, s]
        at_last = (last == s).unsqueeze(1)
        if dh_last is not None:
            gh = gh + dh_last.double() * at_last
        if dc_last is not None:
            gc = gc + dc_last.double() * at_last
        i, f, g, o, tc = acts[s]
        d_o = gh * tc
        dcn = gc + gh * o * (1 - tc * tc)
        dz = torch.cat([dcn * g * i * (1 - i), dcn * cs[s] * f * (1 - f),
                        dcn * i * (1 - g * g), d_o * o * (1 - o)], 1)
        gc = dcn * f
        gh = dz @ R.t()
        dxs[:, s] = dz @ W.t()
        dW += xs[:, s].t() @ dz
        dR += hs[s].t() @ dz
        db += dz.sum(0)
    dx = torch.zeros_like(x)
    dx[rows.unsqueeze(1), src] = dxs
    out.update(dx=dx, dW=dW, dR=dR, db=db)
    return out
