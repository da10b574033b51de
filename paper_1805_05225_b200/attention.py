"""The decoder's MLP attention step over the C ABI (sl_attention_step_fwd/bwd,
csrc/attention.cu) — one step of the Listing-1 attention subnet (reference
models.cpp:107-154: s_tr, weight_feedback, e = tanh(...) v + b, a =
softmax_over_spatial(e), accum_a, att = generic_attention(a, encoder))."""
from __future__ import annotations

import ctypes

import torch

from . import lstm


class _Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("batch", "src_time", "key_dim", "enc_dim", "state_dim")]


class Attention:
    def __init__(self, batch: int, src_time: int, key_dim: int, enc_dim: int, state_dim: int, device=None):
        self.B, self.Ts, self.K, self.E, self.H = batch, src_time, key_dim, enc_dim, state_dim
        self.desc = _Desc(batch, src_time, key_dim, enc_dim, state_dim)
        self.device = torch.device(device or "cuda")
        L = lstm.lib()
        vp, P = ctypes.c_void_p, ctypes.POINTER
        L.sl_attention_workspace_size.restype = ctypes.c_size_t
        L.sl_attention_workspace_size.argtypes = [P(_Desc)]
        L.sl_attention_step_fwd.argtypes = [P(_Desc)] + [vp] * 15 + [ctypes.c_size_t, vp]
        L.sl_attention_step_bwd.argtypes = [P(_Desc)] + [vp] * 23 + [ctypes.c_int, vp, ctypes.c_size_t, vp]
        self.ws_bytes = L.sl_attention_workspace_size(ctypes.byref(self.desc))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)

    def forward(self, src_lens, enc_ctx, enc, s, accum, W_s, b_s, W_fb, b_fb, v, b_v):
        """Returns (att [B, E], a [B, Ts], accum' [B, Ts])."""
        B, Ts, E = self.B, self.Ts, self.E
        att = torch.empty(B, E, device=self.device)
        a = torch.empty(B, Ts, device=self.device)
        acc2 = torch.empty(B, Ts, device=self.device)
        p = lstm._p
        lstm._check(lstm.lib().sl_attention_step_fwd(
            ctypes.byref(self.desc), p(src_lens), p(enc_ctx), p(enc), p(s), p(accum), p(W_s), p(b_s), p(W_fb),
            p(b_fb), p(v), p(b_v), p(att), p(a), p(acc2), p(self.ws), self.ws_bytes, lstm._stream()))
        return att, a, acc2

    def backward(self, src_lens, enc_ctx, enc, s, accum, W_s, b_s, W_fb, b_fb, v, a, d_att, d_accum_out=None,
                 accumulate=False):
        """Returns a dict of the gradients of every input."""
        B, Ts, K, E, H = self.B, self.Ts, self.K, self.E, self.H
        dev = self.device
        g = {"enc_ctx": torch.empty(B, Ts, K, device=dev), "enc": torch.empty(B, Ts, E, device=dev),
             "s": torch.empty(B, H, device=dev), "accum": torch.empty(B, Ts, device=dev),
             "W_s": torch.empty(H, K, device=dev), "b_s": torch.empty(K, device=dev),
             "W_fb": torch.empty(1, K, device=dev), "b_fb": torch.empty(K, device=dev),
             "v": torch.empty(K, 1, device=dev), "b_v": torch.empty(1, device=dev)}
        p = lstm._p
        lstm._check(lstm.lib().sl_attention_step_bwd(
            ctypes.byref(self.desc), p(src_lens), p(enc_ctx), p(enc), p(s), p(accum), p(W_s), p(b_s), p(W_fb),
            p(b_fb), p(v), p(a), p(d_att), p(d_accum_out), p(g["enc_ctx"]), p(g["enc"]), p(g["s"]), p(g["accum"]),
            p(g["W_s"]), p(g["b_s"]), p(g["W_fb"]), p(g["b_fb"]), p(g["v"]), p(g["b_v"]), int(accumulate),
            p(self.ws), self.ws_bytes, lstm._stream()))
        return g
