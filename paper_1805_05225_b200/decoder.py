"""The Listing-1 attention decoder over a teacher-forced target sequence, over
the C ABI (sl_attn_decoder_fwd/bwd, csrc/decoder.cu): the reference's `output`
subnetwork — RnnCell `s` (lstm_step on [prev trg ‖ prev att]), weight_feedback,
s_tr, e = tanh(...) v + b, a = softmax_over_spatial, accum_a, att =
generic_attention over the encoder, readout = relu(linear([s, prev trg, att]))
(models.cpp:83-166, run step by step by compiler.cpp:770-905) — plus the base
layer enc_ctx (models.cpp:60).  The output_prob layer and its loss are
output.OutputCE on the readout.

Parameter names follow the reference's qualified manifest names
(compiler.cpp:470-500): enc_ctx/{W,b} and output/{s,weight_feedback,s_tr,e,
readout,trg}/... — see NAMES.  An out-of-range previous-target id raises the
reference's IndexError from check_ids() (which synchronises)."""
from __future__ import annotations

import ctypes

import torch

from . import lstm

# (C ABI field, reference manifest name)
NAMES = [("enc_ctx_W", "enc_ctx/W"), ("enc_ctx_b", "enc_ctx/b"),
         ("s_W", "output/s/W"), ("s_R", "output/s/R"), ("s_b", "output/s/b"),
         ("fb_W", "output/weight_feedback/W"), ("fb_b", "output/weight_feedback/b"),
         ("s_tr_W", "output/s_tr/W"), ("s_tr_b", "output/s_tr/b"),
         ("e_W", "output/e/W"), ("e_b", "output/e/b"),
         ("readout_W", "output/readout/W"), ("readout_b", "output/readout/b"),
         ("trg_W", "output/trg/W")]


def param_shapes(emb: int, enc: int, hidden: int, key: int, readout: int, trg_vocab: int):
    """Reference shapes of every decoder parameter, in NAMES order."""
    E, H, K, R = enc, hidden, key, readout
    return {"enc_ctx_W": (E, K), "enc_ctx_b": (K,), "s_W": (emb + E, 4 * H), "s_R": (H, 4 * H), "s_b": (4 * H,),
            "fb_W": (1, K), "fb_b": (K,), "s_tr_W": (H, K), "s_tr_b": (K,), "e_W": (K, 1), "e_b": (1,),
            "readout_W": (H + emb + E, R), "readout_b": (R,), "trg_W": (trg_vocab, emb)}


class _Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("batch", "src_time", "trg_time", "embed_dim", "enc_dim", "hidden",
                                               "key_dim", "readout_dim", "trg_vocab")]


class _Ptrs(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n, _ in NAMES]


class AttnDecoder:
    def __init__(self, batch: int, src_time: int, trg_time: int, emb: int, enc: int, hidden: int, key: int,
                 readout: int, trg_vocab: int, device=None, layer: str = "output/trg", precision: str = "bf16"):
        """precision "bf16": enc is the padded bf16 encoder output (sl_attn_decoder_*);
        "fp32": the reference's precision — enc fp32 [B, Ts, E], split-bf16 tensor-core
        GEMMs and fp32 attention (sl_attn_decoder_*_f32, rel. 1e-4)."""
        self.B, self.Ts, self.T, self.Emb, self.E, self.H, self.K, self.Rd, self.Vt = (
            batch, src_time, trg_time, emb, enc, hidden, key, readout, trg_vocab)
        self.layer = layer
        self.device = torch.device(device or "cuda")
        self.desc = _Desc(batch, src_time, trg_time, emb, enc, hidden, key, readout, trg_vocab)
        self.shapes = param_shapes(emb, enc, hidden, key, readout, trg_vocab)
        L = lstm.lib()
        vp, P, sz = ctypes.c_void_p, ctypes.POINTER, ctypes.c_size_t
        L.sl_attn_decoder_workspace_size.restype = sz
        L.sl_attn_decoder_workspace_size.argtypes = [P(_Desc)]
        L.sl_attn_decoder_fwd.argtypes = [P(_Desc), P(_Ptrs), vp, ctypes.c_int64, vp, vp, vp, vp, vp, sz, vp]
        L.sl_attn_decoder_bwd.argtypes = [P(_Desc), P(_Ptrs), P(_Ptrs), vp, ctypes.c_int64, vp, vp, vp, vp, vp,
                                          vp, sz, vp]
        L.sl_attn_decoder_f32_workspace_size.restype = sz
        L.sl_attn_decoder_f32_workspace_size.argtypes = [P(_Desc)]
        L.sl_attn_decoder_fwd_f32.argtypes = [P(_Desc), P(_Ptrs), vp, vp, vp, vp, vp, vp, sz, vp]
        L.sl_attn_decoder_bwd_f32.argtypes = [P(_Desc), P(_Ptrs), P(_Ptrs), vp, vp, vp, vp, vp, vp, vp, sz, vp]
        if precision not in ("bf16", "fp32"):
            raise ValueError(f"precision must be bf16 or fp32, got {precision!r}")
        self.precision = precision
        self.ws_bytes = (L.sl_attn_decoder_f32_workspace_size if precision == "fp32" else
                         L.sl_attn_decoder_workspace_size)(ctypes.byref(self.desc))
        if self.ws_bytes == 0:
            raise lstm.ShapeError(L.sl_last_error().decode())
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.bad = torch.full((1,), 2**31 - 1, dtype=torch.int32, device=self.device)

    def _ptrs(self, d, what):
        vals = []
        for n, _ in NAMES:
            t = d[n]
            lstm._need(t, self.shapes[n], f"{what}[{n}]")
            vals.append(t.data_ptr())
        return _Ptrs(*vals)

    def forward(self, enc_bf16, src_lens, prev_ids, params, readout=None):
        """enc_bf16 [B, Ts, ld] (padded bf16 encoder output, 1.0 at column E; fp32
        [B, Ts, E] for precision fp32), prev_ids [B, T] int32 (< 0: the zero initial
        output), params: dict of fp32 tensors (NAMES) -> readout [B, T, Rd] fp32."""
        if self.precision == "fp32":
            lstm._need(enc_bf16, (self.B, self.Ts, self.E), "enc")
        else:
            assert enc_bf16.dtype == torch.bfloat16 and enc_bf16.shape[:2] == (self.B, self.Ts)
        lstm._need(src_lens, (self.B,), "src_lens", torch.int32)
        lstm._need(prev_ids, (self.B, self.T), "prev_ids", torch.int32)
        if readout is None:
            readout = torch.empty(self.B, self.T, self.Rd, dtype=torch.float32, device=self.device)
        self._pp = self._ptrs(params, "params")
        if self.precision == "fp32":
            lstm._check(lstm.lib().sl_attn_decoder_fwd_f32(
                ctypes.byref(self.desc), ctypes.byref(self._pp), enc_bf16.data_ptr(), src_lens.data_ptr(),
                prev_ids.data_ptr(), readout.data_ptr(), self.bad.data_ptr(), self.workspace.data_ptr(),
                self.ws_bytes, lstm._stream()))
            return readout
        lstm._check(lstm.lib().sl_attn_decoder_fwd(
            ctypes.byref(self.desc), ctypes.byref(self._pp), enc_bf16.data_ptr(), enc_bf16.stride(1),
            src_lens.data_ptr(), prev_ids.data_ptr(), readout.data_ptr(), self.bad.data_ptr(),
            self.workspace.data_ptr(), self.ws_bytes, lstm._stream()))
        return readout

    def backward(self, enc_bf16, src_lens, prev_ids, params, readout, d_readout, grads, d_enc=None):
        """Overwrites every tensor in grads (dict, NAMES) and returns d_enc [B, Ts, E]."""
        if d_enc is None:
            d_enc = torch.empty(self.B, self.Ts, self.E, dtype=torch.float32, device=self.device)
        lstm._need(d_readout, (self.B, self.T, self.Rd), "d_readout")
        pp, gp = self._ptrs(params, "params"), self._ptrs(grads, "grads")
        if self.precision == "fp32":
            lstm._check(lstm.lib().sl_attn_decoder_bwd_f32(
                ctypes.byref(self.desc), ctypes.byref(pp), ctypes.byref(gp), enc_bf16.data_ptr(), src_lens.data_ptr(),
                prev_ids.data_ptr(), readout.data_ptr(), d_readout.data_ptr(), d_enc.data_ptr(),
                self.workspace.data_ptr(), self.ws_bytes, lstm._stream()))
            return d_enc
        lstm._check(lstm.lib().sl_attn_decoder_bwd(
            ctypes.byref(self.desc), ctypes.byref(pp), ctypes.byref(gp), enc_bf16.data_ptr(), enc_bf16.stride(1),
            src_lens.data_ptr(), prev_ids.data_ptr(), readout.data_ptr(), d_readout.data_ptr(), d_enc.data_ptr(),
            self.workspace.data_ptr(), self.ws_bytes, lstm._stream()))
        return d_enc

    def check_ids(self, prev_ids=None):
        """Synchronise; raise IndexError like the reference (tape.cpp:455-460)."""
        row = int(self.bad.item())
        if row == 2**31 - 1:
            return
        what = f"id {int(prev_ids.reshape(-1)[row])} " if prev_ids is not None else ""
        raise IndexError(f"{what}out of range [0, {self.Vt}) in layer '{self.layer}'")
