"""Embedding lookup over the C ABI (sl_embedding_*, csrc/embedding.cu) — the
reference's Linear layer applied to ids, gather_rows(table = {layer}/W, ids)
(compiler.cpp:584-589, tape.cpp:448-492), and its scatter-add adjoint in the
reference's summation order.  An id outside [0, V) raises IndexError naming
the layer, like the reference (tape.cpp:464-467); the check synchronises, so
callers that stay asynchronous (a captured step) call check_ids() later."""
from __future__ import annotations

import ctypes

import torch

from . import lstm

_NONE = 2 ** 31 - 1  # *bad_row when every id is in range
SL_EMB_ONES_COLUMN, SL_EMB_NEGATIVE_ZERO = 1, 2  # include/seqloom_cuda.h sl_embedding_flags


class Embedding:
    def __init__(self, vocab: int, dim: int, max_ids: int, layer: str = "emb", device=None):
        self.V, self.D, self.layer = vocab, dim, layer
        self.device = torch.device(device or "cuda")
        L = lstm.lib()
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.sl_embedding_workspace_size.restype = ctypes.c_size_t
        L.sl_embedding_workspace_size.argtypes = [i64, i32]
        L.sl_embedding_fwd.argtypes = [i64, vp, i32, i32, vp, vp, i64, ctypes.c_int, vp, vp]
        L.sl_embedding_fwd_bf16.argtypes = [i64, vp, i32, i32, vp, vp, i64, ctypes.c_int, vp, vp]
        L.sl_embedding_bwd.argtypes = [i64, vp, i32, i32, vp, i64, vp, ctypes.c_int, vp, ctypes.c_size_t, vp]
        self.max_ids = max_ids
        self.ws_bytes = L.sl_embedding_workspace_size(max_ids, vocab)
        self.workspace = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=self.device)
        self.bad = torch.full((1,), _NONE, dtype=torch.int32, device=self.device)
        self._ids = None

    def _ids_ok(self, ids):
        if ids.dtype != torch.int32 or not ids.is_cuda or not ids.is_contiguous():
            raise ValueError(f"ids: expected contiguous CUDA int32, got {ids.dtype} {ids.device}")
        if ids.numel() > self.max_ids:
            raise lstm.ShapeError(f"ids: {ids.numel()} ids exceed max_ids={self.max_ids}")

    @staticmethod
    def _rows(t, lead, name, dtype):
        """t viewed as rows: leading dims `lead` contiguous-compatible, last dim
        strided by its row stride (a column slice of a wider buffer is fine)."""
        if t.dtype != dtype or not t.is_cuda or tuple(t.shape[:-1]) != tuple(lead) or t.stride(-1) != 1:
            raise ValueError(f"{name}: expected CUDA {dtype} [{', '.join(map(str, lead))}, *] with unit "
                             f"last stride, got {t.dtype} {tuple(t.shape)}")
        ld = t.stride(-2) if t.dim() > 1 else t.shape[-1]
        for i in range(t.dim() - 2):  # leading dims must flatten onto the row stride
            if t.stride(i) != t.stride(i + 1) * t.shape[i + 1]:
                raise ValueError(f"{name}: leading dimensions must be dense over the row stride")
        return ld

    def forward(self, ids, table, out=None, bf16_pitch: int | None = None, negative_zero: bool = False):
        """out = table[ids]: fp32 [*ids.shape, D] (or a [.., >= D] column slice of a
        wider buffer, written in [0, D)), or with bf16_pitch the padded bf16 layer-0
        LSTM input [*ids.shape, pitch] with the ones column at D.  negative_zero:
        ids < 0 give zero rows (the previous-target embedding at t = 0)."""
        self._ids_ok(ids)
        lstm._need(table, (self.V, self.D), "table")
        n = ids.numel()
        L = lstm.lib()
        flags = SL_EMB_NEGATIVE_ZERO if negative_zero else 0
        if bf16_pitch is None and (out is None or out.dtype == torch.float32):
            if out is None:
                out = torch.empty(*ids.shape, self.D, dtype=torch.float32, device=self.device)
            ld = self._rows(out, ids.shape, "out", torch.float32)
            lstm._check(L.sl_embedding_fwd(n, lstm._p(ids), self.V, self.D, lstm._p(table), lstm._p(out), ld,
                                           flags, lstm._p(self.bad), lstm._stream()))
        else:
            if bf16_pitch is not None:
                flags |= SL_EMB_ONES_COLUMN
                if out is None:
                    out = torch.empty(*ids.shape, bf16_pitch, dtype=torch.bfloat16, device=self.device)
                lstm._need(out, tuple(ids.shape) + (bf16_pitch,), "out", torch.bfloat16)
            ld = self._rows(out, ids.shape, "out", torch.bfloat16)
            lstm._check(L.sl_embedding_fwd_bf16(n, lstm._p(ids), self.V, self.D, lstm._p(table), lstm._p(out),
                                                ld, flags, lstm._p(self.bad), lstm._stream()))
        self._ids = ids
        return out

    def backward(self, ids, d_out, d_table, accumulate: bool = False):
        """d_table (+)= scatter of the d_out rows by id (ascending row order per id);
        d_out may be a [.., >= D] column slice of a wider fp32 buffer."""
        self._ids_ok(ids)
        ld = self._rows(d_out, ids.shape, "d_out", torch.float32)
        lstm._need(d_table, (self.V, self.D), "d_table")
        lstm._check(lstm.lib().sl_embedding_bwd(ids.numel(), lstm._p(ids), self.V, self.D, lstm._p(d_out), ld,
                                                lstm._p(d_table), int(accumulate), lstm._p(self.workspace),
                                                self.ws_bytes, lstm._stream()))
        return d_table

    def check_ids(self, ids=None):
        """Synchronise; raise IndexError like the reference for the first bad id."""
        row = int(self.bad.item())
        if row == _NONE:
            return
        ids = self._ids if ids is None else ids
        v = int(ids.reshape(-1)[row]) if ids is not None else None
        raise IndexError(f"id {v} out of range [0, {self.V}) in layer '{self.layer}'")
