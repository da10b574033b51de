"""The decoder's output layer and training loss over the C ABI (sl_output_ce,
csrc/softmax_ce.cu): logits = x W + b, log_softmax, label-smoothed cross
entropy averaged over the valid positions, and its gradients — the reference's
Softmax layer + ce loss (compiler.cpp:651-663, tape.cpp:879-924, 1224-1298).
Errors map like the reference: epsilon outside [0, 1) -> ValueError
(std::invalid_argument), an out-of-range target id -> IndexError naming the
layer (checked by check_targets(), which synchronises)."""
from __future__ import annotations

import ctypes

import torch

from . import lstm


class OutputCE:
    def __init__(self, batch: int, time: int, input_dim: int, vocab: int, epsilon: float = 0.1,
                 layer: str = "output_prob", device=None, precision: str = "bf16"):
        """precision "bf16": bf16 logits with the fused online-softmax epilogue
        (sl_output_ce); "fp32": the reference's precision — fp32 logits and
        split-bf16 tensor-core GEMMs (sl_output_ce_f32, rel. 1e-4)."""
        self.B, self.T, self.D, self.V = batch, time, input_dim, vocab
        self.eps, self.layer = epsilon, layer
        self.device = torch.device(device or "cuda")
        L = lstm.lib()
        i32 = ctypes.c_int32
        L.sl_output_ce_workspace_size.restype = ctypes.c_size_t
        L.sl_output_ce_workspace_size.argtypes = [i32] * 4
        vp = ctypes.c_void_p
        L.sl_output_ce.argtypes = [i32] * 4 + [vp] * 5 + [ctypes.c_float] + [vp] * 4 + [ctypes.c_int, vp,
                                                                                         ctypes.c_size_t, vp, vp]
        L.sl_output_ce_f32_workspace_size.restype = ctypes.c_size_t
        L.sl_output_ce_f32_workspace_size.argtypes = [i32] * 4
        L.sl_output_ce_f32.argtypes = L.sl_output_ce.argtypes
        if precision not in ("bf16", "fp32"):
            raise ValueError(f"precision must be bf16 or fp32, got {precision!r}")
        self.precision = precision
        self._call = L.sl_output_ce_f32 if precision == "fp32" else L.sl_output_ce
        self.ws_bytes = (L.sl_output_ce_f32_workspace_size if precision == "fp32" else
                         L.sl_output_ce_workspace_size)(batch, time, input_dim, vocab)
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.loss = torch.zeros((), dtype=torch.float32, device=self.device)
        self.bad = torch.zeros(1, dtype=torch.int32, device=self.device)

    def forward_backward(self, x, targets, seq_lens, W, b, dx=None, dW=None, db=None, accumulate=False,
                         need_dx=True):
        B, T, D, V = self.B, self.T, self.D, self.V
        lstm._need(x, (B, T, D), "x")
        lstm._need(targets, (B, T), "targets", torch.int32)
        lstm._need(seq_lens, (B,), "seq_lens", torch.int32)
        lstm._need(W, (D, V), "W")
        lstm._need(b, (V,), "b")
        dev = self.device
        if dx is None and need_dx:
            dx = torch.empty(B, T, D, dtype=torch.float32, device=dev)
        if dW is None:
            dW = torch.empty(D, V, dtype=torch.float32, device=dev)
        if db is None:
            db = torch.empty(V, dtype=torch.float32, device=dev)
        lstm._check(self._call(B, T, D, V, lstm._p(x), lstm._p(targets), lstm._p(seq_lens),
                                            lstm._p(W), lstm._p(b), self.eps, lstm._p(self.loss), lstm._p(dx),
                                            lstm._p(dW), lstm._p(db), int(accumulate), lstm._p(self.workspace),
                                            self.ws_bytes, lstm._p(self.bad), lstm._stream()))
        return self.loss, dx, dW, db

    def check_targets(self, targets=None):
        """Synchronise; raise IndexError like the reference (tape.cpp:1265-1268)."""
        if int(self.bad.item()) == 0:
            return
        what = ""
        if targets is not None:
            bad = targets[(targets < 0) | (targets >= self.V)]
            if bad.numel():
                what = f"target id {int(bad[0])} "
        raise IndexError(f"{what}out of range [0, {self.V}) in layer '{self.layer}'")
