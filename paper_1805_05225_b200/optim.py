"""Adam with global-norm clipping over the flat parameter buffer (C ABI
sl_adam_step, csrc/adam.cu) — the optimizer of the config-4 training step
(reference SPEC.md:429-437 adam_step; clip 5.0 before Adam).
Asynchronous on the current stream; check_finite() synchronises and raises
like the reference ("non-finite gradient -> error naming the parameter")."""
from __future__ import annotations

import ctypes
from typing import Sequence, Tuple

import torch

from . import lstm


class Adam:
    def __init__(self, params: torch.Tensor, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 clip_norm: float = 5.0, names: Sequence[Tuple[str, int, int]] = ()):
        if params.dtype != torch.float32 or not params.is_cuda or not params.is_contiguous():
            raise ValueError("Adam: params must be one contiguous CUDA fp32 buffer")
        self.params = params
        self.lr, self.betas, self.eps, self.clip_norm = lr, betas, eps, clip_norm
        self.names = list(names)  # (name, offset, numel) for error messages
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        self.t = 0
        L = lstm.lib()
        L.sl_adam_scratch_size.restype = ctypes.c_size_t
        # the scratch also carries the device-side step counter (step == 0 below),
        # so the step can be captured in a CUDA graph and replayed
        self.scratch = torch.zeros(L.sl_adam_scratch_size(), dtype=torch.uint8, device=params.device)
        self.grad_norm = torch.zeros(1, dtype=torch.float32, device=params.device)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=params.device)

    def step(self, grads: torch.Tensor, grad_scale: float = 1.0, lr: float | None = None):
        if grads.shape != self.params.shape or grads.dtype != torch.float32:
            raise lstm.ShapeError(f"Adam.step: grads {tuple(grads.shape)} vs params {tuple(self.params.shape)}")
        self.t += 1
        L = lstm.lib()
        f, vp = ctypes.c_float, ctypes.c_void_p
        L.sl_adam_step.argtypes = [ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int32, f, f, f, f, f, f, vp, vp,
                                   vp, vp]
        lstm._check(L.sl_adam_step(self.params.numel(), lstm._p(self.params), lstm._p(grads), lstm._p(self.m),
                                   lstm._p(self.v), 0, self.lr if lr is None else lr, self.betas[0],
                                   self.betas[1], self.eps, grad_scale, self.clip_norm, lstm._p(self.scratch),
                                   lstm._p(self.grad_norm), lstm._p(self.nonfinite), lstm._stream()))

    # the device-side step counter (AdamScratch::t, csrc/adam.h: after a double
    # and an unsigned) — read / written for checkpoints (checkpoint.py)
    def device_step(self) -> int:
        return int(self.scratch[12:16].view(torch.int32).item())

    def set_device_step(self, t: int) -> None:
        self.scratch[12:16].view(torch.int32).fill_(int(t))
        self.t = int(t)

    def check_finite(self, grads: torch.Tensor | None = None):
        """Synchronise; raise FloatingPointError naming the first parameter whose
        gradient is non-finite (the step was skipped, parameters untouched)."""
        if int(self.nonfinite.item()) == 0:
            return
        name = "<unnamed>"
        if grads is not None:
            for n, off, k in self.names:
                if not torch.isfinite(grads[off:off + k]).all():
                    name = n
                    break
        raise FloatingPointError(f"adam_step: non-finite gradient in parameter {name}")
