"""ORACLE — test infrastructure only (see oracle/__init__.py).

fp64 numpy restatement of the optimizer step the training loop wraps around
the LSTM hot path.  The reference ships NO code for it: its semantics are the
SPEC's trainer module,
  adam_step (reference SPEC.md:429-437): m <- b1 m + (1-b1) g;
      v <- b2 v + (1-b2) g^2; bias-corrected m^, v^;
      theta <- theta - lr m^ / (sqrt(v^) + eps); hyperparameters b1=0.9,
      b2=0.999, eps=1e-8; non-finite gradient -> error naming
      the parameter;
  global-norm gradient clipping at 5.0 applied before Adam.
Parity is pinned to the SPEC's worked examples, which the
CPU tests check against this restatement.
"""
from __future__ import annotations

import numpy as np


def adam_step(params, grads, m, v, step, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8,
              grad_scale=1.0, clip_norm=5.0):
    """One step in float64; returns (params, m, v, grad_norm) as new arrays."""
    p = np.asarray(params, np.float64).copy()
    g = np.asarray(grads, np.float64) * grad_scale
    m = np.asarray(m, np.float64).copy()
    v = np.asarray(v, np.float64).copy()
    if not np.all(np.isfinite(g)):
        raise FloatingPointError("non-finite gradient")
    norm = float(np.sqrt(np.sum(g * g)))
    if clip_norm > 0 and norm > clip_norm:          # SPEC.md:484, before Adam
        g = g * (clip_norm / norm)
    m = beta1 * m + (1 - beta1) * g
    v = beta2 * v + (1 - beta2) * g * g
    mhat = m / (1 - beta1 ** step)
    vhat = v / (1 - beta2 ** step)
    p = p - lr * mhat / (np.sqrt(vhat) + eps)
    return p, m, v, norm
