"""The reference's input dropout over the C ABI (sl_dropout_fwd/bwd, csrc/dropout.cu):
Tape::dropout (tape.cpp:540-600) as eval_layer applies it to a layer input
(compiler.cpp:554-562) — a counter-based mask (rng.hpp) that is a pure function of
(seed, layer, input index, batch counter, position), bit-identical to the reference
and recomputed in the backward.  An invalid rate raises ValueError
(std::invalid_argument, tape.cpp:541-544)."""
from __future__ import annotations

import ctypes

from . import lstm

_M64 = (1 << 64) - 1


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def _mix64(a: int, b: int) -> int:
    return _splitmix64(a ^ ((_splitmix64(b) + 0x9E3779B97F4A7C15) & _M64))


def _fnv1a(s: str) -> int:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h = ((h ^ ch) * 0x100000001B3) & _M64
    return h


def layer_key(seed: int, layer: str, input_index: int = 0) -> int:
    """key0 = mix64(seed, fnv1a("<layer>#<input index>")) (compiler.cpp:559); the
    per-batch key mixes in the batch counter on the device."""
    return _mix64(seed & _M64, _fnv1a(f"{layer}#{input_index}"))


class Dropout:
    def __init__(self, rate: float, seed: int, layer: str, input_index: int = 0):
        if not 0.0 <= rate < 1.0:
            raise ValueError(f"dropout rate must be in [0, 1), got {rate}")
        self.rate, self.key0 = float(rate), layer_key(seed, layer, input_index)
        L = lstm.lib()
        args = [ctypes.c_int32] * 3 + [ctypes.c_float, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.sl_dropout_fwd.argtypes = args
        L.sl_dropout_bwd.argtypes = args

    def _call(self, fn, x, out, counter, counter_value):
        B, T, F = x.shape
        lstm._check(fn(B, T, F, self.rate, self.key0, lstm._p(counter), int(counter_value), lstm._p(x),
                       lstm._p(out), lstm._stream()))
        return out

    def forward(self, x, out, counter=None, counter_value: int = 0):
        """x, out [B, T, F] fp32 device; counter: device int32 batch counter (or counter_value)."""
        return self._call(lstm.lib().sl_dropout_fwd, x, out, counter, counter_value)

    def backward(self, dy, dx, counter=None, counter_value: int = 0):
        return self._call(lstm.lib().sl_dropout_bwd, dy, dx, counter, counter_value)
