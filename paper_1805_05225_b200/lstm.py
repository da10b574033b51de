"""Python mirror of the reference's LSTM-layer interface over the C ABI.

The reference's public surface for this path is

    NodeId seqloom::lstm_sequence(Tape&, NodeId W, NodeId R, NodeId b, NodeId xs, int direction)
        reference core/include/seqloom/layers.hpp:17, core/src/layers.cpp:8-37
    Tape::LstmOut Tape::lstm_step(W, R, b, x, h_prev, c_prev)
        reference core/include/seqloom/tape.hpp:123-129, core/src/tape.cpp:1074-1222

This module exposes the same operations on device tensors (torch is used only
for device memory and streams) by calling ``lib/libseqloom_cuda.so`` through
ctypes — the same C ABI (include/seqloom_cuda.h) a C++ or cgo/JNI host binds.
There is no CPU path: if the library or a CUDA device is missing, every entry
point raises.  Errors map like the reference: invalid direction ->
ValueError (std::invalid_argument, layers.cpp:14-16); bad shapes ->
ShapeError (seqloom::ShapeError, tape.cpp:1092-1094).
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SL_LIB_PATH") or os.path.join(_PKG, "lib", "libseqloom_cuda.so")

SL_OK, SL_ERR_INVALID_ARGUMENT, SL_ERR_SHAPE, SL_ERR_CUDA, SL_ERR_WORKSPACE, SL_ERR_UNSUPPORTED = range(6)
PRECISIONS = {"fp32": 0, "bf16": 1}
PATHS = {1: "bf16_tc", 2: "fp32_x3_tc", 3: "fp32_simt"}  # seqloom_cuda.h enum sl_path
SL_LAYER_X_BF16, SL_LAYER_Y_BF16 = 1, 2
SL_LAYER_X_X3, SL_LAYER_Y_X3 = 16, 32


def x3_image(batch: int, time: int, features: int, device=None) -> "torch.Tensor":
    """A zero-initialised split-bf16 activation image of [batch, time, features]
    (SL_LAYER_Y_X3 / SL_LAYER_X_X3): two bf16 planes [2, batch*time, pitch]."""
    return torch.zeros((2, batch * time, bf16_pitch(features)), dtype=torch.bfloat16, device=device)


def bf16_pitch(features: int) -> int:
    """Row pitch of the padded bf16 activation layout (seqloom_cuda.h sl_lstm_bf16_pitch)."""
    return (features + 1 + 63) // 64 * 64


class ShapeError(RuntimeError):
    """Mirror of seqloom::ShapeError (reference tensor.hpp:37-40)."""


class _Layer(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("batch", "time", "input_dim", "hidden", "num_dirs", "direction", "precision",
                 "flags")]


_lib = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_1805_05225_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32
        P = ctypes.POINTER
        L.sl_version.restype = ctypes.c_int
        L.sl_last_error.restype = ctypes.c_char_p
        L.sl_lstm_layer_check.argtypes = [P(_Layer)]
        L.sl_lstm_layer_path.argtypes = [P(_Layer)]
        L.sl_lstm_reserve_size.restype = sz
        L.sl_lstm_reserve_size.argtypes = [P(_Layer)]
        L.sl_lstm_workspace_size.restype = sz
        L.sl_lstm_workspace_size.argtypes = [P(_Layer)]
        L.sl_lstm_layer_fwd.argtypes = [P(_Layer), vp, vp, P(vp), P(vp), P(vp), vp, vp, vp, vp, sz,
                                        vp, sz, vp]
        L.sl_lstm_layer_bwd.argtypes = [P(_Layer), vp, vp, P(vp), P(vp), vp, vp, vp, vp, P(vp),
                                        P(vp), P(vp), ctypes.c_int, vp, sz, vp, sz, vp]
        L.sl_lstm_bf16_pitch.restype = ctypes.c_int64
        L.sl_lstm_bf16_pitch.argtypes = [i32]
        L.sl_lstm_cell_fwd.argtypes = [i32, i32, i32, i32] + [vp] * 9 + [vp]
        L.sl_lstm_cell_bwd.argtypes = [i32, i32, i32, i32] + [vp] * 14 + [ctypes.c_int, vp]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == SL_OK:
        return
    msg = lib().sl_last_error().decode()
    if rc == SL_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == SL_ERR_SHAPE:
        raise ShapeError(msg)
    raise RuntimeError(f"seqloom_cuda error {rc}: {msg}")


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _arr(ts):
    return (ctypes.c_void_p * len(ts))(*[None if t is None else t.data_ptr() for t in ts])


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need(t, shape, name, dtype=torch.float32):
    if t.dtype != dtype or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name}: expected contiguous CUDA {dtype}, got {t.dtype} {t.device}")
    if tuple(t.shape) != tuple(shape):
        raise ShapeError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")


class LSTMLayer:
    """One LSTM layer (1 or 2 directions over the same input) on the GPU.

    forward() is lstm_sequence for every direction (bidirectional = the
    Listing-1 enc{i}_fw / enc{i}_bw pair with outputs concatenated [fw ‖ bw],
    compiler.cpp:600-608); backward() is the adjoint of everything that
    forward put on the reference tape.  Weights are per direction in the
    reference layout W [D, 4H], R [H, 4H], b [4H] with gate blocks (i,f,g,o).
    """

    def __init__(self, batch: int, time: int, input_dim: int, hidden: int, num_dirs: int = 1,
                 direction: int = 1, precision: str = "fp32", device=None, x_bf16: bool = False,
                 y_bf16: bool = False, train: bool = True, workspace=None, x_x3: bool = False,
                 y_x3: bool = False):
        # x_bf16 / y_bf16: padded bf16 activations between stacked layers
        # (SL_LAYER_X_BF16 / SL_LAYER_Y_BF16, bf16 precision only); x_x3 / y_x3: the
        # split-bf16 images instead (SL_LAYER_X_X3 / SL_LAYER_Y_X3, fp32 precision, x3_image()).
        # train=False: an inference-only layer (the reference's grad-disabled
        # Tape(false), tape.cpp:103) — no reserve is allocated and forward()
        # saves nothing.  workspace: an optional caller-owned uint8 buffer of at
        # least workspace_size() bytes (stacked inference layers can share one).
        flags = (SL_LAYER_X_BF16 if x_bf16 else 0) | (SL_LAYER_Y_BF16 if y_bf16 else 0) | \
            (SL_LAYER_X_X3 if x_x3 else 0) | (SL_LAYER_Y_X3 if y_x3 else 0)
        self.x_bf16, self.y_bf16, self.x_x3, self.y_x3 = x_bf16, y_bf16, x_x3, y_x3
        self.desc = _Layer(batch, time, input_dim, hidden, num_dirs, direction,
                           PRECISIONS[precision], flags)
        self.device = torch.device(device or "cuda")
        L = lib()
        _check(L.sl_lstm_layer_check(ctypes.byref(self.desc)))
        self.reserve_bytes = L.sl_lstm_reserve_size(ctypes.byref(self.desc))
        self.workspace_bytes = L.sl_lstm_workspace_size(ctypes.byref(self.desc))
        if workspace is not None:
            if workspace.dtype != torch.uint8 or workspace.numel() < self.workspace_bytes:
                raise ValueError(f"workspace: need >= {self.workspace_bytes} uint8 bytes")
            self.workspace = workspace
        else:
            self.workspace = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=self.device)
        self.train = train
        if not train:
            self.reserve_bytes = 0
        self.reserve = torch.empty(self.reserve_bytes, dtype=torch.uint8, device=self.device) if train else None
        self._saved = None

    @staticmethod
    def workspace_size(batch, time, input_dim, hidden, num_dirs=1, direction=1, precision="fp32",
                       x_bf16=False, y_bf16=False, x_x3=False, y_x3=False) -> int:
        flags = (SL_LAYER_X_BF16 if x_bf16 else 0) | (SL_LAYER_Y_BF16 if y_bf16 else 0) | \
            (SL_LAYER_X_X3 if x_x3 else 0) | (SL_LAYER_Y_X3 if y_x3 else 0)
        d = _Layer(batch, time, input_dim, hidden, num_dirs, direction, PRECISIONS[precision], flags)
        return lib().sl_lstm_workspace_size(ctypes.byref(d))

    @property
    def path(self) -> str:
        """The kernels this layer runs on: "bf16_tc", "fp32_x3_tc" (fp32-class on
        the tensor cores) or "fp32_simt" (sl_lstm_layer_path)."""
        return PATHS[lib().sl_lstm_layer_path(ctypes.byref(self.desc))]

    @property
    def shape(self):
        d = self.desc
        return d.batch, d.time, d.input_dim, d.hidden, d.num_dirs

    def forward(self, x, seq_lens, W: Sequence, R: Sequence, b: Sequence, y=None, h_last=None,
                c_last=None, train: bool = True):
        B, T, D, H, nd = self.shape
        if train and not self.train:
            raise RuntimeError("forward(train=True) on an inference-only layer (constructed with train=False)")
        if self.x_bf16:
            _need(x, (B, T, bf16_pitch(D)), "x", torch.bfloat16)
        elif self.x_x3:
            _need(x, (2, B * T, bf16_pitch(D)), "x", torch.bfloat16)
        else:
            _need(x, (B, T, D), "x")
        _need(seq_lens, (B,), "seq_lens", torch.int32)
        for k in range(nd):
            _need(W[k], (D, 4 * H), f"W[{k}]")
            _need(R[k], (H, 4 * H), f"R[{k}]")
            _need(b[k], (4 * H,), f"b[{k}]")
        if y is None and self.y_bf16:
            y = torch.zeros((B, T, bf16_pitch(nd * H)), dtype=torch.bfloat16, device=self.device)
        elif y is None and self.y_x3:
            y = x3_image(B, T, nd * H, self.device)
        elif y is None:
            y = torch.empty((B, T, nd * H), dtype=torch.float32, device=self.device)
        elif self.y_bf16:
            _need(y, (B, T, bf16_pitch(nd * H)), "y", torch.bfloat16)
        elif self.y_x3:
            _need(y, (2, B * T, bf16_pitch(nd * H)), "y", torch.bfloat16)
        if h_last is None:
            h_last = torch.empty((nd, B, H), dtype=torch.float32, device=self.device)
        if c_last is None:
            c_last = torch.empty((nd, B, H), dtype=torch.float32, device=self.device)
        _check(lib().sl_lstm_layer_fwd(
            ctypes.byref(self.desc), _p(x), _p(seq_lens), _arr(W), _arr(R), _arr(b), _p(y),
            _p(h_last), _p(c_last), _p(self.reserve) if train else None,
            self.reserve_bytes if train else 0, _p(self.workspace), self.workspace_bytes,
            _stream()))
        self._saved = (x, seq_lens, list(W), list(R)) if train else None
        return y, h_last, c_last

    def backward(self, dy, dh_last=None, dc_last=None, dx=None, dW=None, dR=None, db=None,
                 accumulate: bool = False, need_dx: bool = True):
        if self._saved is None:
            raise RuntimeError("backward() needs a preceding forward(train=True)")
        x, seq_lens, W, R = self._saved
        B, T, D, H, nd = self.shape
        _need(dy, (B, T, nd * H), "dy")
        dev = self.device
        if dx is None and need_dx:
            dx = torch.empty((B, T, D), dtype=torch.float32, device=dev)
        if dW is None:
            dW = [torch.empty((D, 4 * H), dtype=torch.float32, device=dev) for _ in range(nd)]
        if dR is None:
            dR = [torch.empty((H, 4 * H), dtype=torch.float32, device=dev) for _ in range(nd)]
        if db is None:
            db = [torch.empty((4 * H,), dtype=torch.float32, device=dev) for _ in range(nd)]
        _check(lib().sl_lstm_layer_bwd(
            ctypes.byref(self.desc), _p(x), _p(seq_lens), _arr(W), _arr(R), _p(dy), _p(dh_last),
            _p(dc_last), _p(dx), _arr(dW), _arr(dR), _arr(db), int(accumulate), _p(self.reserve),
            self.reserve_bytes, _p(self.workspace), self.workspace_bytes, _stream()))
        return dx, dW, dR, db


def lstm_sequence(x, seq_lens, W, R, b, direction: int, precision: str = "fp32"):
    """Forward of reference ``lstm_sequence`` (layers.cpp:8-37): returns y [B, T, H]."""
    if direction not in (1, -1):
        raise ValueError("lstm_sequence: direction must be +1 or -1")
    if x.dim() != 3:
        raise ShapeError(f"lstm_sequence: input needs Batch and Time axes, got {tuple(x.shape)}")
    B, T, D = x.shape
    H = R.shape[0]
    layer = LSTMLayer(B, T, D, H, 1, direction, precision, x.device)
    y, _, _ = layer.forward(x, seq_lens, [W], [R], [b], train=False)
    return y


def lstm_step(x, h0, c0, W, R, b, precision: str = "fp32", saved=None):
    """Tape::lstm_step forward (tape.cpp:1074-1141): returns (h, c, saved[B,5H])."""
    B, D = x.shape
    H = R.shape[0]
    for t, shp, n in ((h0, (B, H), "h_prev"), (c0, (B, H), "c_prev"), (W, (D, 4 * H), "W"),
                      (R, (H, 4 * H), "R"), (b, (4 * H,), "b")):
        _need(t, shp, f"lstm_step: {n}")
    h = torch.empty((B, H), dtype=torch.float32, device=x.device)
    c = torch.empty((B, H), dtype=torch.float32, device=x.device)
    if saved is None:
        saved = torch.empty((B, 5 * H), dtype=torch.float32, device=x.device)
    _check(lib().sl_lstm_cell_fwd(B, D, H, PRECISIONS[precision], _p(x), _p(h0), _p(c0), _p(W),
                                  _p(R), _p(b), _p(h), _p(c), _p(saved), _stream()))
    return h, c, saved


def lstm_step_backward(x, h0, c0, W, R, saved, gh=None, gc=None, precision: str = "fp32"):
    """The lstm_step backward closure (tape.cpp:1142-1219): (dx, dh0, dc0, dW, dR, db)."""
    B, D = x.shape
    H = R.shape[0]
    dev = x.device
    out = [torch.empty(s, dtype=torch.float32, device=dev)
           for s in ((B, D), (B, H), (B, H), (D, 4 * H), (H, 4 * H), (4 * H,))]
    _check(lib().sl_lstm_cell_bwd(B, D, H, PRECISIONS[precision], _p(x), _p(h0), _p(c0), _p(W),
                                  _p(R), _p(saved), _p(gh), _p(gc), *[_p(o) for o in out], 0,
                                  _stream()))
    return tuple(out)
