"""The caller of the boundary for the BASELINE workload: an L-layer BLSTM encoder.

Mirrors how the reference's executor drives the LSTM path for the Listing-1
encoder: for every `rec` layer enc{l}_{fw,bw}, eval_layer's Rec branch
concatenates the inputs (concat_feature) and calls lstm_sequence with the
layer's `{q}/W, {q}/R, {q}/b` params (compiler.cpp:600-608, param names and
shapes compiler.cpp:485-494, topology models.cpp).  Here each layer is ONE
bidirectional sl_lstm_layer call (both directions concurrent) writing the
[fw ‖ bw] concat in place, and all parameters / gradients live in flat device
buffers so the data-parallel gradient all-reduce can run per layer bucket,
overlapped with the BPTT of the layers below.
"""
from __future__ import annotations

import torch

from . import lstm


class BLSTMEncoder:
    @staticmethod
    def numel(num_layers: int, input_dim: int, hidden: int) -> int:
        H = hidden
        return sum(2 * (D * 4 * H + H * 4 * H + 4 * H)
                   for D in [input_dim] + [2 * H] * (num_layers - 1))

    def __init__(self, num_layers: int, batch: int, time: int, input_dim: int, hidden: int,
                 precision: str = "bf16", device=None, params=None, grads=None, train: bool = True,
                 x0_bf16: bool = False, top_bf16: bool = False):
        """params / grads: optional flat fp32 views (numel() elements) to live in,
        e.g. slices of a whole model's buffers; by default the encoder owns them.
        train=False: inference only (no reserves, no gradients, one workspace
        shared by all layers — BASELINE config 5).  x0_bf16 (bf16): layer 0 takes
        the padded bf16 input directly (e.g. written by the embedding lookup);
        top_bf16 (bf16): the top layer writes that layout too (the attention
        decoder's input, decoder.py) instead of fp32."""
        self.L, self.B, self.T, self.D0, self.H = num_layers, batch, time, input_dim, hidden
        self.precision = precision
        self.device = torch.device(device or "cuda")
        H = hidden
        self.in_dims = [input_dim if l == 0 else 2 * H for l in range(num_layers)]
        # flat parameter / gradient storage, one contiguous bucket per layer
        self.layer_numel = [2 * (D * 4 * H + H * 4 * H + 4 * H) for D in self.in_dims]
        total = sum(self.layer_numel)
        self.params = params if params is not None else torch.empty(total, dtype=torch.float32,
                                                                     device=self.device)
        if grads is None:
            grads = torch.zeros(total if train else 0, dtype=torch.float32, device=self.device)
        self.grads = grads
        self.train = train
        assert self.params.numel() == total and (self.grads.numel() == total or not train)
        self.p_views, self.g_views, self.buckets = [], [], []
        off = 0
        for l, D in enumerate(self.in_dims):
            n = self.layer_numel[l]
            if train:
                self.buckets.append(self.grads[off:off + n])
            pv, gv = [], []
            for _ in range(2):  # fw, bw
                for shape in ((D, 4 * H), (H, 4 * H), (4 * H,)):
                    k = 1
                    for s in shape:
                        k *= s
                    pv.append(self.params[off:off + k].view(shape))
                    if train:
                        gv.append(self.grads[off:off + k].view(shape))
                    off += k
            self.p_views.append(pv)
            self.g_views.append(gv)
        # bf16: the activations between layers stay in the padded bf16 layout the
        # next layer's input GEMM reads (SL_LAYER_Y_BF16 -> SL_LAYER_X_BF16); only
        # the top layer's output is fp32
        # fp32: the same chaining with the split-bf16 images the next layer's fp32-class
        # input GEMM reads (SL_LAYER_Y_X3 -> SL_LAYER_X_X3): no split pass per layer
        chain = precision == "bf16"
        chain_x3 = precision == "fp32" and num_layers > 1 and lstm.PATHS[lstm.lib().sl_lstm_layer_path(
            lstm.ctypes.byref(lstm._Layer(batch, time, 2 * H, H, 2, 1, lstm.PRECISIONS[precision], 0)))] == "fp32_x3_tc"
        last = num_layers - 1 + (1 if chain and top_bf16 else 0)
        fl = lambda l: dict(x_bf16=chain and (l > 0 or x0_bf16), y_bf16=chain and l < last,
                            x_x3=chain_x3 and l > 0, y_x3=chain_x3 and l < num_layers - 1)
        shared = None
        if not train:  # the layers run one after another: one workspace serves all of them
            need = max(lstm.LSTMLayer.workspace_size(batch, time, D, H, 2, 1, precision, **fl(l))
                       for l, D in enumerate(self.in_dims))
            shared = torch.empty(need, dtype=torch.uint8, device=self.device)
        self.layers = [lstm.LSTMLayer(batch, time, D, H, 2, 1, precision, self.device, train=train,
                                      workspace=shared, **fl(l))
                       for l, D in enumerate(self.in_dims)]
        def act(l):  # layer l's output buffer
            if chain and l < last:
                return torch.zeros(batch, time, lstm.bf16_pitch(2 * H), dtype=torch.bfloat16, device=self.device)
            if chain_x3 and l < num_layers - 1:
                return lstm.x3_image(batch, time, 2 * H, self.device)
            return torch.empty(batch, time, 2 * H, dtype=torch.float32, device=self.device)
        if train:
            self.acts = [act(l) for l in range(num_layers)]
        else:  # inference keeps nothing for a backward: the inner layers ping-pong two buffers
            top = num_layers - 1
            inner = [act(l) for l in range(min(2, top))]
            self.acts = [inner[l % 2] for l in range(top)] + [act(top)]
        self.dxs = [torch.empty(batch, time, D, dtype=torch.float32, device=self.device)
                    for D in self.in_dims] if train else []

    def param_names(self):
        """Reference naming (compiler.cpp:488-492): enc{l}_{fw,bw}/{W,R,b}."""
        return [f"enc{l}_{d}/{n}" for l in range(self.L) for d in ("fw", "bw")
                for n in ("W", "R", "b")]

    def param_slices(self):
        """(name, offset, numel) of every parameter inside the flat buffer."""
        out, off = [], 0
        for l, D in enumerate(self.in_dims):
            for d in ("fw", "bw"):
                for n, k in (("W", D * 4 * self.H), ("R", self.H * 4 * self.H), ("b", 4 * self.H)):
                    out.append((f"enc{l}_{d}/{n}", off, k))
                    off += k
        return out

    def init_uniform(self, seed: int = 0):
        """W, R, b ~ U(+-1/sqrt(H)) (SURVEY §8(d) synthetic inputs)."""
        g = torch.Generator(device=self.device).manual_seed(seed)
        s = 1.0 / self.H ** 0.5
        self.params.uniform_(-s, s, generator=g)

    def _wrb(self, l):
        v = self.p_views[l]
        return [v[0], v[3]], [v[1], v[4]], [v[2], v[5]]

    def forward(self, x, seq_lens, train: bool = None):
        train = self.train if train is None else train
        inp = x
        for l in range(self.L):
            W, R, b = self._wrb(l)
            self.layers[l].forward(inp, seq_lens, W, R, b, y=self.acts[l], train=train)
            inp = self.acts[l]
        return inp

    def backward(self, dy, on_layer_grads=None):
        """BPTT from the top layer down; on_layer_grads(l, bucket) fires as soon
        as layer l's gradients are complete (used to start its all-reduce)."""
        g = dy
        for l in reversed(range(self.L)):
            gv = self.g_views[l]
            dx, _, _, _ = self.layers[l].backward(
                g, dx=self.dxs[l], dW=[gv[0], gv[3]], dR=[gv[1], gv[4]], db=[gv[2], gv[5]],
                need_dx=True)
            if on_layer_grads is not None:
                on_layer_grads(l, self.buckets[l])
            g = dx
        return g
