"""The config-4 training step around the LSTM hot path (BASELINE configs[3]).

Two models:
- Seq2SeqAttention (below Seq2SeqLSTM) is the bench workload: the full
  Listing-1 step (models.cpp:17-184) with the MLP attention decoder, the relu
  readout, dropout and the output softmax + label-smoothed CE.
- Seq2SeqLSTM is the simpler pre-attention step (`bench.py --no-attention`):
  6-layer BLSTM encoder + one decoder LSTM layer + the output layer, fwd + bwd,
  data-parallel gradient all-reduce, fused clip + Adam.  Its decoder input is
  [target embedding ‖ context] with the context stand-in c_t = encoder output
  at t (an identity alignment, T_src = T_tgt), so encoder gradients still flow
  through the decoder as they do through attention.  The output layer reads
  the decoder state directly, and the decoder runs as one unidirectional LSTM
  layer over the teacher-forced inputs.

With src_vocab / trg_vocab the step starts from token ids like the
reference: the `src` layer's embedding lookup feeds encoder layer 0 (written
straight into its padded bf16 input), and the `trg` layer's lookup of the
PREVIOUS target (zero at t = 0: initial_output 0, models.cpp:94-97) fills
the embedding half of the decoder input; their backward passes scatter-add
into the two tables (embedding.py).

All parameters (encoder then decoder) and their gradients live in ONE flat
fp32 buffer each: the gradient all-reduce buckets are slices of it and the
optimizer is one fused kernel over it.
"""
from __future__ import annotations

import torch

from . import lstm
from .embedding import Embedding
from .encoder import BLSTMEncoder
from .optim import Adam
from .output import OutputCE


class Seq2SeqLSTM:
    def __init__(self, enc_layers: int, batch: int, time: int, emb: int, hidden: int,
                 precision: str = "bf16", device=None, lr: float = 1e-3, clip_norm: float = 5.0,
                 vocab: int = 0, label_smoothing: float = 0.1, src_vocab: int = 0, trg_vocab: int = 0):
        """vocab > 0 adds the output softmax layer [hidden, vocab] and the CE loss
        (step() then takes target ids instead of an upstream gradient).
        src_vocab > 0: step() takes source token ids [B, T] (the `src` embedding
        layer) instead of source embeddings; trg_vocab > 0 (needs vocab): the
        decoder's target-embedding input comes from the `trg` layer's lookup of
        the previous target id instead of set_target_embeddings()."""
        self.L, self.B, self.T, self.E, self.H = enc_layers, batch, time, emb, hidden
        self.device = torch.device(device or "cuda")
        H = hidden
        self.Dd = emb + 2 * H  # decoder input [embedding ‖ context] (models.cpp:161: 620 + 2000)
        n_enc = BLSTMEncoder.numel(enc_layers, emb, H)
        n_dec = self.Dd * 4 * H + H * 4 * H + 4 * H
        self.V = vocab
        n_out = H * vocab + vocab if vocab else 0
        if trg_vocab and not vocab:
            raise ValueError("trg_vocab needs the output layer (vocab > 0): the previous target ids")
        self.Vs, self.Vt = src_vocab, trg_vocab
        n_src, n_trg = src_vocab * emb, trg_vocab * emb
        self.params = torch.empty(n_enc + n_dec + n_out + n_src + n_trg, dtype=torch.float32,
                                  device=self.device)
        self.grads = torch.zeros_like(self.params)
        bf16 = precision == "bf16"
        self.enc = BLSTMEncoder(enc_layers, batch, time, emb, H, precision, self.device,
                                params=self.params[:n_enc], grads=self.grads[:n_enc],
                                x0_bf16=bf16 and src_vocab > 0)
        off = n_enc
        self.dec_p, self.dec_g = [], []
        for shape in ((self.Dd, 4 * H), (H, 4 * H), (4 * H,)):
            k = 1
            for s in shape:
                k *= s
            self.dec_p.append(self.params[off:off + k].view(shape))
            self.dec_g.append(self.grads[off:off + k].view(shape))
            off += k
        self.dec_bucket = self.grads[n_enc:n_enc + n_dec]
        if vocab:  # output softmax layer (compiler.cpp:651-663): W [H, V], b [V]
            self.out_p = [self.params[off:off + H * vocab].view(H, vocab),
                          self.params[off + H * vocab:off + n_out]]
            self.out_g = [self.grads[off:off + H * vocab].view(H, vocab),
                          self.grads[off + H * vocab:off + n_out]]
            self.out_bucket = self.grads[off:off + n_out]
            self.out = OutputCE(batch, time, H, vocab, label_smoothing, device=self.device)
            self.dec_dy = torch.empty(batch, time, H, dtype=torch.float32, device=self.device)
        off = n_enc + n_dec + n_out
        if src_vocab:  # `src` layer: embedding table [Vs, E] (compiler.cpp:584-589)
            self.src_p = self.params[off:off + n_src].view(src_vocab, emb)
            self.src_g = self.grads[off:off + n_src].view(src_vocab, emb)
            self.src_bucket = self.grads[off:off + n_src]
            self.src_emb = Embedding(src_vocab, emb, batch * time, layer="src", device=self.device)
            self.x0 = (torch.zeros(batch, time, lstm.bf16_pitch(emb), dtype=torch.bfloat16, device=self.device)
                       if bf16 else torch.empty(batch, time, emb, dtype=torch.float32, device=self.device))
            off += n_src
        if trg_vocab:  # `trg` layer: embedding table [Vt, E] of the previous target
            self.trg_p = self.params[off:off + n_trg].view(trg_vocab, emb)
            self.trg_g = self.grads[off:off + n_trg].view(trg_vocab, emb)
            self.trg_bucket = self.grads[off:off + n_trg]
            self.trg_emb = Embedding(trg_vocab, emb, batch * time, layer="trg", device=self.device)
            self.prev_ids = torch.full((batch, time), -1, dtype=torch.int32, device=self.device)
        self.dec = lstm.LSTMLayer(batch, time, self.Dd, H, 1, 1, precision, self.device, x_bf16=bf16)
        if bf16:  # padded bf16 decoder input, ones column at Dd (seqloom_cuda.h SL_LAYER_X_BF16)
            self.dec_in = torch.zeros(batch, time, lstm.bf16_pitch(self.Dd), dtype=torch.bfloat16,
                                      device=self.device)
            self.dec_in[:, :, self.Dd] = 1.0
        else:
            self.dec_in = torch.zeros(batch, time, self.Dd, dtype=torch.float32, device=self.device)
        self.dec_y = torch.empty(batch, time, H, dtype=torch.float32, device=self.device)
        self.dec_dx = torch.empty(batch, time, self.Dd, dtype=torch.float32, device=self.device)
        self.enc_dy = torch.empty(batch, time, 2 * H, dtype=torch.float32, device=self.device)
        names = self.enc.param_slices() + [
            (f"dec/{n}", n_enc + o, k) for n, o, k in
            (("W", 0, self.Dd * 4 * H), ("R", self.Dd * 4 * H, H * 4 * H),
             ("b", self.Dd * 4 * H + H * 4 * H, 4 * H))]
        if vocab:
            names += [("output_prob/W", n_enc + n_dec, H * vocab), ("output_prob/b", n_enc + n_dec + H * vocab, vocab)]
        if src_vocab:
            names += [("src/W", n_enc + n_dec + n_out, n_src)]
        if trg_vocab:
            names += [("trg/W", n_enc + n_dec + n_out + n_src, n_trg)]
        self.opt = Adam(self.params, lr=lr, clip_norm=clip_norm, names=names)
        # checkpoint manifest (name, offset, shape) in the reference's layer/param naming
        shapes = {}
        for l, D in enumerate(self.enc.in_dims):
            for d in ("fw", "bw"):
                shapes.update({f"enc{l}_{d}/W": (D, 4 * H), f"enc{l}_{d}/R": (H, 4 * H), f"enc{l}_{d}/b": (4 * H,)})
        shapes.update({"dec/W": (self.Dd, 4 * H), "dec/R": (H, 4 * H), "dec/b": (4 * H,),
                       "output_prob/W": (H, vocab), "output_prob/b": (vocab,),
                       "src/W": (src_vocab, emb), "trg/W": (trg_vocab, emb)})
        self.manifest = [(n, o, shapes[n]) for n, o, _ in names]

    def save(self, directory: str, **state):
        """Checkpoint in the reference trainer's format (checkpoint.py)."""
        from . import checkpoint
        checkpoint.save(directory, self.params, self.manifest, optimizer=self.opt, **state)

    def load(self, directory: str):
        from . import checkpoint
        return checkpoint.load(directory, self.params, self.manifest, optimizer=self.opt)

    def init_uniform(self, seed: int = 0):
        g = torch.Generator(device=self.device).manual_seed(seed)
        s = 1.0 / self.H ** 0.5
        self.params.uniform_(-s, s, generator=g)

    def set_target_embeddings(self, emb: torch.Tensor):
        """emb [B, T, E]: the teacher-forced target-side embeddings."""
        self.dec_in[:, :, :self.E] = emb.to(self.dec_in.dtype)

    def set_targets(self, targets):
        """The `trg` layer input: previous target ids, -1 (a zero embedding) at t = 0."""
        self.prev_ids[:, 1:].copy_(targets[:, :-1])

    def forward(self, x, seq_lens, targets=None):
        """x: source embeddings [B, T, E] — or, with src_vocab, source ids [B, T]
        int32; targets (trg_vocab): the target ids whose predecessors feed the
        decoder."""
        if self.Vs:
            self.src_ids = x
            x = self.src_emb.forward(x, self.src_p, out=self.x0,
                                     bf16_pitch=self.x0.shape[-1] if self.x0.dtype == torch.bfloat16 else None)
        y = self.enc.forward(x, seq_lens)
        self.dec_in[:, :, self.E:self.Dd] = y.to(self.dec_in.dtype)  # context stand-in c_t = enc_t
        if self.Vt:
            self.set_targets(targets)
            self.trg_emb.forward(self.prev_ids, self.trg_p, out=self.dec_in[:, :, :self.E], negative_zero=True)
        W, R, b = self.dec_p
        self.dec.forward(self.dec_in, seq_lens, [W], [R], [b], y=self.dec_y)
        return self.dec_y

    def backward(self, dy_dec, on_grads=None):
        W, R, b = self.dec_g
        self.dec.backward(dy_dec, dx=self.dec_dx, dW=[W], dR=[R], db=[b])
        if on_grads is not None:
            on_grads(-1, self.dec_bucket)
        if self.Vt:
            self.trg_emb.backward(self.prev_ids, self.dec_dx[:, :, :self.E], self.trg_g)
            if on_grads is not None:
                on_grads(-3, self.trg_bucket)
        self.enc_dy.copy_(self.dec_dx[:, :, self.E:])
        dx = self.enc.backward(self.enc_dy, on_layer_grads=on_grads)
        if self.Vs:
            self.src_emb.backward(self.src_ids, dx, self.src_g)
            if on_grads is not None:
                on_grads(-4, self.src_bucket)
        return dx

    def check_ids(self):
        """Synchronise; raise the reference's IndexError for a bad source / target id."""
        if self.Vs:
            self.src_emb.check_ids()
        if self.Vt:
            self.trg_emb.check_ids()
        if self.V:
            self.out.check_targets()

    def loss_and_output_grads(self, targets, seq_lens, on_grads=None):
        """Output layer + label-smoothed CE on the decoder states: returns the
        (device) loss; dL/d(decoder output) lands in self.dec_dy."""
        W, b = self.out_p
        loss, _, _, _ = self.out.forward_backward(self.dec_y, targets, seq_lens, W, b, dx=self.dec_dy,
                                                  dW=self.out_g[0], db=self.out_g[1])
        if on_grads is not None:
            on_grads(-2, self.out_bucket)
        return loss

    def step(self, x, seq_lens, dy_or_targets, reducer=None, grad_scale: float = 1.0):
        """One training step.  With the output layer (vocab > 0) the last
        argument is the target ids [B, T] and the step returns the device loss;
        without it, the upstream gradient of the decoder output."""
        self.forward(x, seq_lens, dy_or_targets if self.Vt else None)
        loss = None
        if self.V:
            loss = self.loss_and_output_grads(dy_or_targets, seq_lens, on_grads=reducer)
            self.backward(self.dec_dy, on_grads=reducer)
        else:
            self.backward(dy_or_targets, on_grads=reducer)
        if reducer is not None:
            reducer.wait()
        self.opt.step(self.grads, grad_scale=grad_scale)
        return loss


class Seq2SeqAttention:
    """The full Listing-1 attention model's training step (BASELINE configs[3]:
    "6-layer BLSTM n=1000 encoder + 1-layer LSTM decoder with MLP attention, full
    training step with Adam"; make_attention_model, models.cpp:26-184):

      src (embedding of the source ids) -> enc0..enc{L-1} (BLSTM, lstm_sequence)
      -> encoder -> enc_ctx;  the `output` subnetwork (decoder.AttnDecoder: the
      RnnCell s with input feeding of the previous attention, the MLP attention,
      the readout) over the teacher-forced target;  output_prob (softmax +
      label-smoothed CE, output.OutputCE) on the readout;  then the fused
      global-norm clip + Adam step.

    Dropout 0.3 on the output_prob input (models.hpp:18) is the reference's own
    counter-based mask (dropout.py: bit-identical), its batch counter read from the
    optimizer's device-side step counter so a captured graph draws a new mask each
    step (dropout=0 turns it off).  The encoder's top
    layer writes the padded bf16 layout the decoder's GEMMs read directly.
    Parameters use the reference's qualified manifest names
    (compiler.cpp:470-500) and live in ONE flat fp32 buffer; the gradient
    buckets (output_prob, the decoder subnetwork, each encoder layer, src) are
    slices of it, reduced as soon as each is complete (dp.BucketAllReducer)."""

    def __init__(self, enc_layers: int, batch: int, src_time: int, trg_time: int, emb: int, hidden: int,
                 vocab: int, src_vocab: int, trg_vocab: int, key: int | None = None, readout: int | None = None,
                 device=None, lr: float = 1e-3, clip_norm: float = 5.0, label_smoothing: float = 0.1,
                 dropout: float = 0.3, seed: int = 1, precision: str = "bf16"):
        """precision "fp32": every layer at the reference's precision (rel. 1e-4;
        split-bf16 "x3" tensor-core GEMMs and recurrences, fp32 activations);
        "bf16": bf16 operands with fp32 accumulation and state (rel. 2e-2)."""
        from .decoder import NAMES, AttnDecoder, param_shapes
        if precision not in ("bf16", "fp32"):
            raise ValueError(f"precision must be bf16 or fp32, got {precision!r}")
        self.precision = precision
        bf16 = precision == "bf16"
        self.L, self.B, self.Ts, self.T, self.E, self.H = enc_layers, batch, src_time, trg_time, emb, hidden
        self.K, self.Rd = key or hidden, readout or hidden
        self.V, self.Vs, self.Vt = vocab, src_vocab, trg_vocab
        self.device = torch.device(device or "cuda")
        H, Ed = hidden, 2 * hidden
        n_enc = BLSTMEncoder.numel(enc_layers, emb, H)
        dshapes = param_shapes(emb, Ed, H, self.K, self.Rd, trg_vocab)
        # every parameter starts on a 128 B boundary (the kernels' vector accesses and the
        # GEMM epilogues' 16 B stores); the padding holds zeros and zero gradients
        al = lambda n: (n + 31) // 32 * 32
        layout, off = [], al(n_enc)
        for field, ref_name in NAMES:
            layout.append((field, ref_name, off, dshapes[field]))
            off = al(off + _numel(dshapes[field]))
        dec_end = off
        out_w, out_b = off, al(off + self.Rd * vocab)
        off = al(out_b + vocab)
        out_end = off
        src_off = off
        total = al(src_off + src_vocab * emb)
        self.params = torch.zeros(total, dtype=torch.float32, device=self.device)
        self.grads = torch.zeros_like(self.params)
        self.enc = BLSTMEncoder(enc_layers, batch, src_time, emb, H, precision, self.device,
                                params=self.params[:n_enc], grads=self.grads[:n_enc], x0_bf16=bf16, top_bf16=bf16)
        names = self.enc.param_slices()
        shapes = {}
        for l, D in enumerate(self.enc.in_dims):
            for d in ("fw", "bw"):
                shapes.update({f"enc{l}_{d}/W": (D, 4 * H), f"enc{l}_{d}/R": (H, 4 * H), f"enc{l}_{d}/b": (4 * H,)})
        self.dec_p, self.dec_g = {}, {}
        for field, ref_name, o, shp in layout:
            k = _numel(shp)
            self.dec_p[field] = self.params[o:o + k].view(shp)
            self.dec_g[field] = self.grads[o:o + k].view(shp)
            names.append((ref_name, o, k))
            shapes[ref_name] = shp
        self.dec_bucket = self.grads[al(n_enc):dec_end]
        self.out_p = [self.params[out_w:out_w + self.Rd * vocab].view(self.Rd, vocab),
                      self.params[out_b:out_b + vocab]]
        self.out_g = [self.grads[out_w:out_w + self.Rd * vocab].view(self.Rd, vocab),
                      self.grads[out_b:out_b + vocab]]
        self.out_bucket = self.grads[out_w:out_end]
        names += [("output/output_prob/W", out_w, self.Rd * vocab), ("output/output_prob/b", out_b, vocab)]
        shapes.update({"output/output_prob/W": (self.Rd, vocab), "output/output_prob/b": (vocab,)})
        n_src = src_vocab * emb
        self.src_p = self.params[src_off:src_off + n_src].view(src_vocab, emb)
        self.src_g = self.grads[src_off:src_off + n_src].view(src_vocab, emb)
        self.src_bucket = self.grads[src_off:src_off + n_src]
        names.append(("src/W", src_off, n_src))
        shapes["src/W"] = (src_vocab, emb)
        self.src_emb = Embedding(src_vocab, emb, batch * src_time, layer="src", device=self.device)
        self.x0 = (torch.zeros(batch, src_time, lstm.bf16_pitch(emb), dtype=torch.bfloat16, device=self.device)
                   if bf16 else torch.zeros(batch, src_time, emb, dtype=torch.float32, device=self.device))
        self.dec = AttnDecoder(batch, src_time, trg_time, emb, Ed, H, self.K, self.Rd, trg_vocab, self.device,
                               precision=precision)
        self.out = OutputCE(batch, trg_time, self.Rd, vocab, label_smoothing, device=self.device,
                            precision=precision)
        self.readout = torch.empty(batch, trg_time, self.Rd, dtype=torch.float32, device=self.device)
        self.d_readout = torch.empty_like(self.readout)
        self.dropout = None
        if dropout > 0:
            from .dropout import Dropout
            self.dropout = Dropout(dropout, seed, "output/output_prob", 0)
            self.dropped = torch.empty_like(self.readout)
            self.d_dropped = torch.empty_like(self.readout)
        self.d_enc = torch.empty(batch, src_time, Ed, dtype=torch.float32, device=self.device)
        self.prev_ids = torch.full((batch, trg_time), -1, dtype=torch.int32, device=self.device)
        self.opt = Adam(self.params, lr=lr, clip_norm=clip_norm, names=names)
        self.manifest = [(n, o, shapes[n]) for n, o, _ in names]

    def save(self, directory: str, **state):
        from . import checkpoint
        checkpoint.save(directory, self.params, self.manifest, optimizer=self.opt, **state)

    def load(self, directory: str):
        from . import checkpoint
        return checkpoint.load(directory, self.params, self.manifest, optimizer=self.opt)

    def init_uniform(self, seed: int = 0):
        """Every parameter ~ U(+-1/sqrt(H)); the alignment padding stays zero."""
        g = torch.Generator(device=self.device).manual_seed(seed)
        s = 1.0 / self.H ** 0.5
        self.params.uniform_(-s, s, generator=g)
        keep = torch.zeros_like(self.params, dtype=torch.bool)
        for _, o, k in self.opt.names:
            keep[o:o + k] = True
        self.params.masked_fill_(~keep, 0.0)

    def forward(self, src_ids, src_lens, targets):
        """src_ids [B, Ts], targets [B, T] int32 -> readout [B, T, Rd] (fp32)."""
        self.src_ids = src_ids
        self.src_emb.forward(src_ids, self.src_p, out=self.x0,
                             bf16_pitch=self.x0.shape[-1] if self.x0.dtype == torch.bfloat16 else None)
        self.enc_out = self.enc.forward(self.x0, src_lens)
        self.prev_ids[:, 1:].copy_(targets[:, :-1])  # prev:trg, the zero initial output at t = 0
        self.src_lens = src_lens
        return self.dec.forward(self.enc_out, src_lens, self.prev_ids, self.dec_p, readout=self.readout)

    def forward_backward(self, src_ids, src_lens, targets, trg_lens=None, reducer=None):
        """Loss and every parameter gradient of one batch (into self.grads), no
        optimizer update; returns the device loss (mean label-smoothed CE over the
        valid target positions, trg_lens defaulting to src_lens).  reducer(bucket id,
        bucket) fires as each gradient bucket completes (dp.BucketAllReducer)."""
        trg_lens = src_lens if trg_lens is None else trg_lens
        self.forward(src_ids, src_lens, targets)
        W, b = self.out_p
        if self.dropout is not None:  # batch counter = optimizer steps done (the device-side Adam counter)
            ctr = self.dropout_counter()
            self.dropout.forward(self.readout, self.dropped, counter=ctr)
            loss, _, _, _ = self.out.forward_backward(self.dropped, targets, trg_lens, W, b, dx=self.d_dropped,
                                                      dW=self.out_g[0], db=self.out_g[1])
            self.dropout.backward(self.d_dropped, self.d_readout, counter=ctr)
        else:
            loss, _, _, _ = self.out.forward_backward(self.readout, targets, trg_lens, W, b, dx=self.d_readout,
                                                      dW=self.out_g[0], db=self.out_g[1])
        if reducer is not None:
            reducer(-2, self.out_bucket)
        self.dec.backward(self.enc_out, src_lens, self.prev_ids, self.dec_p, self.readout, self.d_readout,
                          self.dec_g, d_enc=self.d_enc)
        if reducer is not None:
            reducer(-1, self.dec_bucket)
        dx = self.enc.backward(self.d_enc, on_layer_grads=reducer)
        self.src_emb.backward(self.src_ids, dx, self.src_g)
        if reducer is not None:
            reducer(-4, self.src_bucket)
        return loss

    def dropout_counter(self):
        """The dropout batch counter: the optimizer's device-side step counter."""
        return self.opt.scratch[12:16].view(torch.int32)

    def step(self, src_ids, src_lens, targets, trg_lens=None, reducer=None, grad_scale: float = 1.0):
        """One training step: forward_backward, the data-parallel gradient
        all-reduce (reducer), then the fused clip + Adam update; returns the device
        loss."""
        loss = self.forward_backward(src_ids, src_lens, targets, trg_lens, reducer)
        if reducer is not None:
            reducer.wait()
        self.opt.step(self.grads, grad_scale=grad_scale)
        return loss

    def named_params(self):
        """{manifest name: (param view, grad view)} of every parameter."""
        out = {}
        for name, off, shape in self.manifest:
            n = _numel(shape)
            out[name] = (self.params[off:off + n].view(shape), self.grads[off:off + n].view(shape))
        return out

    def check_ids(self):
        """Synchronise; raise the reference's IndexError for a bad source / target id."""
        self.src_emb.check_ids()
        self.dec.check_ids(self.prev_ids)
        self.out.check_targets()


def _numel(shape):
    k = 1
    for s in shape:
        k *= s
    return k


class GraphedStep:
    """A model's whole training step captured once as a CUDA graph and replayed —
    the user-facing call for repeated steps of one shape: every kernel of the
    step (embeddings, encoder, decoder, output layer, optimizer with its
    device-side step counter) replays without host launch gaps.  Each call
    copies the step's host inputs (pinned) into the captured device buffers,
    replays the graph and returns the loss read back to the host.

        step = GraphedStep(model, src_ids, src_lens, targets)   # device tensors of the shape
        loss = step(src_host, lens_host, trg_host)               # pinned host tensors

    Data-parallel: pass the step's `reducer` (dp.BucketAllReducer) and
    `grad_scale`; the bucketed NCCL all-reduces are captured with the kernels
    (every rank must build its GraphedStep at the same point)."""

    def __init__(self, model, src_ids, src_lens, targets, reducer=None, grad_scale: float = 1.0):
        self.model = model
        self.inputs = [src_ids.clone(), src_lens.clone(), targets.clone()]
        self.loss_h = torch.empty((), dtype=torch.float32).pin_memory()
        kw = dict(reducer=reducer, grad_scale=grad_scale) if reducer is not None or grad_scale != 1.0 else {}
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside the capture (lazy allocations, attributes)
            model.step(*self.inputs, **kw)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss = model.step(*self.inputs, **kw)

    def __call__(self, src_ids, src_lens, targets, sync: bool = True):
        for dst, src in zip(self.inputs, (src_ids, src_lens, targets)):
            dst.copy_(src, non_blocking=True)
        self.graph.replay()
        self.loss_h.copy_(self.loss, non_blocking=True)
        if not sync:
            return self.loss_h
        torch.cuda.current_stream().synchronize()
        return float(self.loss_h)
