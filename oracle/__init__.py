"""ORACLE — test infrastructure only.

Loaders for the two CPU checkers of the LSTM hot path:

* ``restatement()`` — ``_build/liblstm_oracle.so``: the plain-C fp64
  restatement in ``lstm_oracle.c`` (each function cites the reference
  file:line it follows).
* ``reference(bits)`` — ``_ref/libseqloom_ref{32,64}.so``: the REFERENCE's own
  ``tensor.cpp tape.cpp layers.cpp gradcheck.cpp`` compiled unmodified from
  /root/reference plus ``ref_bridge.cpp`` (built by ``make -C oracle``; the
  .so travels to the GPU box with the snapshot, /root/reference does not).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product (``paper_1805_05225_b200``) never does: it has no CPU path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_P = ctypes.POINTER
_d = _P(ctypes.c_double)
_i = _P(ctypes.c_int)


def build(force: bool = False) -> None:
    """Compile the restatement and, when /root/reference exists, the reference."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj"):
        targets += ["ref", "ref-tests", "dropin", "dropin-step"]
    subprocess.run(["make", "-C", HERE, "-j8"] + (["-B"] if force else []) + targets,
                   check=True, stdout=subprocess.DEVNULL)


def _ptr(a, typ=_d):
    return None if a is None else a.ctypes.data_as(typ)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class Restatement:
    """fp64 C restatement (oracle/lstm_oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_build", "liblstm_oracle.so")
        if not os.path.exists(path):
            build()
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.orc_lstm_sequence_fwd.argtypes = [ctypes.c_int] * 5 + [_d, _i, _d, _d, _d, _d, _d, _d]
        L.orc_lstm_sequence_bwd.argtypes = [ctypes.c_int] * 5 + [_d, _i, _d, _d, _d, _d, _d, _d,
                                                                 _d, _d, _d, _d]
        L.orc_lstm_step_fwd.argtypes = [ctypes.c_int] * 3 + [_d] * 9
        L.orc_lstm_step_bwd.argtypes = [ctypes.c_int] * 3 + [_d] * 14

    def sequence_fwd(self, x, lens, W, R, b, direction):
        B, T, D = x.shape
        H = R.shape[0]
        x, W, R, b = map(_f64, (x, W, R, b))
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        y = np.zeros((B, T, H))
        hl = np.zeros((B, H))
        cl = np.zeros((B, H))
        self.lib.orc_lstm_sequence_fwd(B, T, D, H, direction, _ptr(x), _ptr(lens, _i), _ptr(W),
                                       _ptr(R), _ptr(b), _ptr(y), _ptr(hl), _ptr(cl))
        return y, hl, cl

    def sequence_bwd(self, x, lens, W, R, b, direction, dy, dh_last=None, dc_last=None):
        B, T, D = x.shape
        H = R.shape[0]
        x, W, R, b, dy, dh_last, dc_last = map(_f64, (x, W, R, b, dy, dh_last, dc_last))
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        dx = np.zeros((B, T, D))
        dW = np.zeros((D, 4 * H))
        dR = np.zeros((H, 4 * H))
        db = np.zeros((4 * H,))
        self.lib.orc_lstm_sequence_bwd(B, T, D, H, direction, _ptr(x), _ptr(lens, _i), _ptr(W),
                                       _ptr(R), _ptr(b), _ptr(dy), _ptr(dh_last), _ptr(dc_last),
                                       _ptr(dx), _ptr(dW), _ptr(dR), _ptr(db))
        return dx, dW, dR, db

    def step_fwd(self, x, h0, c0, W, R, b):
        B, D = x.shape
        H = R.shape[0]
        x, h0, c0, W, R, b = map(_f64, (x, h0, c0, W, R, b))
        h = np.zeros((B, H))
        c = np.zeros((B, H))
        sv = np.zeros((B, 5 * H))
        self.lib.orc_lstm_step_fwd(B, D, H, _ptr(x), _ptr(h0), _ptr(c0), _ptr(W), _ptr(R),
                                   _ptr(b), _ptr(h), _ptr(c), _ptr(sv))
        return h, c, sv

    def step_bwd(self, x, h0, c0, W, R, b, gh=None, gc=None):
        B, D = x.shape
        H = R.shape[0]
        _, _, sv = self.step_fwd(x, h0, c0, W, R, b)
        x, h0, c0, W, R, gh, gc = map(_f64, (x, h0, c0, W, R, gh, gc))
        out = [np.zeros((B, D)), np.zeros((B, H)), np.zeros((B, H)), np.zeros((D, 4 * H)),
               np.zeros((H, 4 * H)), np.zeros((4 * H,))]
        self.lib.orc_lstm_step_bwd(B, D, H, _ptr(x), _ptr(h0), _ptr(c0), _ptr(W), _ptr(R),
                                   _ptr(sv), _ptr(gh), _ptr(gc), *[_ptr(o) for o in out])
        return tuple(out)  # dx, dh0, dc0, dW, dR, db


class Reference:
    """The reference implementation itself (oracle/_ref/libseqloom_ref{32,64}.so)."""

    def __init__(self, bits: int = 64, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", f"libseqloom_ref{bits}.so")
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} missing: build it with `make -C oracle ref` where /root/reference exists")
        self.lib = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
        L = self.lib
        c = ctypes.c_char_p
        L.ref_real_bytes.restype = ctypes.c_int
        L.ref_lstm_sequence.argtypes = [ctypes.c_int] * 5 + [_d, _i] + [_d] * 9 + [c, ctypes.c_int]
        L.ref_lstm_step.argtypes = [ctypes.c_int] * 3 + [_d] * 16 + [c, ctypes.c_int]
        L.ref_blstm_stack.argtypes = ([ctypes.c_int] * 5 + [_d, _i, _P(_d), _d, _d, _d, _P(_d)] +
                                      [c, ctypes.c_int])
        if hasattr(L, "ref_attention_step"):
            L.ref_attention_step.argtypes = ([ctypes.c_int] * 5 + [_i] + [_d] * 9 + [ctypes.c_double] +
                                             [_d] * 15 + [c, ctypes.c_int])
        if hasattr(L, "ref_gather_rows"):
            L.ref_gather_rows.argtypes = [ctypes.c_int] * 4 + [_d, _i, _d, _d, _d, c, ctypes.c_int]
        if hasattr(L, "ref_dropout"):
            L.ref_dropout.argtypes = ([ctypes.c_int] * 3 + [_d, ctypes.c_double, ctypes.c_ulonglong, c, ctypes.c_int,
                                                            ctypes.c_ulonglong, _d, _d, _d, c, ctypes.c_int])
        if hasattr(L, "ref_output_ce"):
            L.ref_output_ce.argtypes = ([ctypes.c_int] * 4 + [_d, _i, _i, _d, _d, ctypes.c_double] + [_d] * 4 +
                                        [c, ctypes.c_int])
        if hasattr(L, "ref_lstm_two_steps"):
            L.ref_lstm_two_steps.argtypes = [ctypes.c_int] * 3 + [_d] * 13 + [c, ctypes.c_int]
        if hasattr(L, "ref_param_manifest_order"):
            L.ref_param_manifest_order.argtypes = [c, c, ctypes.c_int, c, ctypes.c_int]
        self.bits = 8 * L.ref_real_bytes()

    def two_steps(self, x, h0, c0, W, R, b):
        """The graph of the reference's lstm_step FD test (tape_test.cpp:477-492):
        L = sum(step2.h) + sum(step1.h); returns (L, dx, dh0, dc0, dW, dR, db)."""
        x, h0, c0, W, R, b = map(_f64, (x, h0, c0, W, R, b))
        B, D = x.shape
        H = R.shape[0]
        out = [np.zeros_like(a) for a in (x, h0, c0, W, R, b)]
        loss = np.zeros(1)
        err = ctypes.create_string_buffer(512)
        self._check(self.lib.ref_lstm_two_steps(B, D, H, *(_ptr(a) for a in (x, h0, c0, W, R, b)), _ptr(loss),
                                                *(_ptr(a) for a in out), err, 512), err)
        return (float(loss[0]), *out)

    def param_manifest_order(self, names):
        """The reference ParamStore::manifest() order of these parameter names."""
        out = ctypes.create_string_buffer(sum(len(n) + 1 for n in names) + 16)
        err = ctypes.create_string_buffer(512)
        self._check(self.lib.ref_param_manifest_order("\n".join(names).encode(), out, len(out), err, 512), err)
        return [n for n in out.value.decode().split("\n") if n]

    @staticmethod
    def _check(rc, err):
        if rc != 0:
            raise RuntimeError(err.value.decode())

    def sequence(self, x, lens, W, R, b, direction, dy=None):
        """Returns y, and (dx, dW, dR, db) when dy is given (else None)."""
        B, T, D = x.shape
        H = R.shape[0]
        x, W, R, b, dy = map(_f64, (x, W, R, b, dy))
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        y = np.zeros((B, T, H))
        g = None
        if dy is not None:
            g = (np.zeros((B, T, D)), np.zeros((D, 4 * H)), np.zeros((H, 4 * H)), np.zeros(4 * H))
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_lstm_sequence(B, T, D, H, direction, _ptr(x), _ptr(lens, _i), _ptr(W),
                                        _ptr(R), _ptr(b), _ptr(dy), _ptr(y),
                                        *([_ptr(a) for a in g] if g else [None] * 4), err, 512)
        self._check(rc, err)
        return y, g

    def step(self, x, h0, c0, W, R, b, gh=None, gc=None):
        B, D = x.shape
        H = R.shape[0]
        x, h0, c0, W, R, b, gh, gc = map(_f64, (x, h0, c0, W, R, b, gh, gc))
        h = np.zeros((B, H))
        c = np.zeros((B, H))
        grad = gh is not None or gc is not None
        g = [np.zeros((B, D)), np.zeros((B, H)), np.zeros((B, H)), np.zeros((D, 4 * H)),
             np.zeros((H, 4 * H)), np.zeros(4 * H)] if grad else None
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_lstm_step(B, D, H, _ptr(x), _ptr(h0), _ptr(c0), _ptr(W), _ptr(R),
                                    _ptr(b), _ptr(gh), _ptr(gc), _ptr(h), _ptr(c),
                                    *([_ptr(a) for a in g] if g else [None] * 6), err, 512)
        self._check(rc, err)
        return h, c, (tuple(g) if g else None)

    def blstm_stack(self, x, lens, params, dy=None):
        """params: list over layers of (W_fw, R_fw, b_fw, W_bw, R_bw, b_bw)."""
        B, T, D0 = x.shape
        L = len(params)
        H = params[0][1].shape[0]
        flat = [_f64(p) for layer in params for p in layer]
        parr = (_d * len(flat))(*[_ptr(p) for p in flat])
        x, dy = _f64(x), _f64(dy)
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        y = np.zeros((B, T, 2 * H))
        dx = np.zeros_like(x) if dy is not None else None
        grads = [np.zeros_like(p) for p in flat] if dy is not None else None
        garr = (_d * len(flat))(*[_ptr(g) for g in grads]) if grads else None
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_blstm_stack(L, B, T, D0, H, _ptr(x), _ptr(lens, _i), parr, _ptr(dy),
                                      _ptr(y), _ptr(dx), garr, err, 512)
        self._check(rc, err)
        if grads is not None:
            grads = [tuple(grads[l * 6:(l + 1) * 6]) for l in range(L)]
        return y, dx, grads


def _output_ce(self, x, lens, targets, W, b, eps):
    """The reference's Softmax layer + ce_label_smoothing: (loss, dx, dW, db)."""
    B, T, D = x.shape
    V = W.shape[1]
    x, W, b = map(_f64, (x, W, b))
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    targets = np.ascontiguousarray(targets, dtype=np.int32)
    loss = np.zeros(1)
    dx, dW, db = np.zeros((B, T, D)), np.zeros((D, V)), np.zeros(V)
    err = ctypes.create_string_buffer(512)
    rc = self.lib.ref_output_ce(B, T, D, V, _ptr(x), _ptr(lens, _i), _ptr(targets, _i), _ptr(W), _ptr(b),
                                float(eps), _ptr(loss), _ptr(dx), _ptr(dW), _ptr(db), err, 512)
    self._check(rc, err)
    return float(loss[0]), dx, dW, db


Reference.output_ce = _output_ce


def _gather_rows(self, table, ids, d_out=None):
    """The reference's gather_rows over ids [B, T]: (out [B, T, D], d_table or None).
    An out-of-range id raises IndexError with the reference's message."""
    V, D = table.shape
    B, T = ids.shape
    table, d_out = _f64(table), _f64(d_out)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    out = np.zeros((B, T, D))
    dt = np.zeros((V, D)) if d_out is not None else None
    err = ctypes.create_string_buffer(512)
    rc = self.lib.ref_gather_rows(B, T, V, D, _ptr(table), _ptr(ids, _i), _ptr(d_out), _ptr(out), _ptr(dt),
                                  err, 512)
    if rc != 0 and "out of range" in err.value.decode():
        raise IndexError(err.value.decode())
    self._check(rc, err)
    return out, dt


Reference.gather_rows = _gather_rows


def gather_rows_np(table, ids, d_out=None, layer="emb"):
    """Restatement of Tape::gather_rows (tape.cpp:448-492) in the table's dtype:
    out[r] = table[ids[r]]; the adjoint adds the d_out rows into a zero table
    gradient one row at a time in ascending r (tape.cpp:478-486) — the exact
    float summation order of the reference's fp32 build."""
    table = np.asarray(table)
    V, D = table.shape
    flat = np.asarray(ids, dtype=np.int64).reshape(-1)
    for v in flat:
        if v < 0 or v >= V:
            raise IndexError(f"id {int(v)} out of range [0, {V}) in layer '{layer}'")
    out = table[flat].reshape(tuple(np.shape(ids)) + (D,))
    if d_out is None:
        return out, None
    g = np.asarray(d_out, dtype=table.dtype).reshape(-1, D)
    dt = np.zeros((V, D), dtype=table.dtype)
    for r, v in enumerate(flat):
        dt[v] += g[r]
    return out, dt


def _attention_step(self, lens, enc_ctx, enc, s, accum, Ws, bs, Wfb, bfb, v, bv, d_att=None, d_accum=None):
    """The reference's attention subnet step: (att, a, accum', grads dict or None)."""
    B, Ts, K = enc_ctx.shape
    E = enc.shape[2]
    H = s.shape[1]
    ins = [_f64(a) for a in (enc_ctx, enc, s, accum, Ws, bs, Wfb, bfb, v)]
    d_att, d_accum = _f64(d_att), _f64(d_accum)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    att, a, acc2 = np.zeros((B, E)), np.zeros((B, Ts)), np.zeros((B, Ts))
    names = ["enc_ctx", "enc", "s", "accum", "Ws", "bs", "Wfb", "bfb", "v", "bv"]
    shapes = [(B, Ts, K), (B, Ts, E), (B, H), (B, Ts), (H, K), (K,), (1, K), (K,), (K, 1), (1,)]
    g = [np.zeros(sh) for sh in shapes] if d_att is not None else None
    err = ctypes.create_string_buffer(512)
    rc = self.lib.ref_attention_step(B, Ts, K, E, H, _ptr(lens, _i), *[_ptr(x) for x in ins], float(bv),
                                     _ptr(d_att), _ptr(d_accum), _ptr(att), _ptr(a), _ptr(acc2),
                                     *([_ptr(x) for x in g] if g else [None] * 10), err, 512)
    self._check(rc, err)
    return att, a, acc2, (dict(zip(names, g)) if g else None)


Reference.attention_step = _attention_step


def attention_step_np(lens, enc_ctx, enc, s, accum, Ws, bs, Wfb, bfb, v, bv, d_att=None, d_accum=None):
    """fp64 numpy restatement of the same step (models.cpp:107-154 wiring; ops
    tape.cpp:327-356 matmul, 134-174 broadcast add, 926-985 softmax_over_spatial,
    987-1072 generic_attention).  Returns (att, a, accum', grads or None)."""
    enc_ctx, enc, s, accum, Ws, bs, Wfb, bfb, v = (np.asarray(x, np.float64) for x in
                                                   (enc_ctx, enc, s, accum, Ws, bs, Wfb, bfb, v))
    B, Ts, K = enc_ctx.shape
    valid = np.arange(Ts)[None, :] < np.asarray(lens)[:, None]           # [B, Ts]
    s_tr = s @ Ws + bs                                                   # [B, K]
    e_in = enc_ctx + accum[:, :, None] * Wfb[0][None, None, :] + bfb + s_tr[:, None, :]
    u = np.tanh(e_in)
    e = u @ v[:, 0] + bv                                                 # [B, Ts]
    em = np.where(valid, e, -np.inf)
    m = em.max(axis=1, keepdims=True)
    ex = np.where(valid, np.exp(em - m), 0.0)
    a = ex / ex.sum(axis=1, keepdims=True)                               # tape.cpp:952-960
    acc2 = accum + a
    att = np.einsum("bj,bje->be", a, enc)                                # tape.cpp:1005-1014
    if d_att is None:
        return att, a, acc2, None
    d_att = np.asarray(d_att, np.float64)
    # the upstream gradient of accum' is masked at padded source positions like
    # every time-masked tape value (the reference's mul / reduce_sum respect seq_lens)
    d_acc2 = np.zeros((B, Ts)) if d_accum is None else np.where(valid, np.asarray(d_accum, np.float64), 0.0)
    d_a = np.einsum("be,bje->bj", d_att, enc) + d_acc2                   # tape.cpp:1031-1041
    g_enc = a[:, :, None] * d_att[:, None, :]                            # tape.cpp:1047-1058
    dot = (d_a * a).sum(axis=1, keepdims=True)
    d_e = np.where(valid, a * (d_a - dot), 0.0)                          # tape.cpp:966-978
    d_u = d_e[:, :, None] * v[:, 0][None, None, :]
    d_ein = d_u * (1 - u * u)
    g = {"enc_ctx": d_ein, "enc": g_enc, "s": d_ein.sum(axis=1) @ Ws.T, "accum": d_acc2 + d_ein @ Wfb[0],
         "Ws": s.T @ d_ein.sum(axis=1), "bs": d_ein.sum(axis=(0, 1)),
         "Wfb": (accum[:, :, None] * d_ein).sum(axis=(0, 1))[None, :], "bfb": d_ein.sum(axis=(0, 1)),
         "v": np.einsum("bjk,bj->k", u, d_e)[:, None], "bv": np.array([d_e.sum()])}
    return att, a, acc2, g


def output_ce_np(x, lens, targets, W, b, eps):
    """fp64 numpy restatement of the same (compiler.cpp:651-663, tape.cpp:879-924,
    1224-1298): loss = mean over valid rows of lse - (1-eps) z_y - eps/V sum_j z_j."""
    x, W, b = (np.asarray(a, np.float64) for a in (x, W, b))
    B, T, D = x.shape
    V = W.shape[1]
    z = x.reshape(B * T, D) @ W + b                     # matmul + add (tape.cpp:327-356)
    m = z.max(axis=1, keepdims=True)
    lse = m + np.log(np.exp(z - m).sum(axis=1, keepdims=True))
    lp = z - lse                                        # log_softmax (tape.cpp:889-897)
    valid = (np.arange(T)[None, :] < np.asarray(lens)[:, None]).reshape(-1)
    y = np.asarray(targets).reshape(-1)
    n = int(valid.sum())
    rows = np.nonzero(valid)[0]
    loss = (-(1 - eps) * lp[rows, y[rows]] - eps / V * lp[rows].sum(axis=1)).sum() / n  # tape.cpp:1270-1278
    g = np.zeros_like(z)                                # adjoints (tape.cpp:1285-1293, 907-917)
    g[rows] = np.exp(lp[rows]) - eps / V
    g[rows, y[rows]] -= 1 - eps
    g /= n
    return loss, (g @ W.T).reshape(B, T, D), x.reshape(B * T, D).T @ g, g.sum(axis=0)


def seeded_case(seed: int, B: int, T: int, D: int, H: int, ragged: bool = True,
                wscale: float | None = None):
    """Synthetic inputs as SURVEY §8(d): x ~ U(-1,1); W, R, b ~ U(+-1/sqrt(H));
    ragged lens ~ U[ceil(T/2), T] with at least one full-length row."""
    rng = np.random.default_rng(seed)
    s = wscale if wscale is not None else 1.0 / np.sqrt(H)
    x = rng.uniform(-1, 1, (B, T, D))
    W = rng.uniform(-s, s, (D, 4 * H))
    R = rng.uniform(-s, s, (H, 4 * H))
    b = rng.uniform(-s, s, (4 * H,))
    if ragged:
        lens = rng.integers((T + 1) // 2, T + 1, size=B).astype(np.int32)
        lens[0] = T
    else:
        lens = np.full(B, T, dtype=np.int32)
    return x, lens, W, R, b


def lstm_step_np(x, h, c, W, R, b, gh=None, gc=None):
    """fp64 numpy restatement of Tape::lstm_step (tape.cpp:1095-1135) and its
    backward closure (tape.cpp:1157-1215).  Forward: (h', c').  With gh:
    (dx, dh, dc, dW, dR, db) for upstream gh, gc (gc None = 0)."""
    x, h, c, W, R, b = (np.asarray(a, np.float64) for a in (x, h, c, W, R, b))
    H = h.shape[1]
    z = x @ W + h @ R + b
    sig = lambda v: 1.0 / (1.0 + np.exp(-v))
    i, f, g, o = sig(z[:, :H]), sig(z[:, H:2 * H]), np.tanh(z[:, 2 * H:3 * H]), sig(z[:, 3 * H:])
    c2 = f * c + i * g
    tc = np.tanh(c2)
    if gh is None:
        return o * tc, c2
    gh = np.asarray(gh, np.float64)
    gc = np.zeros_like(gh) if gc is None else np.asarray(gc, np.float64)
    d_o = gh * tc
    dc = gc + gh * o * (1 - tc * tc)
    dz = np.concatenate([dc * g * i * (1 - i), dc * c * f * (1 - f), dc * i * (1 - g * g), d_o * o * (1 - o)], axis=1)
    return dz @ W.T, dz @ R.T, dc * f, x.T @ dz, h.T @ dz, dz.sum(axis=0)


def attn_decoder_np(src_lens, enc, prev_ids, P, d_readout=None, relu_mask=None):
    """fp64 restatement of the Listing-1 `output` subnetwork over a teacher-forced
    target sequence as the reference's training loop evaluates it (models.cpp:
    83-166, compiler.cpp:770-905: one step per target position, loop-carried
    prev: values starting at zero, compiler.cpp:674-697) plus the base layer
    enc_ctx (models.cpp:60).  It chains the two pinned per-step restatements —
    lstm_step_np (the RnnCell `s`) and attention_step_np — and a relu Linear
    readout.  P: dict with the decoder.NAMES keys (reference shapes).
    Returns readout [B, T, Rd]; with d_readout also the gradients (dict, same
    keys) and d_enc, by the reverse replay of those steps (tape.cpp:1363-1381).
    relu_mask (optional, [B, T, Rd] bool): the readout's relu derivative to use
    instead of pre > 0 — a lower-precision run may round a pre-activation within
    its error of 0 to the other side; comparing gradients needs the same mask."""
    enc = np.asarray(enc, np.float64)
    P = {k: np.asarray(v, np.float64) for k, v in P.items()}
    B, Ts, E = enc.shape
    T = prev_ids.shape[1]
    H = P["s_R"].shape[0]
    Emb = P["trg_W"].shape[1]
    ids = np.asarray(prev_ids)
    trg = np.where(ids[..., None] >= 0, P["trg_W"][np.maximum(ids, 0)], 0.0)       # [B, T, Emb]
    enc_ctx = enc @ P["enc_ctx_W"] + P["enc_ctx_b"]
    s, c, att, acc = np.zeros((B, H)), np.zeros((B, H)), np.zeros((B, E)), np.zeros((B, Ts))
    att_args = lambda: (P["s_tr_W"], P["s_tr_b"], P["fb_W"], P["fb_b"], P["e_W"], P["e_b"][0])
    saves, S, ATT = [], np.zeros((B, T, H)), np.zeros((B, T, E))
    for t in range(T):
        x = np.concatenate([trg[:, t], att], axis=1)
        s2, c2 = lstm_step_np(x, s, c, P["s_W"], P["s_R"], P["s_b"])
        att2, _, acc2, _ = attention_step_np(src_lens, enc_ctx, enc, s2, acc, *att_args())
        saves.append((x, s, c, s2, acc))
        S[:, t], ATT[:, t] = s2, att2
        s, c, att, acc = s2, c2, att2, acc2
    RO = np.concatenate([S, trg, ATT], axis=2)
    pre = RO @ P["readout_W"] + P["readout_b"]
    readout = np.maximum(pre, 0.0)
    if d_readout is None:
        return readout
    attn_decoder_np.pre = pre
    dpre = np.asarray(d_readout, np.float64) * (pre > 0 if relu_mask is None else np.asarray(relu_mask))
    g = {k: np.zeros_like(v) for k, v in P.items()}
    g["readout_W"] = RO.reshape(B * T, -1).T @ dpre.reshape(B * T, -1)
    g["readout_b"] = dpre.sum(axis=(0, 1))
    dRO = dpre @ P["readout_W"].T
    dS, dTRG, dATT = dRO[:, :, :H], dRO[:, :, H:H + Emb].copy(), dRO[:, :, H + Emb:]
    d_enc, d_ctx = np.zeros_like(enc), np.zeros_like(enc_ctx)
    dh, dc, datt, dacc = np.zeros((B, H)), np.zeros((B, H)), np.zeros((B, E)), np.zeros((B, Ts))
    for t in reversed(range(T)):
        x, s_prev, c_prev, s_t, acc_prev = saves[t]
        _, _, _, ga = attention_step_np(src_lens, enc_ctx, enc, s_t, acc_prev, *att_args(),
                                        d_att=dATT[:, t] + datt, d_accum=dacc)
        d_ctx += ga["enc_ctx"]
        d_enc += ga["enc"]
        for mine, theirs in (("s_tr_W", "Ws"), ("s_tr_b", "bs"), ("fb_W", "Wfb"), ("fb_b", "bfb"), ("e_W", "v"),
                             ("e_b", "bv")):
            g[mine] += ga[theirs]
        dacc = ga["accum"]
        dx, dh, dc, dW, dR, db = lstm_step_np(x, s_prev, c_prev, P["s_W"], P["s_R"], P["s_b"],
                                              gh=dS[:, t] + dh + ga["s"], gc=dc)
        g["s_W"] += dW
        g["s_R"] += dR
        g["s_b"] += db
        dTRG[:, t] += dx[:, :Emb]
        datt = dx[:, Emb:]
    d_enc += d_ctx @ P["enc_ctx_W"].T
    g["enc_ctx_W"] = enc.reshape(B * Ts, E).T @ d_ctx.reshape(B * Ts, -1)
    g["enc_ctx_b"] = d_ctx.sum(axis=(0, 1))
    flat, rows = ids.reshape(-1), dTRG.reshape(B * T, Emb)
    for r in np.argsort(flat, kind="stable"):     # gather_rows adjoint (tape.cpp:476-488)
        if flat[r] >= 0:
            g["trg_W"][flat[r]] += rows[r]
    return readout, g, d_enc



def _dropout(self, x, rate, seed, qualified, input_index, batch_counter, d_out=None):
    """The reference's input dropout on a [B, T, F] value (Tape::dropout): (out, dx or None)."""
    B, T, F = x.shape
    x, d_out = _f64(x), _f64(d_out)
    out = np.zeros((B, T, F))
    dx = np.zeros((B, T, F)) if d_out is not None else None
    err = ctypes.create_string_buffer(512)
    rc = self.lib.ref_dropout(B, T, F, _ptr(x), float(rate), int(seed), qualified.encode(), int(input_index),
                              int(batch_counter), _ptr(d_out), _ptr(out), _ptr(dx), err, 512)
    self._check(rc, err)
    return out, dx


Reference.dropout = _dropout

_M64 = (1 << 64) - 1


def splitmix64(x):
    """rng.hpp splitmix64 on Python ints (uint64 arithmetic)."""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def mix64(a, b):
    return splitmix64(a ^ ((splitmix64(b) + 0x9E3779B97F4A7C15) & _M64))


def fnv1a(s: str):
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h = ((h ^ ch) * 0x100000001B3) & _M64
    return h


def _splitmix64_np(x):
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def dropout_key(seed: int, qualified: str, input_index: int, batch_counter: int) -> int:
    """compiler.cpp:559-560: mix64(mix64(seed, fnv1a(qualified#index)), batch_counter)."""
    return mix64(mix64(seed, fnv1a(f"{qualified}#{input_index}")), batch_counter)


def dropout_mask_np(key: int, B: int, T: int, F: int, rate: float):
    """Keep mask of Tape::dropout for a [B, T, F] value keyed by its own Time
    coordinate (tape.cpp:549-570, 67-71): survives(key, t + 2, b*F + f) =
    u01(mix64(key, mix64(t + 2, pos))) >= rate, u01(h) = (splitmix64(h) >> 11) * 2^-53."""
    with np.errstate(over="ignore"):
        t = np.arange(T, dtype=np.uint64)[None, :, None] + np.uint64(2)
        pos = (np.arange(B, dtype=np.uint64)[:, None, None] * np.uint64(F) +
               np.arange(F, dtype=np.uint64)[None, None, :])
        inner = _splitmix64_np(pos) + np.uint64(0x9E3779B97F4A7C15)   # mix64(t + 2, pos)
        m1 = _splitmix64_np(t ^ inner)
        outer = _splitmix64_np(m1) + np.uint64(0x9E3779B97F4A7C15)     # mix64(key, m1)
        h = _splitmix64_np(np.uint64(key) ^ outer)
        u = (_splitmix64_np(h) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return u >= rate


def dropout_np(x, key, rate, d_out=None, real=np.float32):
    """out = x * keep / (1 - rate) with the reference's inv_keep = Real(1) / (Real(1) - rate)."""
    B, T, F = x.shape
    keep = dropout_mask_np(key, B, T, F, rate)
    inv = real(1) / (real(1) - real(rate))
    out = np.where(keep, np.asarray(x, real) * inv, real(0))
    if d_out is None:
        return out
    return out, np.where(keep, np.asarray(d_out, real) * inv, real(0))
