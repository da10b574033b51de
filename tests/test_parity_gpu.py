"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

Tolerances (norm-wise max|gpu-ref| / max|ref| per tensor):
  SL_PREC_FP32 : 1e-4   (north_star: "relative 1e-4 for the FP32/TF32 path")
  SL_PREC_BF16 : 2e-2   (north_star: "a separately stated looser bound for BF16")
References: the golden fixtures produced by the reference build
(tests/golden/, make_golden.py) at small sizes; the fp64 torch restatement
(oracle/torch_ref.py, pinned to the C restatement by tests/test_oracle.py) at
BASELINE sizes; plus size-independent properties.
"""
import os

import numpy as np
import pytest
import torch

from oracle import torch_ref
import oracle
from paper_1805_05225_b200 import lstm

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"fp32": 1e-4, "bf16": 2e-2}
PRECS = ["fp32", "bf16"]


def rel(a, b):
    a = torch.as_tensor(a).double().cpu()
    b = torch.as_tensor(b).double().cpu()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def cu(a, dtype=torch.float32):
    return torch.as_tensor(np.asarray(a)).to("cuda", dtype).contiguous()


def run_layer(x, lens, params, nd, direction, prec, dy, dh=None, dc=None, accumulate_twice=False):
    B, T, D = x.shape
    H = params[0][1].shape[0]
    layer = lstm.LSTMLayer(B, T, D, H, nd, direction, prec)
    W = [p[0] for p in params]
    R = [p[1] for p in params]
    b = [p[2] for p in params]
    y, hl, cl = layer.forward(x, lens, W, R, b)
    dx, dW, dR, db = layer.backward(dy, dh, dc)
    if accumulate_twice:
        layer.backward(dy, dh, dc, dx=dx, dW=dW, dR=dR, db=db, accumulate=True)
    torch.cuda.synchronize()
    return dict(y=y, h_last=hl, c_last=cl, dx=dx, dW=dW, dR=dR, db=db)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", ["config1_fw", "config1_bw", "t1_bw", "lens35_fw", "odd_bw"])
def test_golden_sequence(cuda, name, prec):
    f = np.load(os.path.join(GOLD, name + ".npz"))
    d = int(f["direction"])
    out = run_layer(cu(f["x"]), cu(f["lens"], torch.int32), [(cu(f["W"]), cu(f["R"]), cu(f["b"]))],
                    1, d, prec, cu(f["dy"]))
    tol = TOL[prec]
    assert rel(out["y"], f["y_ref64"]) < tol
    assert rel(out["dx"], f["dx_ref64"]) < tol
    assert rel(out["dW"][0], f["dW_ref64"]) < tol
    assert rel(out["dR"][0], f["dR_ref64"]) < tol
    assert rel(out["db"][0], f["db_ref64"]) < tol
    # padded outputs are exactly zero (tape.cpp:797-798)
    lens = f["lens"]
    y = out["y"].cpu().numpy()
    for r, L in enumerate(lens):
        assert np.all(y[r, L:] == 0.0)


@pytest.mark.parametrize("prec", PRECS)
def test_golden_bidirectional_stack(cuda, prec):
    f = np.load(os.path.join(GOLD, "blstm2.npz"))
    L = int(f["L"])
    lens = cu(f["lens"], torch.int32)
    x = cu(f["x"])
    layers, inputs = [], [x]
    for l in range(L):
        B, T, D = inputs[-1].shape
        H = f[f"R_fw_{l}"].shape[0]
        layer = lstm.LSTMLayer(B, T, D, H, 2, 1, prec)
        P = [[cu(f[f"{n}_{k}_{l}"]) for k in ("fw", "bw")] for n in ("W", "R", "b")]
        y, _, _ = layer.forward(inputs[-1], lens, *P)
        layers.append((layer, P))
        inputs.append(y)
    assert rel(inputs[-1], f["y_ref64"]) < TOL[prec]
    g = cu(f["dy"])
    for l in reversed(range(L)):
        layer, P = layers[l]
        dx, dW, dR, db = layer.backward(g)
        for k, n in enumerate(("fw", "bw")):
            assert rel(dW[k], f[f"dW_{n}_{l}_ref64"]) < TOL[prec]
            assert rel(dR[k], f[f"dR_{n}_{l}_ref64"]) < TOL[prec]
            assert rel(db[k], f[f"db_{n}_{l}_ref64"]) < TOL[prec]
        g = dx
    assert rel(g, f["dx_ref64"]) < TOL[prec]


def _seeded(seed, B, T, D, H, ragged=True):
    x, lens, W, R, b = oracle.seeded_case(seed, B, T, D, H, ragged=ragged)
    return cu(x), cu(lens, torch.int32), cu(W), cu(R), cu(b)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("direction", [1, -1])
def test_config2_full_size_vs_fp64(cuda, prec, direction):
    # BASELINE configs[1]: H = D = 1024, B = 128, T = 60 (ragged lengths)
    x, lens, W, R, b = _seeded(100 + direction, 128, 60, 1024, 1024)
    g = torch.Generator(device="cuda").manual_seed(3)
    dy = torch.rand(128, 60, 1024, device="cuda", generator=g) * 2 - 1
    dh = torch.rand(1, 128, 1024, device="cuda", generator=g) * 2 - 1
    dc = torch.rand(1, 128, 1024, device="cuda", generator=g) * 2 - 1
    out = run_layer(x, lens, [(W, R, b)], 1, direction, prec, dy, dh, dc)
    ref = torch_ref.sequence(x, lens, W, R, b, direction, dy, dh[0], dc[0])
    tol = TOL[prec]
    assert rel(out["y"], ref["y"]) < tol
    assert rel(out["h_last"][0], ref["h_last"]) < tol
    assert rel(out["c_last"][0], ref["c_last"]) < tol
    assert rel(out["dx"], ref["dx"]) < tol
    assert rel(out["dW"][0], ref["dW"]) < tol
    assert rel(out["dR"][0], ref["dR"]) < tol
    assert rel(out["db"][0], ref["db"]) < tol


@pytest.mark.parametrize("prec", PRECS)
def test_config3_layer_bidirectional_vs_fp64(cuda, prec):
    # BASELINE configs[2] layer shapes: H = 1000, D0 = 620, both directions concurrent
    B, T, D, H = 64, 60, 620, 1000
    x, lens, _, _, _ = _seeded(7, B, T, D, H)
    params = [_seeded(8 + k, 1, 1, D, H)[2:] for k in range(2)]
    dy = torch.rand(B, T, 2 * H, device="cuda") * 2 - 1
    out = run_layer(x, lens, params, 2, 1, prec, dy)
    dx = 0
    for k, d in enumerate((1, -1)):
        W, R, b = params[k]
        ref = torch_ref.sequence(x, lens, W, R, b, d, dy[:, :, k * H:(k + 1) * H])
        assert rel(out["y"][:, :, k * H:(k + 1) * H], ref["y"]) < TOL[prec]
        assert rel(out["dW"][k], ref["dW"]) < TOL[prec]
        assert rel(out["dR"][k], ref["dR"]) < TOL[prec]
        assert rel(out["db"][k], ref["db"]) < TOL[prec]
        dx = dx + ref["dx"]
    assert rel(out["dx"], dx) < TOL[prec]


@pytest.mark.parametrize("prec", PRECS)
def test_masked_inputs_cannot_leak(cuda, prec):
    # tape_test.cpp:535-566 / SPEC.md:106: perturbing padded positions changes
    # neither valid outputs nor gradients (bitwise)
    x, lens, W, R, b = _seeded(9, 16, 24, 40, 48)
    dy = torch.rand(16, 24, 2 * 48, device="cuda")
    a = run_layer(x, lens, [(W, R, b)] * 2, 2, 1, prec, dy)
    x2 = x.clone()
    for r, L in enumerate(lens.tolist()):
        x2[r, L:] = 123.5
    dy2 = dy.clone()
    for r, L in enumerate(lens.tolist()):
        dy2[r, L:] = -7.0
    c = run_layer(x2, lens, [(W, R, b)] * 2, 2, 1, prec, dy2)
    assert torch.equal(a["y"], c["y"])
    for k in ("dW", "dR", "db"):
        for u, v in zip(a[k], c[k]):
            assert torch.equal(u, v), k
    valid = (torch.arange(24, device="cuda")[None] < lens[:, None])[..., None]
    assert torch.equal(a["dx"] * valid, c["dx"] * valid)
    assert torch.all(c["dx"][~valid.expand_as(c["dx"])] == 0)


@pytest.mark.parametrize("prec", PRECS)
def test_deterministic_bitwise(cuda, prec):
    # tape_test.cpp:513-533: repeated runs are bitwise identical
    x, lens, W, R, b = _seeded(10, 32, 20, 64, 96)
    dy = torch.rand(32, 20, 96, device="cuda")
    a = run_layer(x, lens, [(W, R, b)], 1, -1, prec, dy)
    c = run_layer(x, lens, [(W, R, b)], 1, -1, prec, dy)
    for k in ("y", "dx", "h_last", "c_last"):
        assert torch.equal(a[k], c[k]), k
    for k in ("dW", "dR", "db"):
        assert torch.equal(a[k][0], c[k][0]), k


@pytest.mark.parametrize("prec", PRECS)
def test_time1_both_directions_equal(cuda, prec):
    # SPEC.md:316
    x, lens, W, R, b = _seeded(11, 8, 1, 16, 32, ragged=False)
    dy = torch.rand(8, 1, 32, device="cuda")
    a = run_layer(x, lens, [(W, R, b)], 1, 1, prec, dy)
    c = run_layer(x, lens, [(W, R, b)], 1, -1, prec, dy)
    assert torch.equal(a["y"], c["y"])


@pytest.mark.parametrize("prec", PRECS)
def test_backward_direction_is_rev_forward_rev(cuda, prec):
    # dir -1 == reverse_per_seq . dir +1 . reverse_per_seq
    x, lens, W, R, b = _seeded(12, 24, 33, 48, 64)
    def rev(t):
        out = t.clone()
        for r, L in enumerate(lens.tolist()):
            out[r, :L] = t[r, :L].flip(0)
        return out
    dy = torch.rand(24, 33, 64, device="cuda")
    a = run_layer(x, lens, [(W, R, b)], 1, -1, prec, dy)
    c = run_layer(rev(x), lens, [(W, R, b)], 1, 1, prec, rev(dy))
    assert rel(a["y"], rev(c["y"])) < 1e-6
    assert rel(a["dW"][0], c["dW"][0]) < 1e-5
    assert rel(a["dx"], rev(c["dx"])) < 1e-5


@pytest.mark.parametrize("prec", PRECS)
def test_accumulate_contract(cuda, prec):
    # GradBuffer::accumulate (tape.cpp:76-89): accumulate=1 adds into existing grads
    x, lens, W, R, b = _seeded(13, 8, 10, 12, 16)
    dy = torch.rand(8, 10, 16, device="cuda")
    once = run_layer(x, lens, [(W, R, b)], 1, 1, prec, dy)
    twice = run_layer(x, lens, [(W, R, b)], 1, 1, prec, dy, accumulate_twice=True)
    assert rel(twice["dx"], 2 * once["dx"]) < 1e-6
    for k in ("dW", "dR", "db"):
        assert rel(twice[k][0], 2 * once[k][0]) < 1e-6


@pytest.mark.parametrize("prec", PRECS)
def test_lstm_step_golden(cuda, prec):
    f = np.load(os.path.join(GOLD, "lstm_step.npz"))
    z = lambda *s: torch.zeros(*s, device="cuda")
    h, c, _ = lstm.lstm_step(z(1, 2), z(1, 3), torch.full((1, 3), 2.0, device="cuda"), z(2, 12),
                             z(3, 12), z(12), prec)
    assert rel(c, f["hand_c2_c"]) < 1e-6 and rel(h, f["hand_c2_h"]) < 1e-6
    args = [cu(f["rand_" + k]) for k in ("x", "h0", "c0", "W", "R", "b")]
    h, c, saved = lstm.lstm_step(*args, precision=prec)
    assert rel(h, f["rand_h"]) < TOL[prec] and rel(c, f["rand_c"]) < TOL[prec]
    g = lstm.lstm_step_backward(*args[:5], saved, cu(f["rand_gh"]), cu(f["rand_gc"]), prec)
    for k, v in zip(("dx", "dh0", "dc0", "dW", "dR", "db"), g):
        assert rel(v, f["rand_" + k]) < TOL[prec], k


def test_lstm_sequence_functional_matches_layer(cuda):
    x, lens, W, R, b = _seeded(14, 4, 6, 5, 7)
    y = lstm.lstm_sequence(x, lens, W, R, b, -1)
    ref = torch_ref.sequence(x, lens, W, R, b, -1)
    assert rel(y, ref["y"]) < 1e-4


@pytest.mark.parametrize("prec", PRECS)
def test_batch_chunks_beyond_256(cuda, prec):
    # B > 256: the tensor-core recurrences run as several 256-row batch launches
    B, T, D, H = 300, 12, 24, 40
    x, lens, W, R, b = _seeded(21, B, T, D, H)
    dy = torch.rand(B, T, 2 * H, device="cuda") * 2 - 1
    params = [(W, R, b), _seeded(22, 1, 1, D, H)[2:]]
    out = run_layer(x, lens, params, 2, 1, prec, dy)
    dx = 0
    for k, d in enumerate((1, -1)):
        Wk, Rk, bk = params[k]
        ref = torch_ref.sequence(x, lens, Wk, Rk, bk, d, dy[:, :, k * H:(k + 1) * H])
        assert rel(out["y"][:, :, k * H:(k + 1) * H], ref["y"]) < TOL[prec]
        assert rel(out["h_last"][k], ref["h_last"]) < TOL[prec]
        for g in ("dW", "dR", "db"):
            assert rel(out[g][k], ref[g]) < TOL[prec], g
        dx = dx + ref["dx"]
    assert rel(out["dx"], dx) < TOL[prec]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("shape", [(1, 7, 5, 3), (3, 4, 9, 13), (5, 17, 33, 100)])
def test_small_and_odd_shapes(cuda, prec, shape):
    # B = 1, H not a multiple of 8 / 16 (partial unit slices), D not aligned
    B, T, D, H = shape
    x, lens, W, R, b = _seeded(23, B, T, D, H)
    dy = torch.rand(B, T, H, device="cuda") * 2 - 1
    out = run_layer(x, lens, [(W, R, b)], 1, -1, prec, dy)
    ref = torch_ref.sequence(x, lens, W, R, b, -1, dy)
    for k in ("y", "dx"):
        assert rel(out[k], ref[k]) < TOL[prec], k
    for k in ("dW", "dR", "db"):
        assert rel(out[k][0], ref[k]) < TOL[prec], k


@pytest.mark.parametrize("prec", PRECS)
def test_inference_mode_matches_training_forward(cuda, prec):
    # forward without a reserve (inference: nothing saved) gives the same y / final states
    x, lens, W, R, b = _seeded(24, 16, 20, 32, 48)
    layer = lstm.LSTMLayer(16, 20, 32, 48, 2, 1, prec)
    y1, h1, c1 = layer.forward(x, lens, [W, W], [R, R], [b, b], train=True)
    y2, h2, c2 = layer.forward(x, lens, [W, W], [R, R], [b, b], train=False)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(h1, h2) and torch.equal(c1, c2)


def test_bf16_activation_io_matches_fp32_io(cuda):
    # SL_LAYER_X_BF16 / SL_LAYER_Y_BF16 only change the I/O format: fed the same
    # bf16-rounded x, the layer computes exactly what the fp32-I/O layer computes
    B, T, D, H = 37, 11, 70, 48
    x, lens, W, R, b = _seeded(31, B, T, D, H)
    x = x.bfloat16().float()
    W2, R2, b2 = _seeded(32, 1, 1, D, H)[2:]
    dy = torch.rand(B, T, 2 * H, device="cuda") * 2 - 1
    ref = lstm.LSTMLayer(B, T, D, H, 2, 1, "bf16")
    y0, h0, c0 = ref.forward(x, lens, [W, W2], [R, R2], [b, b2])
    g0 = ref.backward(dy)
    xp = torch.zeros(B, T, lstm.bf16_pitch(D), dtype=torch.bfloat16, device="cuda")
    xp[:, :, :D] = x.bfloat16()
    xp[:, :, D] = 1.0
    lay = lstm.LSTMLayer(B, T, D, H, 2, 1, "bf16", x_bf16=True, y_bf16=True)
    y1, h1, c1 = lay.forward(xp, lens, [W, W2], [R, R2], [b, b2])
    g1 = lay.backward(dy)
    torch.cuda.synchronize()
    assert y1.shape == (B, T, lstm.bf16_pitch(2 * H)) and y1.dtype == torch.bfloat16
    assert torch.equal(y1[:, :, :2 * H], y0.bfloat16())
    assert torch.equal(y1[:, :, 2 * H], torch.ones(B, T, dtype=torch.bfloat16, device="cuda"))
    assert torch.equal(h1, h0) and torch.equal(c1, c0)
    assert torch.equal(g1[0], g0[0])
    for k in (1, 2, 3):
        for d in range(2):
            assert torch.equal(g1[k][d], g0[k][d])


@pytest.mark.parametrize("prec", PRECS)
def test_encoder_stack_matches_fp64(cuda, prec):
    # the BASELINE caller (3-layer BLSTM, bf16 activations chained between
    # layers on the bf16 path) against a layer-by-layer fp64 restatement
    from paper_1805_05225_b200.encoder import BLSTMEncoder
    Lyr, B, T, D0, H = 3, 20, 9, 24, 32
    enc = BLSTMEncoder(Lyr, B, T, D0, H, prec)
    enc.init_uniform(5)
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.rand(B, T, D0, device="cuda", generator=g) * 2 - 1
    lens = torch.randint(T // 2, T + 1, (B,), device="cuda", generator=g).int()
    dy = torch.rand(B, T, 2 * H, device="cuda", generator=g) * 2 - 1
    y = enc.forward(x, lens)
    dx = enc.backward(dy)
    torch.cuda.synchronize()
    # fp64 reference: forward through the stack, then backward layer by layer
    inp, saved = x.double(), []
    for l in range(Lyr):
        W, R, bb = enc._wrb(l)
        outs = [torch_ref.sequence(inp, lens, W[k], R[k], bb[k], (1, -1)[k]) for k in range(2)]
        saved.append(inp)
        inp = torch.cat([o["y"] for o in outs], dim=2)
    assert rel(y, inp) < TOL[prec] * 2
    gy = dy.double()
    for l in reversed(range(Lyr)):
        W, R, bb = enc._wrb(l)
        gx = 0
        for k in range(2):
            ref = torch_ref.sequence(saved[l], lens, W[k], R[k], bb[k], (1, -1)[k],
                                     gy[:, :, k * H:(k + 1) * H])
            gv = enc.g_views[l]
            assert rel(gv[3 * k + 0], ref["dW"]) < TOL[prec] * 2, (l, k, "dW")
            assert rel(gv[3 * k + 1], ref["dR"]) < TOL[prec] * 2, (l, k, "dR")
            assert rel(gv[3 * k + 2], ref["db"]) < TOL[prec] * 2, (l, k, "db")
            gx = gx + ref["dx"]
        gy = gx
    assert rel(dx, gy) < TOL[prec] * 2


@pytest.mark.parametrize("L", [60, 41])
def test_equal_lengths_tma_paths_match(cuda, L):
    # equal sequence lengths (the throughput workload: every row at the same
    # time index per step) switch the bf16 forward to TMA-loaded x W tiles;
    # results must equal the per-row load path bit for bit and the fp64 oracle
    B, T, D, H = 200, 60, 96, 1000
    x, _, W, R, b = _seeded(41, B, T, D, H)
    lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
    W2, R2, b2 = _seeded(42, 1, 1, D, H)[2:]
    dy = torch.rand(B, T, 2 * H, device="cuda") * 2 - 1
    outs = []
    for flags in (0, 64):  # 64: experiments switch that disables the TMA x W path
        lstm.lib().sl_debug_set_flags(flags)
        try:
            outs.append(run_layer(x, lens, [(W, R, b), (W2, R2, b2)], 2, 1, "bf16", dy))
        finally:
            lstm.lib().sl_debug_set_flags(0)
    for k in ("y", "h_last", "c_last", "dx"):
        assert torch.equal(outs[0][k], outs[1][k]), k
    for k in ("dW", "dR", "db"):
        for d in range(2):
            assert torch.equal(outs[0][k][d], outs[1][k][d]), k
    for k, (Wk, Rk, bk, d) in enumerate(((W, R, b, 1), (W2, R2, b2, -1))):
        ref = torch_ref.sequence(x, lens, Wk, Rk, bk, d, dy[:, :, k * H:(k + 1) * H])
        assert rel(outs[0]["y"][:, :, k * H:(k + 1) * H], ref["y"]) < TOL["bf16"]
        assert rel(outs[0]["dR"][k], ref["dR"]) < TOL["bf16"]


@pytest.mark.parametrize("prec", PRECS)
def test_seq2seq_training_step_matches_fp64(cuda, prec):
    # the bench's config-4 step (model.py): encoder + decoder over
    # [target embedding ‖ encoder output], gradients through both, then Adam
    from paper_1805_05225_b200.model import Seq2SeqLSTM
    from oracle import adam_ref
    Lyr, B, T, E, H = 2, 12, 7, 20, 24
    m = Seq2SeqLSTM(Lyr, B, T, E, H, prec, lr=1e-2, clip_norm=5.0)
    m.init_uniform(3)
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.rand(B, T, E, device="cuda", generator=g) * 2 - 1
    emb = (torch.rand(B, T, E, device="cuda", generator=g) * 2 - 1)
    if prec == "bf16":
        emb = emb.bfloat16().float()  # the decoder's bf16 input carries it exactly
    lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
    dy = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    m.set_target_embeddings(emb)
    p0 = m.params.clone()
    # fp64 reference of the same composition (with the pre-step parameters)
    inp, saved = x.double(), []
    for l in range(Lyr):
        W, R, bb = [[v.double() for v in vs] for vs in m.enc._wrb(l)]
        outs = [torch_ref.sequence(inp, lens, W[k], R[k], bb[k], (1, -1)[k]) for k in range(2)]
        saved.append((inp, W, R, bb))
        inp = torch.cat([o["y"] for o in outs], dim=2)
    enc_out = inp
    if prec == "bf16":  # the decoder input is stored in bf16 (both parts)
        enc_out = enc_out.bfloat16().double()
    dec_in = torch.cat([emb.double(), enc_out], dim=2)
    Wd, Rd, bd = [t.double() for t in m.dec_p]
    dref = torch_ref.sequence(dec_in, lens, Wd, Rd, bd, 1, dy.double())
    m.step(x, lens, dy)
    torch.cuda.synchronize()
    m.opt.check_finite(m.grads)
    tol = TOL[prec] * 2
    assert rel(m.dec_y, dref["y"]) < tol
    grads_ref = [dref["dW"], dref["dR"], dref["db"]]
    gy = dref["dx"][:, :, E:]
    enc_grads = []
    for l in reversed(range(Lyr)):
        inp_l, W, R, bb = saved[l]
        gx, gl = 0, []
        for k in range(2):
            ref = torch_ref.sequence(inp_l, lens, W[k], R[k], bb[k], (1, -1)[k], gy[:, :, k * H:(k + 1) * H])
            gl += [ref["dW"], ref["dR"], ref["db"]]
            gx = gx + ref["dx"]
        enc_grads = gl + enc_grads
        gy = gx
    flat_ref = torch.cat([t.reshape(-1) for t in enc_grads + grads_ref])
    for (name, off, k) in m.opt.names:
        assert rel(m.grads[off:off + k], flat_ref[off:off + k]) < tol, name
    # and the optimizer applied clip + Adam to exactly these gradients
    pr, _, _, _ = adam_ref.adam_step(p0.double().cpu().numpy(), m.grads.double().cpu().numpy(),
                                     np.zeros(p0.numel()), np.zeros(p0.numel()), 1, lr=float(np.float32(1e-2)),
                                     beta1=float(np.float32(0.9)), beta2=float(np.float32(0.999)),
                                     eps=float(np.float32(1e-8)), clip_norm=5.0)
    assert np.abs(m.params.double().cpu().numpy() - pr).max() < 1e-6



def test_cuda_graph_replay_matches_eager_steps(cuda):
    # the bench times the training step captured as a CUDA graph: replays must
    # reproduce eager steps bit for bit (incl. Adam's device-side step counter)
    from paper_1805_05225_b200.model import Seq2SeqLSTM
    Lyr, B, T, E, H = 2, 40, 9, 24, 64

    def make():
        m = Seq2SeqLSTM(Lyr, B, T, E, H, "bf16", lr=1e-2)
        m.init_uniform(8)
        return m
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.rand(B, T, E, device="cuda", generator=g) * 2 - 1
    emb = torch.rand(B, T, E, device="cuda", generator=g) * 2 - 1
    lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
    dy = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    a, b = make(), make()
    for m in (a, b):
        m.set_target_embeddings(emb)
    for _ in range(3):
        a.step(x, lens, dy)
    b.step(x, lens, dy)  # warm-up outside the capture (allocations, attributes)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        b.step(x, lens, dy)
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(a.params, b.params)
    assert torch.equal(a.opt.m, b.opt.m) and torch.equal(a.opt.v, b.opt.v)


def test_seq2seq_with_output_layer_matches_fp64(cuda):
    # the full bench step incl. the output softmax + label-smoothed CE: the
    # decoder receives dL/dy from the output layer (not a synthetic gradient)
    from paper_1805_05225_b200.model import Seq2SeqLSTM
    Lyr, B, T, E, H, V = 1, 12, 6, 16, 32, 300
    m = Seq2SeqLSTM(Lyr, B, T, E, H, "fp32", vocab=V, label_smoothing=0.1)
    m.init_uniform(5)
    g = torch.Generator(device="cuda").manual_seed(6)
    x = torch.rand(B, T, E, device="cuda", generator=g) * 2 - 1
    emb = torch.rand(B, T, E, device="cuda", generator=g) * 2 - 1
    lens = torch.randint(T // 2, T + 1, (B,), device="cuda", generator=g).int()
    tg = torch.randint(0, V, (B, T), device="cuda", generator=g).int()
    m.set_target_embeddings(emb)
    # fp64 reference of the composition, pre-step parameters
    inp = x.double()
    W, R, bb = [[v.double() for v in vs] for vs in m.enc._wrb(0)]
    enc_out = torch.cat([torch_ref.sequence(inp, lens, W[k], R[k], bb[k], (1, -1)[k])["y"] for k in range(2)], 2)
    dec_in = torch.cat([emb.double(), enc_out], dim=2)
    Wd, Rd, bd = [t.double() for t in m.dec_p]
    dec_y = torch_ref.sequence(dec_in, lens, Wd, Rd, bd, 1)["y"]
    loss, ddy, dWo, dbo = oracle.output_ce_np(dec_y.cpu().numpy(), lens.cpu().numpy(), tg.cpu().numpy(),
                                              m.out_p[0].double().cpu().numpy(), m.out_p[1].double().cpu().numpy(),
                                              0.1)
    dref = torch_ref.sequence(dec_in, lens, Wd, Rd, bd, 1, torch.as_tensor(ddy, device="cuda"))
    l = m.step(x, lens, tg)
    torch.cuda.synchronize()
    # the output layer runs on bf16 tensor cores even in the fp32 LSTM mode
    assert abs(float(l) - loss) < 2e-3 * max(1.0, abs(loss))
    assert rel(m.out_g[0], dWo) < 2e-2 and rel(m.out_g[1], dbo) < 2e-2
    for t_, r_ in zip(m.dec_g, (dref["dW"], dref["dR"], dref["db"])):
        assert rel(t_, r_) < 3e-2


@pytest.mark.parametrize("prec", PRECS)
def test_inference_encoder_matches_training_forward(cuda, prec):
    # BASELINE config 5 path: an inference-only encoder (no reserves, shared
    # workspace, ping-pong activations) gives bit-identical outputs to the
    # training encoder's forward on the same parameters and ragged lengths
    from paper_1805_05225_b200.encoder import BLSTMEncoder
    L, B, T, D, H = 3, 5, 9, 7, 24
    tr = BLSTMEncoder(L, B, T, D, H, precision=prec)
    tr.init_uniform(3)
    inf = BLSTMEncoder(L, B, T, D, H, precision=prec, params=tr.params.clone(), train=False)
    assert all(layer.reserve is None for layer in inf.layers)
    g = torch.Generator().manual_seed(5)
    x = (torch.rand(B, T, D, generator=g) * 2 - 1).cuda()
    lens = torch.tensor([9, 5, 1, 7, 9], dtype=torch.int32).cuda()
    y_tr = tr.forward(x, lens).clone()
    y_inf = inf.forward(x, lens)
    torch.cuda.synchronize()
    assert torch.equal(y_tr, y_inf)
    with pytest.raises(RuntimeError):
        inf.layers[0].forward(x, lens, *inf._wrb(0), train=True)


@pytest.mark.parametrize("prec", PRECS)
def test_seq2seq_from_token_ids_matches_supplied_embeddings(cuda, prec):
    # the `src` / `trg` embedding layers in the config-4 step:
    # starting from ids must give bit-identical losses / gradients to feeding the
    # looked-up embeddings directly, and the two table gradients must be the
    # reference-order scatter of the input gradients (oracle.gather_rows_np)
    from paper_1805_05225_b200.model import Seq2SeqLSTM
    Lyr, B, T, E, H, V, Vs, Vt = 2, 3, 6, 16, 24, 11, 13, 17
    m1 = Seq2SeqLSTM(Lyr, B, T, E, H, prec, vocab=V, src_vocab=Vs, trg_vocab=Vt)
    m1.init_uniform(5)
    m2 = Seq2SeqLSTM(Lyr, B, T, E, H, prec, vocab=V)
    n = m2.params.numel()
    m2.params.copy_(m1.params[:n])
    g = torch.Generator().manual_seed(6)
    src = torch.randint(0, Vs, (B, T), generator=g, dtype=torch.int32).cuda()
    src[0, :4] = 2  # duplicate ids: scatter order matters
    tgt = torch.randint(0, V, (B, T), generator=g, dtype=torch.int32).cuda()
    tgt[1, :] = 3
    tgt %= min(V, Vt)
    lens = torch.tensor([6, 4, 5], dtype=torch.int32).cuda()
    x = m1.src_p[src.long()]
    prev = torch.cat([torch.full((B, 1), -1, dtype=torch.int32, device="cuda"), tgt[:, :-1]], dim=1)
    emb = m1.trg_p[prev.clamp_min(0).long()] * (prev >= 0).unsqueeze(-1)
    m2.set_target_embeddings(emb)
    m1.forward(src, lens, tgt)
    l1 = m1.loss_and_output_grads(tgt, lens)
    m1.backward(m1.dec_dy)
    m2.forward(x, lens)
    l2 = m2.loss_and_output_grads(tgt, lens)
    dx2 = m2.backward(m2.dec_dy)
    torch.cuda.synchronize()
    m1.check_ids()
    assert float(l1) == float(l2)
    assert torch.equal(m1.dec_y, m2.dec_y)
    assert torch.equal(m1.grads[:n], m2.grads)
    _, gs = oracle.gather_rows_np(m1.src_p.cpu().numpy(), src.cpu().numpy(), dx2.cpu().numpy())
    assert np.array_equal(m1.src_g.cpu().numpy(), gs)
    d_emb = m2.dec_dx[:, :, :E].cpu().numpy().reshape(-1, E)
    gt = np.zeros((Vt, E), np.float32)
    for r, v in enumerate(prev.cpu().numpy().reshape(-1)):
        if v >= 0:
            gt[v] += d_emb[r]
    assert np.array_equal(m1.trg_g.cpu().numpy(), gt)


def test_checkpoint_resume_is_bitwise(cuda, tmp_path):
    # SPEC invariant "save -> load -> continue == uninterrupted, bitwise": two
    # steps straight vs one step, save, load into a fresh model, one more step
    from paper_1805_05225_b200.model import Seq2SeqLSTM
    Lyr, B, T, E, H, V = 2, 3, 5, 16, 24, 11
    mk = lambda: Seq2SeqLSTM(Lyr, B, T, E, H, "bf16", vocab=V, src_vocab=13, trg_vocab=V)
    g = torch.Generator().manual_seed(9)
    src = torch.randint(0, 13, (B, T), generator=g, dtype=torch.int32).cuda()
    tgt = torch.randint(0, V, (B, T), generator=g, dtype=torch.int32).cuda()
    lens = torch.tensor([5, 3, 4], dtype=torch.int32).cuda()
    a = mk()
    a.init_uniform(1)
    b = mk()
    b.params.copy_(a.params)
    a.step(src, lens, tgt)
    a.step(src, lens, tgt)
    b.step(src, lens, tgt)
    b.save(str(tmp_path), epoch=1)
    c = mk()
    meta = c.load(str(tmp_path))
    assert meta["epoch"] == 1 and meta["params"][-1]["name"] == "trg/W"
    assert c.opt.device_step() == 1
    c.step(src, lens, tgt)
    torch.cuda.synchronize()
    assert torch.equal(a.params, c.params)
