"""CPU tests: pin the oracle before trusting it (no GPU needed).

* the C restatement (oracle/lstm_oracle.c) against the golden fixtures that the
  REFERENCE produced (tests/golden/make_golden.py),
* against the reference build itself on fresh seeded cases when
  oracle/_ref is present,
* against the reference's own known answers (tape_test.cpp:191-213,
  SPEC.md:305-318) and central finite differences (gradcheck.cpp:25-68),
* the torch fp64 restatement (oracle/torch_ref.py) against the C restatement,
* the reference's own unit tests compiled unmodified (oracle/_ref/tape_test64).
"""
import glob
import os
import subprocess

import numpy as np
import pytest
import torch

import oracle
from oracle import torch_ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REF = os.path.join(os.path.dirname(oracle.__file__), "_ref")


@pytest.fixture(scope="module")
def orc():
    return oracle.Restatement()


def _ref_available():
    return os.path.exists(os.path.join(REF, "libseqloom_ref64.so"))


def rel(a, b):
    """Norm-wise relative error max|a-b| / max|b| (SURVEY §9 parity metric)."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


SEQ_FIXTURES = ["config1_fw", "config1_bw", "t1_bw", "lens35_fw", "odd_bw"]


@pytest.mark.parametrize("name", SEQ_FIXTURES)
def test_restatement_matches_reference_goldens(orc, name):
    f = np.load(os.path.join(GOLD, name + ".npz"))
    d = int(f["direction"])
    y, _, _ = orc.sequence_fwd(f["x"], f["lens"], f["W"], f["R"], f["b"], d)
    assert rel(y, f["y_ref64"]) < 1e-12
    g = orc.sequence_bwd(f["x"], f["lens"], f["W"], f["R"], f["b"], d, f["dy"])
    for k, v in zip(("dx", "dW", "dR", "db"), g):
        assert rel(v, f[k + "_ref64"]) < 1e-12, k
        # the reference's own float build agrees with its fp64 build to fp32 rounding
        assert rel(f[k + "_ref32"], f[k + "_ref64"]) < 1e-4, k


def test_masked_outputs_exactly_zero(orc):
    # seq_lens [3, 5] -> entry 0's output at t >= 3 is zero
    f = np.load(os.path.join(GOLD, "lens35_fw.npz"))
    assert np.all(f["y_ref64"][0, 3:] == 0.0)
    y, _, _ = orc.sequence_fwd(f["x"], f["lens"], f["W"], f["R"], f["b"], 1)
    assert np.all(y[0, 3:] == 0.0)
    assert np.all(np.abs(y[0, :3]) > 0)


def test_t1_both_directions_identical(orc):
    # Time=1 -> identical output for both directions
    f = np.load(os.path.join(GOLD, "t1_bw.npz"))
    yf, _, _ = orc.sequence_fwd(f["x"], f["lens"], f["W"], f["R"], f["b"], 1)
    yb, _, _ = orc.sequence_fwd(f["x"], f["lens"], f["W"], f["R"], f["b"], -1)
    assert np.array_equal(yf, yb)


def test_backward_is_rev_forward_rev(orc):
    # direction -1 == reverse_per_seq . (direction +1) . reverse_per_seq
    x, lens, W, R, b = oracle.seeded_case(3, 4, 9, 5, 6)
    def rev(a):
        out = a.copy()
        for r, L in enumerate(lens):
            out[r, :L] = a[r, :L][::-1]
        return out
    yb, _, _ = orc.sequence_fwd(x, lens, W, R, b, -1)
    yf, _, _ = orc.sequence_fwd(rev(x), lens, W, R, b, 1)
    assert np.allclose(yb, rev(yf), rtol=0, atol=1e-15)


def test_step_hand_values(orc):
    # tape_test.cpp:191-213 (and the reference's own values in the fixture)
    f = np.load(os.path.join(GOLD, "lstm_step.npz"))
    z = np.zeros
    h, c, _ = orc.step_fwd(z((1, 2)), z((1, 3)), z((1, 3)), z((2, 12)), z((3, 12)), z(12))
    assert np.all(h == 0) and np.all(c == 0)
    h, c, _ = orc.step_fwd(z((1, 2)), z((1, 3)), np.full((1, 3), 2.0), z((2, 12)), z((3, 12)),
                           z(12))
    assert np.allclose(c, 1.0) and np.allclose(h, 0.5 * np.tanh(1.0))
    assert np.allclose(f["hand_c2_h"], 0.5 * np.tanh(1.0)) and np.allclose(f["hand_c2_c"], 1.0)
    args = [f["rand_" + k] for k in ("x", "h0", "c0", "W", "R", "b")]
    h, c, _ = orc.step_fwd(*args)
    assert rel(h, f["rand_h"]) < 1e-14 and rel(c, f["rand_c"]) < 1e-14
    g = orc.step_bwd(*args, f["rand_gh"], f["rand_gc"])
    for k, v in zip(("dx", "dh0", "dc0", "dW", "dR", "db"), g):
        assert rel(v, f["rand_" + k]) < 1e-13, k


def test_finite_differences(orc):
    # central differences, fp64, rel < 1e-4 (gradcheck.cpp:25-68, tape_test.cpp:477-492)
    x, lens, W, R, b = oracle.seeded_case(21, 3, 5, 4, 3)
    dy = np.random.default_rng(5).uniform(-1, 1, (3, 5, 3))
    for d in (1, -1):
        g = orc.sequence_bwd(x, lens, W, R, b, d, dy)
        def loss(x_, W_, R_, b_):
            y, _, _ = orc.sequence_fwd(x_, lens, W_, R_, b_, d)
            return float((y * dy).sum())
        vals = [x, W, R, b]
        rng = np.random.default_rng(9)
        for i, a in enumerate(vals):
            for _ in range(12):
                idx = tuple(rng.integers(0, s) for s in a.shape)
                ap, am = a.copy(), a.copy()
                ap[idx] += 1e-6
                am[idx] -= 1e-6
                up = loss(*[ap if j == i else v for j, v in enumerate(vals)])
                dn = loss(*[am if j == i else v for j, v in enumerate(vals)])
                num = (up - dn) / 2e-6
                an = g[i][idx]
                assert abs(an - num) / max(abs(an), abs(num), 1e-8) < 1e-4 or abs(an - num) < 1e-9


def test_final_state_gradients_fd(orc):
    # h_last / c_last extension: dL/d(inputs) through dh_last, dc_last
    x, lens, W, R, b = oracle.seeded_case(22, 3, 6, 4, 3)
    dh = np.random.default_rng(1).uniform(-1, 1, (3, 3))
    dc = np.random.default_rng(2).uniform(-1, 1, (3, 3))
    dy0 = np.zeros((3, 6, 3))
    for d in (1, -1):
        g = orc.sequence_bwd(x, lens, W, R, b, d, dy0, dh, dc)
        def loss(W_):
            _, hl, cl = orc.sequence_fwd(x, lens, W_, R, b, d)
            return float((hl * dh).sum() + (cl * dc).sum())
        for idx in [(0, 0), (1, 5), (3, 11)]:
            Wp, Wm = W.copy(), W.copy()
            Wp[idx] += 1e-6
            Wm[idx] -= 1e-6
            num = (loss(Wp) - loss(Wm)) / 2e-6
            assert abs(g[1][idx] - num) < 1e-7 + 1e-5 * abs(num)


@pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("d", [1, -1])
def test_restatement_matches_reference_build(orc, d):
    ref = oracle.Reference(64)
    x, lens, W, R, b = oracle.seeded_case(40 + d, 6, 11, 7, 9)
    dy = np.random.default_rng(3).uniform(-1, 1, (6, 11, 9))
    y, g = ref.sequence(x, lens, W, R, b, d, dy)
    yo, _, _ = orc.sequence_fwd(x, lens, W, R, b, d)
    go = orc.sequence_bwd(x, lens, W, R, b, d, dy)
    assert rel(yo, y) < 1e-12
    for a, c in zip(go, g):
        assert rel(a, c) < 1e-12


@pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built")
def test_reference_stack_matches_golden():
    f = np.load(os.path.join(GOLD, "blstm2.npz"))
    L = int(f["L"])
    params = [tuple(f[f"{n}_{l}"] for n in ("W_fw", "R_fw", "b_fw", "W_bw", "R_bw", "b_bw"))
              for l in range(L)]
    y, dx, grads = oracle.Reference(64).blstm_stack(f["x"], f["lens"], params, f["dy"])
    assert rel(y, f["y_ref64"]) < 1e-13 and rel(dx, f["dx_ref64"]) < 1e-13


def test_restatement_stack_matches_golden(orc):
    # the BLSTM stack from layer restatements: input of layer l = [fw ‖ bw] of layer l-1
    f = np.load(os.path.join(GOLD, "blstm2.npz"))
    L = int(f["L"])
    xs = [f["x"]]
    inp = f["x"]
    for l in range(L):
        ys = [orc.sequence_fwd(inp, f["lens"], f[f"W_{n}_{l}"], f[f"R_{n}_{l}"], f[f"b_{n}_{l}"],
                               1 if n == "fw" else -1)[0] for n in ("fw", "bw")]
        inp = np.concatenate(ys, axis=2)
        xs.append(inp)
    assert rel(inp, f["y_ref64"]) < 1e-13
    g = f["dy"]
    for l in reversed(range(L)):
        H = f[f"R_fw_{l}"].shape[0]
        dx = 0
        for k, n in enumerate(("fw", "bw")):
            gx, gW, gR, gb = orc.sequence_bwd(xs[l], f["lens"], f[f"W_{n}_{l}"], f[f"R_{n}_{l}"],
                                              f[f"b_{n}_{l}"], 1 if n == "fw" else -1,
                                              g[:, :, k * H:(k + 1) * H])
            assert rel(gW, f[f"dW_{n}_{l}_ref64"]) < 1e-12
            assert rel(gR, f[f"dR_{n}_{l}_ref64"]) < 1e-12
            assert rel(gb, f[f"db_{n}_{l}_ref64"]) < 1e-12
            dx = dx + gx
        g = dx
    assert rel(g, f["dx_ref64"]) < 1e-12


@pytest.mark.parametrize("d", [1, -1])
def test_torch_restatement_matches_c(orc, d):
    x, lens, W, R, b = oracle.seeded_case(50 + d, 5, 8, 6, 7)
    dy = np.random.default_rng(4).uniform(-1, 1, (5, 8, 7))
    dh = np.random.default_rng(5).uniform(-1, 1, (5, 7))
    dc = np.random.default_rng(6).uniform(-1, 1, (5, 7))
    T = lambda a: torch.from_numpy(np.asarray(a))
    out = torch_ref.sequence(T(x), T(lens), T(W), T(R), T(b), d, T(dy), T(dh), T(dc))
    y, hl, cl = orc.sequence_fwd(x, lens, W, R, b, d)
    g = orc.sequence_bwd(x, lens, W, R, b, d, dy, dh, dc)
    assert rel(out["y"].numpy(), y) < 1e-13
    assert rel(out["h_last"].numpy(), hl) < 1e-13 and rel(out["c_last"].numpy(), cl) < 1e-13
    for k, v in zip(("dx", "dW", "dR", "db"), g):
        assert rel(out[k].numpy(), v) < 1e-12, k


@pytest.mark.skipif(not os.path.exists(os.path.join(REF, "tape_test64")),
                    reason="reference unit tests not built")
def test_reference_own_unit_tests_pass():
    # the reference's tape_test.cpp / tensor_test.cpp, unmodified, on our shims
    for exe in ("tape_test64", "tensor_test"):
        r = subprocess.run([os.path.join(REF, exe)], capture_output=True, text=True,
                           env={**os.environ, "OPENBLAS_NUM_THREADS": "1"})
        assert r.returncode == 0, r.stdout + r.stderr
        assert "failed: 0" in r.stdout


def test_output_ce_restatement_pinned_to_reference():
    # the decoder output layer + loss: numpy restatement vs the
    # reference's own Tape ops (matmul, add, log_softmax, ce_label_smoothing)
    import oracle
    ref = oracle.Reference(64)
    rng = np.random.default_rng(3)
    B, T, D, V = 4, 6, 9, 23
    x = rng.uniform(-1, 1, (B, T, D))
    W = rng.uniform(-0.4, 0.4, (D, V))
    b = rng.uniform(-0.4, 0.4, V)
    lens = np.array([6, 2, 5, 1], np.int32)
    tg = rng.integers(0, V, (B, T)).astype(np.int32)
    for eps in (0.0, 0.1, 0.5):
        a = ref.output_ce(x, lens, tg, W, b, eps)
        n = oracle.output_ce_np(x, lens, tg, W, b, eps)
        assert abs(a[0] - n[0]) < 1e-12
        for p, q in zip(a[1:], n[1:]):
            assert np.abs(p - q).max() < 1e-12
    # uniform logits: every lp = -log V, so the loss is log V for any eps
    loss = oracle.output_ce_np(np.zeros((1, 2, 3)), [2], np.zeros((1, 2), np.int32), np.zeros((3, 7)),
                               np.zeros(7), 0.3)[0]
    assert abs(loss - np.log(7)) < 1e-12
    # the reference's argument errors
    with pytest.raises(RuntimeError, match=r"epsilon must be in \[0, 1\)"):
        ref.output_ce(x, lens, tg, W, b, 1.0)
    bad = tg.copy()
    bad[0, 0] = V
    with pytest.raises(RuntimeError, match="out of range"):
        ref.output_ce(x, lens, bad, W, b, 0.1)


def test_attention_step_restatement_pinned_to_reference():
    # the decoder's MLP attention step: numpy restatement vs the
    # reference's own layer ops (matmul/add/tanh/softmax_over_spatial/generic_attention)
    import oracle
    ref = oracle.Reference(64)
    rng = np.random.default_rng(11)
    B, Ts, K, E, H = 3, 6, 9, 8, 5
    lens = np.array([6, 2, 4], np.int32)
    args = dict(enc_ctx=rng.uniform(-1, 1, (B, Ts, K)), enc=rng.uniform(-1, 1, (B, Ts, E)),
                s=rng.uniform(-1, 1, (B, H)), accum=rng.uniform(0, 1, (B, Ts)), Ws=rng.uniform(-.5, .5, (H, K)),
                bs=rng.uniform(-.5, .5, K), Wfb=rng.uniform(-.5, .5, (1, K)), bfb=rng.uniform(-.5, .5, K),
                v=rng.uniform(-.5, .5, (K, 1)), bv=0.3)
    d_att, d_acc = rng.uniform(-1, 1, (B, E)), rng.uniform(-1, 1, (B, Ts))
    r = ref.attention_step(lens, **args, d_att=d_att, d_accum=d_acc)
    n = oracle.attention_step_np(lens, **args, d_att=d_att, d_accum=d_acc)
    for i in range(3):
        assert np.abs(r[i] - n[i]).max() < 1e-12
    for k in r[3]:
        assert np.abs(r[3][k].reshape(n[3][k].shape) - n[3][k]).max() < 1e-12, k
    # padded source positions get no attention weight
    assert np.all(n[1][1, 2:] == 0) and abs(n[1][1].sum() - 1) < 1e-12


def test_gather_rows_oracle_pinned_to_reference_test():
    # reference tape_test.cpp:81-104: table {1,2,3,4} [2, 2], ids {1, 0} -> {3,4,1,2};
    # ids {0, 0} with L = sum(out) -> table grad {2, 2, 0, 0}; id 7 -> IndexError naming "emb"
    tbl = np.array([[1, 2], [3, 4]], dtype=np.float32)
    out, _ = oracle.gather_rows_np(tbl, np.array([1, 0]))
    assert out.reshape(-1).tolist() == [3, 4, 1, 2]
    _, g = oracle.gather_rows_np(tbl, np.array([0, 0]), d_out=np.ones((2, 2), np.float32))
    assert g.reshape(-1).tolist() == [2, 2, 0, 0]
    with pytest.raises(IndexError, match="emb"):
        oracle.gather_rows_np(tbl, np.array([7]))


@pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built")
def test_gather_rows_restatement_matches_reference_bitwise():
    rng = np.random.default_rng(11)
    V, D, B, T = 13, 7, 5, 9
    tbl = rng.uniform(-1, 1, (V, D)).astype(np.float32)
    ids = rng.integers(0, V, (B, T)).astype(np.int32)
    ids[0, :] = 3  # a long duplicate run: order of the fp32 adds matters
    d_out = rng.uniform(-1, 1, (B, T, D)).astype(np.float32)
    ref = oracle.Reference(32)
    out_r, g_r = ref.gather_rows(tbl, ids, d_out)
    out_o, g_o = oracle.gather_rows_np(tbl, ids, d_out)
    assert np.array_equal(out_r.astype(np.float32), out_o)
    assert np.array_equal(g_r.astype(np.float32), g_o)
    with pytest.raises(IndexError, match="in layer 'emb'"):
        ref.gather_rows(tbl, np.full((1, 1), V, np.int32))


def test_torch64_output_ce_restatement_matches_numpy_restatement():
    """The fp64-torch restatement the config-4 output-layer GPU test uses
    (tests/test_output_gpu.py::_output_ce_torch64) equals oracle.output_ce_np."""
    import torch
    from test_output_gpu import _output_ce_torch64
    rng = np.random.default_rng(4)
    B, T, D, V = 5, 7, 11, 37
    x, W, b = rng.uniform(-1, 1, (B, T, D)), rng.uniform(-1, 1, (D, V)), rng.uniform(-1, 1, V)
    lens = np.array([7, 3, 5, 1, 7], np.int32)
    tg = rng.integers(0, V, (B, T)).astype(np.int32)
    ref = oracle.output_ce_np(x, lens, tg, W, b, 0.1)
    got = _output_ce_torch64(*(torch.as_tensor(a) for a in (x, lens, tg, W, b)), 0.1)
    for r, g in zip(ref, got):
        assert np.allclose(np.asarray(g), r, rtol=1e-12, atol=1e-14)
