"""The Tape::lstm_step drop-in end to end: the reference's
OWN Tape, tensor, layers and gradcheck sources, with Tape::lstm_step supplied by
paper_1805_05225_b200/host/dropin/tape_lstm_step_cuda.cpp (our C ABI on the
GPU) in place of tape.cpp:1074-1222 (oracle/Makefile target dropin-step).

  * the reference's own lstm_step hand values (tape_test.cpp:191-213);
  * the graph of the reference's own lstm_step finite-difference test
    (tape_test.cpp:477-492, two chained steps, every input a parameter) against
    the reference fp64 build, whose gradients this test also FD-checks;
  * the reference's own lstm_sequence (layers.cpp:8-37, which calls
    tape.lstm_step per time step) running on the GPU cell, against the golden
    fixtures and the pure reference build;
  * the decoder cell at the config-4 width (D = 620 + 2000, H = 1000).
fp32 tolerance 1e-4 (max-normalised per tensor)."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
REF = os.path.join(os.path.dirname(oracle.__file__), "_ref")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def libs(cuda):
    p = os.path.join(REF, "libseqloom_dropin_step32.so")
    if not os.path.exists(p):
        pytest.fail("oracle/_ref/libseqloom_dropin_step32.so missing: build() must run make -C oracle dropin-step")
    return (oracle.Reference(path=p), oracle.Reference(path=os.path.join(REF, "libseqloom_ref32.so")),
            oracle.Reference(path=os.path.join(REF, "libseqloom_ref64.so")))


def test_lstm_step_hand_values_through_dropin(libs):
    """tape_test.cpp:191-213: zero weights; c_prev = 0 -> h = c = 0; c_prev = 2 -> c = 1, h = 0.5 tanh 1."""
    dropin, _, _ = libs
    h, dx = 3, 2
    W, R, b = np.zeros((dx, 4 * h)), np.zeros((h, 4 * h)), np.zeros(4 * h)
    x, h0 = np.zeros((1, dx)), np.zeros((1, h))
    h_, c_, _ = dropin.step(x, h0, np.zeros((1, h)), W, R, b)
    assert np.all(h_ == 0) and np.all(c_ == 0)
    h_, c_, _ = dropin.step(x, h0, np.full((1, h), 2.0), W, R, b)
    assert np.allclose(c_, 1.0, rtol=1e-6) and np.allclose(h_, 0.5 * np.tanh(1.0), rtol=1e-6)
    f = np.load(os.path.join(GOLD, "lstm_step.npz"))
    assert np.allclose(h_, f["hand_c2_h"], rtol=1e-6) and np.allclose(c_, f["hand_c2_c"], rtol=1e-6)


def test_lstm_step_golden_gradients_through_dropin(libs):
    dropin, _, _ = libs
    f = np.load(os.path.join(GOLD, "lstm_step.npz"))
    h, c, g = dropin.step(f["rand_x"], f["rand_h0"], f["rand_c0"], f["rand_W"], f["rand_R"], f["rand_b"],
                          gh=f["rand_gh"], gc=f["rand_gc"])
    assert rel(h, f["rand_h"]) < 1e-4 and rel(c, f["rand_c"]) < 1e-4
    for k, a in zip(("dx", "dh0", "dc0", "dW", "dR", "db"), g):
        assert rel(a, f["rand_" + k]) < 1e-4, k


def test_two_chained_steps_match_reference_fd_graph(libs):
    """tape_test.cpp:477-492's graph (B=2, Dx=2, H=3, random weights): loss and the
    gradients of all six inputs through the drop-in vs the fp64 reference build; the
    fp64 reference's gradients are themselves checked by central differences here."""
    dropin, _, ref64 = libs
    rng = np.random.default_rng(11)
    B, D, H = 2, 2, 3
    args = [rng.uniform(-1, 1, s) for s in ((B, D), (B, H), (B, H), (D, 4 * H), (H, 4 * H), (4 * H,))]
    got = dropin.two_steps(*args)
    want = ref64.two_steps(*args)
    assert abs(got[0] - want[0]) < 1e-5 * max(1.0, abs(want[0]))
    for k, (a, r) in enumerate(zip(got[1:], want[1:])):
        assert rel(a, r) < 1e-4, k
    eps = 1e-6  # the reference's own FD check of the fp64 gradients (tape_test.cpp:368-376, rel < 1e-4)
    for i, arr in enumerate(args):
        for j in range(arr.size):
            p = [a.copy() for a in args]
            m = [a.copy() for a in args]
            p[i].flat[j] += eps
            m[i].flat[j] -= eps
            fd = (ref64.two_steps(*p)[0] - ref64.two_steps(*m)[0]) / (2 * eps)
            assert abs(fd - want[1 + i].flat[j]) < 1e-6 + 1e-4 * abs(fd), (i, j)


@pytest.mark.parametrize("name", ["config1_fw", "config1_bw", "odd_bw", "lens35_fw", "t1_bw"])
def test_reference_lstm_sequence_on_the_dropin_cell(libs, name):
    """layers.cpp's own lstm_sequence (T calls of tape.lstm_step) on the GPU cell."""
    dropin, ref32, _ = libs
    f = np.load(os.path.join(GOLD, name + ".npz"))
    args = (f["x"], f["lens"], f["W"], f["R"], f["b"], int(f["direction"]), f["dy"])
    y, g = dropin.sequence(*args)
    yr, gr = ref32.sequence(*args)
    assert rel(y, f["y_ref64"]) < 1e-4 and rel(y, yr) < 1e-4
    for k, a, r in zip(("dx", "dW", "dR", "db"), g, gr):
        assert rel(a, f[k + "_ref64"]) < 1e-4, k


def test_decoder_cell_at_config4_width(libs):
    """The RnnCell `s` of the Listing-1 decoder (compiler.cpp:640-650) at D = 620 + 2000,
    H = 1000, B = 16 through the drop-in, against the fp64 reference build."""
    dropin, _, ref64 = libs
    rng = np.random.default_rng(5)
    B, D, H = 16, 2620, 1000
    s = 1 / np.sqrt(H)
    x, h0, c0 = rng.uniform(-1, 1, (B, D)), rng.uniform(-1, 1, (B, H)), rng.uniform(-1, 1, (B, H))
    W, R, b = rng.uniform(-s, s, (D, 4 * H)), rng.uniform(-s, s, (H, 4 * H)), rng.uniform(-s, s, 4 * H)
    gh, gc = rng.uniform(-1, 1, (B, H)), rng.uniform(-1, 1, (B, H))
    h, c, g = dropin.step(x, h0, c0, W, R, b, gh=gh, gc=gc)
    hr, cr, gr = ref64.step(x, h0, c0, W, R, b, gh=gh, gc=gc)
    assert rel(h, hr) < 1e-4 and rel(c, cr) < 1e-4
    for k, (a, r) in enumerate(zip(g, gr)):
        assert rel(a, r) < 1e-4, k
