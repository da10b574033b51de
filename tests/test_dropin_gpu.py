"""The drop-in, end to end: the reference's OWN Tape (tape.cpp, compiled
unmodified) with seqloom::lstm_sequence supplied by
paper_1805_05225_b200/host/dropin/layers_cuda.cpp (our C ABI, CUDA kernels),
driven through the same bridge entry points as the pure-reference build —
Tape::backward / param_gradients included.  Compared call for call with the
reference's own CPU lstm_sequence (oracle/_ref/libseqloom_ref32.so) and with
the fp64 golden fixtures."""
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
    p = os.path.join(REF, "libseqloom_dropin32.so")
    if not os.path.exists(p):
        pytest.fail("oracle/_ref/libseqloom_dropin32.so missing: build() must run make -C oracle dropin")
    return oracle.Reference(path=p), oracle.Reference(path=os.path.join(REF, "libseqloom_ref32.so"))


@pytest.mark.parametrize("name", ["config1_fw", "config1_bw", "odd_bw", "lens35_fw", "t1_bw"])
def test_dropin_matches_reference(libs, name):
    dropin, ref32 = libs
    f = np.load(os.path.join(GOLD, name + ".npz"))
    d = int(f["direction"])
    args = (f["x"], f["lens"], f["W"], f["R"], f["b"], d, f["dy"])
    y, g = dropin.sequence(*args)
    yr, gr = ref32.sequence(*args)
    assert rel(y, f["y_ref64"]) < 1e-4 and rel(y, yr) < 1e-4
    for k, a, r in zip(("dx", "dW", "dR", "db"), g, gr):
        assert rel(a, f[k + "_ref64"]) < 1e-4, k
        assert rel(a, r) < 1e-4, k
    lens = f["lens"]
    for r_, L in enumerate(lens):
        assert np.all(y[r_, L:] == 0.0)


def test_dropin_bidirectional_stack(libs):
    # the reference's concat_feature + our lstm_sequence, two BLSTM layers
    dropin, _ = libs
    f = np.load(os.path.join(GOLD, "blstm2.npz"))
    L = int(f["L"])
    params = [tuple(f[f"{n}_{l}"] for n in ("W_fw", "R_fw", "b_fw", "W_bw", "R_bw", "b_bw"))
              for l in range(L)]
    y, dx, grads = dropin.blstm_stack(f["x"], f["lens"], params, f["dy"])
    assert rel(y, f["y_ref64"]) < 1e-4
    assert rel(dx, f["dx_ref64"]) < 1e-4
    for l in range(L):
        for j, n in enumerate(("W_fw", "R_fw", "b_fw", "W_bw", "R_bw", "b_bw")):
            assert rel(grads[l][j], f[f"d{n}_{l}_ref64"]) < 1e-4, (l, n)


def test_dropin_errors_like_reference(libs):
    dropin, ref32 = libs
    x, lens, W, R, b = oracle.seeded_case(1, 2, 3, 4, 5)
    for lib in (dropin, ref32):
        with pytest.raises(RuntimeError, match="direction must be \\+1 or -1"):
            lib.sequence(x, lens, W, R, b, 0)


def test_dropin_bf16(libs, monkeypatch):
    dropin, _ = libs
    monkeypatch.setenv("SEQLOOM_CUDA_PRECISION", "bf16")
    f = np.load(os.path.join(GOLD, "config1_bw.npz"))
    y, g = dropin.sequence(f["x"], f["lens"], f["W"], f["R"], f["b"], -1, f["dy"])
    assert rel(y, f["y_ref64"]) < 2e-2
    for k, a in zip(("dx", "dW", "dR", "db"), g):
        assert rel(a, f[k + "_ref64"]) < 2e-2, k
