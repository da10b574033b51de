"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

    make -C oracle ref && python tests/golden/make_golden.py

Every output below is produced by the unmodified reference sources
(/root/reference/proj/core/src/{tensor,tape,layers}.cpp) compiled into
oracle/_ref/libseqloom_ref{32,64}.so — the fp64 build (the reference's
gradient-check build, core/CMakeLists.txt:34-42) for `*_ref64` arrays and the
default float build for `*_ref32`.  Inputs are seeded (oracle.seeded_case).
The fixtures travel with the repo, so the GPU box (which has no
/root/reference) can check the CUDA path against the reference's own numbers.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402


def seq_case(name, seed, B, T, D, H, direction, ragged=True, lens=None):
    r64, r32 = oracle.Reference(64), oracle.Reference(32)
    x, l, W, R, b = oracle.seeded_case(seed, B, T, D, H, ragged=ragged)
    if lens is not None:
        l = np.asarray(lens, dtype=np.int32)
    dy = np.random.default_rng(seed + 1000).uniform(-1, 1, (B, T, H))
    y64, g64 = r64.sequence(x, l, W, R, b, direction, dy)
    y32, g32 = r32.sequence(x, l, W, R, b, direction, dy)
    out = dict(x=x, lens=l, W=W, R=R, b=b, dy=dy, direction=np.int32(direction),
               y_ref64=y64, y_ref32=y32)
    for k, a64, a32 in zip(("dx", "dW", "dR", "db"), g64, g32):
        out[k + "_ref64"] = a64
        out[k + "_ref32"] = a32
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def stack_case(name, seed, L, B, T, D0, H):
    r64 = oracle.Reference(64)
    x, lens, *_ = oracle.seeded_case(seed, B, T, D0, H)
    params = []
    for l in range(L):
        D = D0 if l == 0 else 2 * H
        p = []
        for d in range(2):
            _, _, W, R, b = oracle.seeded_case(seed + 10 * l + d + 1, 1, 1, D, H)
            p += [W, R, b]
        params.append(tuple(p))
    dy = np.random.default_rng(seed + 1000).uniform(-1, 1, (B, T, 2 * H))
    y, dx, grads = r64.blstm_stack(x, lens, params, dy)
    out = dict(x=x, lens=lens, dy=dy, y_ref64=y, dx_ref64=dx, L=np.int32(L))
    for l in range(L):
        for j, n in enumerate(("W_fw", "R_fw", "b_fw", "W_bw", "R_bw", "b_bw")):
            out[f"{n}_{l}"] = params[l][j]
            out[f"d{n}_{l}_ref64"] = grads[l][j]
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def step_cases(name):
    r64 = oracle.Reference(64)
    out = {}
    # tape_test.cpp:191-213 / SPEC.md:305-308: zero weights, c_prev = 0 and 2.
    H, D = 3, 2
    z = lambda *s: np.zeros(s)
    for tag, cval in (("c0", 0.0), ("c2", 2.0)):
        h, c, _ = r64.step(z(1, D), z(1, H), np.full((1, H), cval), z(D, 4 * H), z(H, 4 * H),
                           z(4 * H))
        out[f"hand_{tag}_h"], out[f"hand_{tag}_c"] = h, c
    # random step with gradients (tape_test.cpp:477-492 shapes, larger)
    rng = np.random.default_rng(7)
    B, D, H = 4, 6, 5
    args = [rng.uniform(-1, 1, s) for s in ((B, D), (B, H), (B, H), (D, 4 * H), (H, 4 * H),
                                            (4 * H,), (B, H), (B, H))]
    h, c, g = r64.step(*args)
    for k, v in zip(("x", "h0", "c0", "W", "R", "b", "gh", "gc"), args):
        out["rand_" + k] = v
    out["rand_h"], out["rand_c"] = h, c
    for k, v in zip(("dx", "dh0", "dc0", "dW", "dR", "db"), g):
        out["rand_" + k] = v
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


if __name__ == "__main__":
    oracle.build()
    # config 1 (BASELINE configs[0]): H = D = 128, B = 8, T = 20, both directions, ragged
    seq_case("config1_fw", 11, 8, 20, 128, 128, +1)
    seq_case("config1_bw", 12, 8, 20, 128, 128, -1)
    # SPEC.md:315-318 examples: T=1, and seq_lens [3, 5]
    seq_case("t1_bw", 13, 3, 1, 7, 5, -1, ragged=False)
    seq_case("lens35_fw", 14, 2, 5, 4, 6, +1, lens=[3, 5])
    seq_case("odd_bw", 15, 5, 9, 13, 37, -1)
    # a 2-layer bidirectional stack wired like eval_layer (compiler.cpp:600-608)
    stack_case("blstm2", 16, 2, 4, 7, 9, 6)
    step_cases("lstm_step")
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))
