"""The decoder output layer + label-smoothed CE on the GPU
against the fp64 restatement pinned to the reference (tests/test_oracle.py)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1805_05225_b200.output import OutputCE

pytestmark = pytest.mark.gpu
TOL = 2e-2  # bf16 operands, fp32 accumulation (the bf16 path's bound)


def rel(a, b):
    a = torch.as_tensor(a).double().cpu()
    b = torch.as_tensor(b).double().cpu()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("B,T,D,V,eps", [(8, 5, 64, 300, 0.1), (20, 13, 200, 1003, 0.0), (16, 30, 1000, 4096, 0.1)])
def test_output_ce_matches_reference_restatement(cuda, B, T, D, V, eps):
    g = torch.Generator().manual_seed(B * 131 + V)
    x = torch.rand(B, T, D, generator=g, dtype=torch.float64) * 2 - 1
    W = (torch.rand(D, V, generator=g, dtype=torch.float64) * 2 - 1) * D ** -0.5 * 3
    b = (torch.rand(V, generator=g, dtype=torch.float64) * 2 - 1) * 0.5
    lens = torch.randint(T // 2, T + 1, (B,), generator=g, dtype=torch.int32)
    lens[0] = T
    tg = torch.randint(0, V, (B, T), generator=g, dtype=torch.int32)
    # the GPU computes in bf16: compare against the fp64 restatement on the
    # bf16-rounded operands so only accumulation / softmax error remains
    xr, Wr = x.float().bfloat16().double(), W.float().bfloat16().double()
    loss, dx, dW, db = oracle.output_ce_np(xr.numpy(), lens.numpy(), tg.numpy(), Wr.numpy(), b.numpy(), eps)
    out = OutputCE(B, T, D, V, eps)
    l, gdx, gdW, gdb = out.forward_backward(x.float().cuda(), tg.cuda(), lens.cuda(), W.float().cuda(),
                                            b.float().cuda())
    torch.cuda.synchronize()
    out.check_targets()
    assert abs(float(l) - loss) < 1e-3 * max(1.0, abs(loss))
    assert rel(gdx, dx) < TOL
    assert rel(gdW, dW) < TOL
    assert rel(gdb, db) < TOL
    # masked positions (t >= len) carry no gradient
    for bb in range(B):
        assert float(gdx[bb, int(lens[bb]):].abs().max() if int(lens[bb]) < T else 0.0) == 0.0


def test_output_ce_errors_like_reference(cuda):
    B, T, D, V = 2, 3, 16, 50
    x = torch.rand(B, T, D, device="cuda")
    W = torch.rand(D, V, device="cuda")
    b = torch.zeros(V, device="cuda")
    lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
    tg = torch.randint(0, V, (B, T), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match=r"epsilon must be in \[0, 1\)"):
        OutputCE(B, T, D, V, 1.0).forward_backward(x, tg, lens, W, b)
    bad = tg.clone()
    bad[1, 2] = V + 4
    out = OutputCE(B, T, D, V, 0.1)
    out.forward_backward(x, bad, lens, W, b)
    with pytest.raises(IndexError, match="out of range .* in layer 'output_prob'"):
        out.check_targets(bad)
