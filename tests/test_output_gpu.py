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


@pytest.mark.parametrize("B,T,D,V,eps", [(8, 5, 64, 300, 0.1), (20, 13, 200, 1003, 0.0), (16, 30, 1000, 4096, 0.1),
                                         (256, 60, 1000, 20000, 0.1)])
def test_output_ce_fp32_matches_reference_restatement(cuda, B, T, D, V, eps):
    """precision fp32 (sl_output_ce_f32): fp32 logits, split-bf16 tcgen05 GEMMs —
    per tensor within 1e-4 of the fp64 restatement on the UNROUNDED operands, up
    to the config-4 output layer (B*T = 15360 rows, V = 20000)."""
    g = torch.Generator().manual_seed(B * 131 + V)
    x = torch.rand(B, T, D, generator=g, dtype=torch.float64) * 2 - 1
    W = (torch.rand(D, V, generator=g, dtype=torch.float64) * 2 - 1) * D ** -0.5 * 3
    b = (torch.rand(V, generator=g, dtype=torch.float64) * 2 - 1) * 0.5
    lens = torch.randint(T // 2, T + 1, (B,), generator=g, dtype=torch.int32)
    lens[0] = T
    tg = torch.randint(0, V, (B, T), generator=g, dtype=torch.int32)
    xf, Wf = x.float(), W.float()
    if B * T * V <= 20_000_000:
        loss, dx, dW, db = oracle.output_ce_np(xf.double().numpy(), lens.numpy(), tg.numpy(), Wf.double().numpy(),
                                               b.float().double().numpy(), eps)
    else:  # the same restatement in fp64 torch on the device (numpy would take minutes)
        loss, dx, dW, db = _output_ce_torch64(xf.double().cuda(), lens.cuda(), tg.cuda(), Wf.double().cuda(),
                                              b.float().double().cuda(), eps)
    out = OutputCE(B, T, D, V, eps, precision="fp32")
    l, gdx, gdW, gdb = out.forward_backward(xf.cuda(), tg.cuda(), lens.cuda(), Wf.cuda(), b.float().cuda())
    torch.cuda.synchronize()
    out.check_targets()
    assert abs(float(l) - float(loss)) < 1e-5 * max(1.0, abs(float(loss)))
    assert rel(gdx, dx) < 1e-4, rel(gdx, dx)
    assert rel(gdW, dW) < 1e-4, rel(gdW, dW)
    assert rel(gdb, db) < 1e-4, rel(gdb, db)


def _output_ce_torch64(x, lens, tg, W, b, eps):
    """oracle.output_ce_np (pinned to the reference's Softmax + ce_label_smoothing)
    restated in fp64 torch for the config-4 size."""
    B, T, D = x.shape
    V = W.shape[1]
    z = x.reshape(-1, D) @ W + b
    lse = torch.logsumexp(z, 1, keepdim=True)
    lp = z - lse
    valid = (torch.arange(T, device=x.device)[None, :] < lens[:, None].long()).reshape(-1)
    y = tg.reshape(-1).long()
    rowloss = -(1 - eps) * lp.gather(1, y[:, None])[:, 0] - eps / V * lp.sum(1)
    n = valid.sum()
    loss = (rowloss * valid).sum() / n
    dz = torch.softmax(z, 1) - eps / V
    dz[torch.arange(z.shape[0], device=x.device), y] -= 1 - eps
    dz = dz * valid[:, None] / n
    return loss.cpu(), (dz @ W.T).reshape(B, T, D).cpu(), (x.reshape(-1, D).T @ dz).cpu(), dz.sum(0).cpu()
