"""Optimizer step: the oracle pinned to the SPEC's worked
examples (CPU), then the fused CUDA kernel against the oracle (GPU)."""
import numpy as np
import pytest

from oracle import adam_ref


def test_oracle_spec_examples():
    # g = 0 everywhere, fresh state -> params unchanged
    p = np.linspace(-1, 1, 7)
    p1, m, v, n = adam_ref.adam_step(p, np.zeros(7), np.zeros(7), np.zeros(7), 1)
    assert np.array_equal(p1, p) and n == 0.0
    # fresh state, g = 1, theta = 0, lr = 1e-3 -> theta_1 ~ -1e-3 (|err| < 1e-8 lr)
    p1, m, v, _ = adam_ref.adam_step(np.zeros(1), np.ones(1), np.zeros(1), np.zeros(1), 1, lr=1e-3,
                                     clip_norm=0)
    assert abs(p1[0] + 1e-3) < 1e-8 * 1e-3
    # two identical calls != one call with doubled lr (moments carry state)
    g = np.array([0.3, -2.0, 0.7])
    a, ma, va, _ = adam_ref.adam_step(np.zeros(3), g, np.zeros(3), np.zeros(3), 1)
    a, ma, va, _ = adam_ref.adam_step(a, g, ma, va, 2)
    b, mb, _, _ = adam_ref.adam_step(np.zeros(3), g, np.zeros(3), np.zeros(3), 1, lr=2e-3)
    assert not np.array_equal(a, b) and not np.allclose(ma, mb)


def test_oracle_global_norm_clip():
    # the whole gradient is rescaled to norm 5 before Adam
    g = np.array([6.0, 8.0])  # norm 10
    _, m, _, n = adam_ref.adam_step(np.zeros(2), g, np.zeros(2), np.zeros(2), 1, clip_norm=5.0)
    assert n == pytest.approx(10.0)
    assert np.allclose(m, 0.1 * g * 0.5)
    _, m, _, _ = adam_ref.adam_step(np.zeros(2), g, np.zeros(2), np.zeros(2), 1, clip_norm=0)
    assert np.allclose(m, 0.1 * g)
    with pytest.raises(FloatingPointError):
        adam_ref.adam_step(np.zeros(2), np.array([1.0, np.nan]), np.zeros(2), np.zeros(2), 1)


@pytest.mark.gpu
@pytest.mark.parametrize("clip,scale", [(5.0, 1.0), (5.0, 0.25), (0.0, 1.0), (1e9, 0.5)])
def test_adam_kernel_matches_oracle(cuda, clip, scale):
    import torch
    from paper_1805_05225_b200.optim import Adam
    n = 1_000_003  # vector body + scalar tail
    g = torch.Generator(device="cuda").manual_seed(7)
    p = torch.rand(n, device="cuda", generator=g) * 2 - 1
    opt = Adam(p, lr=3e-3, clip_norm=clip)
    ref_p, ref_m, ref_v = (p.double().cpu().numpy(), np.zeros(n), np.zeros(n))
    for step in range(1, 4):
        grads = (torch.rand(n, device="cuda", generator=g) * 2 - 1) * 0.02 * step
        opt.step(grads, grad_scale=scale)
        # the hyperparameters as the kernel receives them (fp32): beta2 = 0.999f is
        # 1.3e-5 away from 0.999 in (1 - beta2), which would dominate the comparison
        f32 = lambda x: float(np.float32(x))
        ref_p, ref_m, ref_v, norm = adam_ref.adam_step(ref_p, grads.double().cpu().numpy(), ref_m, ref_v,
                                                       step, lr=f32(3e-3), beta1=f32(0.9), beta2=f32(0.999),
                                                       eps=f32(1e-8), grad_scale=scale, clip_norm=clip)
        torch.cuda.synchronize()
        opt.check_finite()
        assert opt.grad_norm.item() == pytest.approx(norm, rel=1e-5)
        for got, ref in ((opt.params, ref_p), (opt.m, ref_m), (opt.v, ref_v)):
            got = got.double().cpu().numpy()
            assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max() + 1e-12


@pytest.mark.gpu
def test_adam_kernel_spec_examples_and_nonfinite(cuda):
    import torch
    from paper_1805_05225_b200.optim import Adam
    p = torch.zeros(5, device="cuda")
    opt = Adam(p, lr=1e-3, clip_norm=0)
    opt.step(torch.zeros(5, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(p, torch.zeros(5, device="cuda"))  # g = 0: unchanged
    p = torch.zeros(5, device="cuda")
    opt = Adam(p, lr=1e-3, clip_norm=0)
    opt.step(torch.ones(5, device="cuda"))
    torch.cuda.synchronize()
    assert torch.allclose(p.double(), torch.full((5,), -1e-3, dtype=torch.float64, device="cuda"),
                          rtol=1e-6, atol=0)  # SPEC.md:436 (fp32 storage)
    # non-finite gradient: the step is skipped and the error names the parameter
    p = torch.ones(12, device="cuda")
    opt = Adam(p, names=[("enc0_fw/W", 0, 4), ("enc0_fw/R", 4, 4), ("enc0_fw/b", 8, 4)])
    bad = torch.zeros(12, device="cuda")
    bad[6] = float("inf")
    opt.step(bad)
    with pytest.raises(FloatingPointError, match="enc0_fw/R"):
        opt.check_finite(bad)
    assert torch.equal(p, torch.ones(12, device="cuda"))
