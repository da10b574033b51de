"""GPU numerics of the BF16 tcgen05 GEMM (K1 / K4) against a torch fp32
reference on the same bf16-rounded operands (tolerance: fp32 accumulation
order only, rel 1e-5)."""
import ctypes

import pytest
import torch

from paper_1805_05225_b200 import lstm

pytestmark = pytest.mark.gpu


def lib():
    L = lstm.lib()
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    L.sl_debug_gemm_bf16.argtypes = [ctypes.c_int] * 3 + [vp, i64, ctypes.c_int, vp, i64,
                                                          ctypes.c_int, vp, i64, ctypes.c_float,
                                                          ctypes.c_float, vp, vp]
    return L


def run(M, N, K, a_mn, b_mn, alpha=1.0, beta=0.0, bias=False, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = (torch.rand((K, M) if a_mn else (M, K), device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand((K, N) if b_mn else (N, K), device="cuda", generator=g) * 2 - 1).bfloat16()
    C = torch.rand(M, N, device="cuda", generator=g)
    bvec = torch.rand(N, device="cuda", generator=g) if bias else None
    opA = A.float().t() if a_mn else A.float()
    opB = B.float() if b_mn else B.float().t()
    ref = alpha * (opA @ opB) + beta * C
    if bias:
        ref = ref + bvec
    rc = lib().sl_debug_gemm_bf16(M, N, K, A.data_ptr(), A.shape[1], int(a_mn), B.data_ptr(),
                                  B.shape[1], int(b_mn), C.data_ptr(), N, alpha, beta,
                                  bvec.data_ptr() if bias else None,
                                  torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib().sl_last_error()
    torch.cuda.synchronize()
    return C, ref


@pytest.mark.parametrize("a_mn,b_mn", [(False, True), (False, False), (True, True), (True, False)])
@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 320), (200, 304, 136),
                                   (1000, 4000, 1024)])
def test_gemm_bf16_tc(cuda, a_mn, b_mn, shape):
    M, N, K = shape
    C, ref = run(M, N, K, a_mn, b_mn)
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


def test_gemm_bf16_tc_epilogue(cuda):
    C, ref = run(384, 520, 200, False, True, alpha=0.5, beta=1.0, bias=True)
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


def test_gemm_bf16_tc_bf16_output(cuda):
    # K1 writes XW as bf16: same GEMM, rounded output
    import ctypes as C
    M, N, K = 300, 520, 136
    g = torch.Generator(device="cuda").manual_seed(3)
    A = (torch.rand((M, K), device="cuda", generator=g) * 2 - 1).bfloat16()
    B = (torch.rand((K, N), device="cuda", generator=g) * 2 - 1).bfloat16()
    bias = torch.rand(N, device="cuda", generator=g)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    L = lib()
    L.sl_debug_gemm_bf16_out.argtypes = [C.c_int] * 3 + [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                                         C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    rc = L.sl_debug_gemm_bf16_out(M, N, K, A.data_ptr(), K, B.data_ptr(), N, out.data_ptr(), N,
                                  bias.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    ref = (A.float() @ B.float() + bias).bfloat16().float()
    assert (out.float() - ref).abs().max().item() <= 2 ** -7 * ref.abs().max().item()


@pytest.mark.parametrize("M,N,K,b_kn", [(256, 1000, 1000, True), (256, 1000, 1000, False), (37, 72, 104, True),
                                        (37, 77, 104, False), (1, 8, 8, True), (300, 130, 56, False)])
def test_small_gemm_matches_torch(cuda, M, N, K, b_kn):
    """The mma.sync small-M GEMM (decoder per-step projections) against an fp32 matmul
    of the same bf16 operands."""
    import ctypes
    from paper_1805_05225_b200 import lstm
    L = lstm.lib()
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    L.sl_debug_small_gemm.argtypes = [ctypes.c_int] * 3 + [vp, i64, vp, i64, ctypes.c_int, vp, i64, vp, vp]
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    pad = lambda n: (n + 7) // 8 * 8 + 8
    A = (torch.rand(M, pad(K), device="cuda", generator=g) * 2 - 1).bfloat16()
    B = ((torch.rand(K, pad(N), device="cuda", generator=g) if b_kn else
          torch.rand(N, pad(K), device="cuda", generator=g)) * 2 - 1).bfloat16()
    bias = torch.rand(N, device="cuda", generator=g)
    C = torch.full((M, N + 3), float("nan"), device="cuda")
    assert L.sl_debug_small_gemm(M, N, K, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], int(b_kn),
                                 C.data_ptr(), C.shape[1], bias.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream) == 0
    opB = B[:, :N].float() if b_kn else B[:, :K].float().t()
    ref = A[:, :K].float() @ opB + bias
    torch.cuda.synchronize()
    assert torch.allclose(C[:, :N], ref, rtol=1e-4, atol=1e-4 * K ** 0.5)
    assert torch.isnan(C[:, N:]).all()  # nothing written past N
