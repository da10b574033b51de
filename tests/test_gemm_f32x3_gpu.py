"""The fp32-class split-bf16 GEMM (gemm_f32x3.cu on the pair GEMM's x3 mode):
C = op(A) op(B) (+ bias, + beta C) against an fp64 torch product, over the
operand layouts (A / A^T, B / B^T), K tails, tiny and tile-starved outputs
(split-K), and long K (chunked accumulation).  Bound: max |C - ref| / max |ref|
< 3e-5 — fp32-class (the reference computes these products in fp32)."""
import ctypes

import pytest
import torch

from paper_1805_05225_b200 import lstm

pytestmark = pytest.mark.gpu
vp, i64 = ctypes.c_void_p, ctypes.c_int64


def lib():
    L = lstm.lib()
    L.sl_debug_gemm_f32x3_ws.restype = ctypes.c_size_t
    L.sl_debug_gemm_f32x3_ws.argtypes = [ctypes.c_int] * 5
    L.sl_debug_gemm_f32x3.argtypes = [ctypes.c_int] * 5 + [vp, i64, vp, i64, ctypes.c_float, vp, i64, vp, vp, vp]
    return L


@pytest.mark.parametrize("tA,tB", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(37, 72, 104), (1, 64, 64), (256, 1000, 1000), (256, 4000, 3000),
                                   (1024, 520, 5000), (300, 300, 20000)])
def test_gemm_f32x3_matches_fp64(cuda, tA, tB, M, N, K):
    L = lib()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K + 2 * tA + tB)
    A = torch.rand((K, M) if tA else (M, K), device="cuda", generator=g) * 2 - 1
    B = torch.rand((N, K) if tB else (K, N), device="cuda", generator=g) * 2 - 1
    bias = torch.rand(N, device="cuda", generator=g) * 2 - 1
    C0 = torch.rand(M, N, device="cuda", generator=g) * 2 - 1
    ref = (A.double().T if tA else A.double()) @ (B.double().T if tB else B.double())
    ws = torch.empty(L.sl_debug_gemm_f32x3_ws(tA, tB, M, N, K), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    # plain product
    C = torch.full((M, N), float("nan"), device="cuda")
    assert L.sl_debug_gemm_f32x3(tA, tB, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), 0.0,
                                 C.data_ptr(), N, None, ws.data_ptr(), st) == 0
    torch.cuda.synchronize()
    err = float((C.double() - ref).abs().max() / ref.abs().max())
    assert err < 3e-5, err
    # with bias and beta (C = op(A) op(B) + bias + 0.5 C0)
    C = C0.clone()
    assert L.sl_debug_gemm_f32x3(tA, tB, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), 0.5,
                                 C.data_ptr(), N, bias.data_ptr(), ws.data_ptr(), st) == 0
    torch.cuda.synchronize()
    ref2 = ref + bias.double() + 0.5 * C0.double()
    err = float((C.double() - ref2).abs().max() / ref2.abs().max())
    assert err < 3e-5, err
    # with bias, beta = 0 (the coalesced epilogue's bias path)
    C = torch.full((M, N), float("nan"), device="cuda")
    assert L.sl_debug_gemm_f32x3(tA, tB, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), 0.0,
                                 C.data_ptr(), N, bias.data_ptr(), ws.data_ptr(), st) == 0
    torch.cuda.synchronize()
    ref3 = ref + bias.double()
    err = float((C.double() - ref3).abs().max() / ref3.abs().max())
    assert err < 3e-5, err
