"""tcgen05 GEMM vs a plain PyTorch fp32 reference of the same op.

Operands are bf16 (exactly representable in fp32), accumulation fp32 in TMEM,
so the only differences are summation order: |err| <= 1e-5 * sum|a||b| + 1e-6.
Covers K-major / MN-major operands, ragged M (variable per-rank batch), N and K
tails, and every fused epilogue the MLP uses."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

EPI_F32, EPI_F32_ACC, EPI_BIAS_RELU_BF16, EPI_BIAS_F32, EPI_BF16, EPI_RELU_GRAD = 0, 1, 2, 3, 4, 5


def run_gemm(torch, A, a_mn, B, b_mn, M, N, K, epi=EPI_F32, bias=None, aux=None, ldd=None, out=None):
    from paper_2007_11831_b200 import _lib

    ldd = ldd or N
    if out is None:
        dt = torch.float32 if epi in (EPI_F32, EPI_F32_ACC, EPI_BIAS_F32) else torch.bfloat16
        out = torch.zeros(M, ldd, dtype=dt, device=A.device)
    st = _lib.lib().dbs_dev_gemm_bf16(A.data_ptr(), a_mn, A.shape[1], B.data_ptr(), b_mn, B.shape[1], out.data_ptr(),
                                      ldd, M, N, K, epi, bias.data_ptr() if bias is not None else None,
                                      aux.data_ptr() if aux is not None else None, _lib.stream_handle())
    assert st == 0, _lib.last_error()
    torch.cuda.synchronize()
    return out


def operands(torch, dev, M, N, K, a_mn, b_mn, pad=0):
    g = torch.Generator(device=dev).manual_seed(M * 7 + N * 3 + K)
    a = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    b = torch.randn(N, K, device=dev, generator=g).to(torch.bfloat16)
    # stored layouts (with optional padded leading dimension)
    A = a.t().contiguous() if a_mn else a
    B = b.t().contiguous() if b_mn else b
    # TMA needs 16-byte row pitch: pad the contiguous dim to a multiple of 8 (+ optional extra)
    A = torch.nn.functional.pad(A, (0, (-A.shape[1]) % 8 + pad))
    B = torch.nn.functional.pad(B, (0, (-B.shape[1]) % 8 + pad))
    return a, b, A, B


def check(torch, got, want, a, b):
    tol = 1e-5 * (a.float().abs() @ b.float().abs().t()) + 1e-5
    err = (got.float() - want).abs()
    assert bool((err <= tol).all()), float((err - tol).max())


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (37, 200, 784), (300, 784, 128), (129, 64, 1000),
                                   (512, 512, 512), (1, 128, 16)])
def test_gemm_shapes(dev, a_mn, b_mn, M, N, K):
    import torch

    a, b, A, B = operands(torch, dev, M, N, K, a_mn, b_mn, pad=8 if (M + N + K) % 2 else 0)
    got = run_gemm(torch, A, a_mn, B, b_mn, M, N, K)
    check(torch, got, a.float() @ b.float().t(), a, b)


def test_gemm_small_n_kmajor(dev):
    import torch

    a, b, A, B = operands(torch, dev, 200, 10, 256, 0, 0)
    got = run_gemm(torch, A, 0, B, 0, 200, 10, 256, ldd=16)
    check(torch, got[:, :10], a.float() @ b.float().t(), a, b)


def test_gemm_epilogues(dev):
    import torch

    M, N, K = 77, 256, 784
    a, b, A, B = operands(torch, dev, M, N, K, 0, 0)
    ref = a.float() @ b.float().t()
    bias = torch.randn(N, device=dev)
    got = run_gemm(torch, A, 0, B, 0, M, N, K, EPI_BIAS_F32, bias=bias)
    check(torch, got, ref + bias, a, b)
    got = run_gemm(torch, A, 0, B, 0, M, N, K, EPI_BIAS_RELU_BF16, bias=bias)
    want = torch.relu(ref + bias)
    assert torch.allclose(got.float(), want, rtol=1e-2, atol=1e-2)
    got = run_gemm(torch, A, 0, B, 0, M, N, K, EPI_BF16)
    assert torch.allclose(got.float(), ref, rtol=1e-2, atol=1e-2)
    aux = torch.randn(M, N, device=dev).to(torch.bfloat16)
    got = run_gemm(torch, A, 0, B, 0, M, N, K, EPI_RELU_GRAD, aux=aux)
    assert torch.allclose(got.float(), ref * (aux.float() > 0), rtol=1e-2, atol=1e-2)
    base = torch.randn(M, N, device=dev)
    out = base.clone()
    run_gemm(torch, A, 0, B, 0, M, N, K, EPI_F32_ACC, out=out)
    check(torch, out, base + ref, a, b)


def test_gemm_variable_batch_no_recompile(dev):
    """Every per-rank batch size the DBS controller may emit runs on the same kernel."""
    import torch

    for M in (37, 58, 73, 128, 129, 137, 255, 512):
        a, b, A, B = operands(torch, dev, M, 256, 784, 0, 0)
        got = run_gemm(torch, A, 0, B, 0, M, 256, 784)
        check(torch, got, a.float() @ b.float().t(), a, b)
