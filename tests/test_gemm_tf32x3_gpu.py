"""fp32-class tensor-core GEMM (3xTF32 on kind::tf32 UMMA, S32 operands) vs an
fp64 PyTorch reference of the same op.

S32 keeps every operand to ~2^-23 relative (hi = rn_tf32(x), lo = rn_tf32(x -
hi)); the dropped lo*lo term is ~2^-24 per product; the tensor core truncates
each accumulation step into TMEM (~2^-24 of the running sum), which the kernel
spreads over 2 [main | correction] accumulator pairs summed in fp32.
Stated tolerances: elementwise |err| <= 2e-6 * sum_k |a||b|; normwise relative
error <= 1.5e-9 * K and >= 300x below a bf16-operand GEMM."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

EPI_F32, EPI_F32_ACC, EPI_BIAS_F32, EPI_F32_ATOMIC = 0, 1, 3, 6
EPI_S32, EPI_BIAS_RELU_S32, EPI_RELU_GRAD_S32 = 8, 9, 10
TOL = 2e-6


def ceil32(x):
    return (x + 31) // 32 * 32


def to_s32(torch, x, ld=None):
    """fp32 [rows][cols] -> S32 [rows][ld] through the library's split kernel."""
    from paper_2007_11831_b200 import _lib

    x = x.float().contiguous()
    rows, cols = x.shape
    ld = ld or ceil32(cols)
    out = torch.empty(rows, 2 * ld, device=x.device, dtype=torch.float32)
    _lib.check(_lib.lib().dbs_dev_split_s32(x.data_ptr(), rows, cols, cols, out.data_ptr(), ld,
                                            _lib.stream_handle()), "split")
    return out, ld


def from_s32(torch, s, rows, cols, ld):
    from paper_2007_11831_b200 import _lib

    out = torch.empty(rows, cols, device=s.device, dtype=torch.float32)
    _lib.check(_lib.lib().dbs_dev_join_s32(s.data_ptr(), rows, cols, ld, out.data_ptr(), cols,
                                           _lib.stream_handle()), "join")
    torch.cuda.synchronize()
    return out


def run(torch, A, a_mn, lda, B, b_mn, ldb, M, N, K, epi=EPI_F32, bias=None, aux=None, out=None, ldd=None):
    from paper_2007_11831_b200 import _lib

    s32 = epi in (EPI_S32, EPI_BIAS_RELU_S32, EPI_RELU_GRAD_S32)
    ldd = ldd or (ceil32(N) if s32 else N)
    if out is None:
        out = torch.zeros(M, 2 * ldd if s32 else ldd, dtype=torch.float32, device=A.device)
    st = _lib.lib().dbs_dev_gemm_tf32x3(A.data_ptr(), a_mn, lda, B.data_ptr(), b_mn, ldb, out.data_ptr(), ldd, M, N,
                                        K, epi, bias.data_ptr() if bias is not None else None,
                                        aux.data_ptr() if aux is not None else None, _lib.stream_handle())
    assert st == 0, _lib.last_error()
    torch.cuda.synchronize()
    return (from_s32(torch, out, M, N, ldd) if s32 else out[:, :N]), out


def operands(torch, dev, M, N, K, a_mn, b_mn):
    g = torch.Generator(device=dev).manual_seed(M * 7 + N * 3 + K)
    a = torch.randn(M, K, device=dev, generator=g, dtype=torch.float64)
    b = torch.randn(N, K, device=dev, generator=g, dtype=torch.float64)
    a32, b32 = a.float(), b.float()
    A, lda = to_s32(torch, a32.t().contiguous() if a_mn else a32)
    B, ldb = to_s32(torch, b32.t().contiguous() if b_mn else b32)
    # the exact product of the fp32 operands, in fp64
    return a32.double(), b32.double(), A, lda, B, ldb


def check(got, want, a, b, tol=TOL):
    bound = tol * (a.abs() @ b.abs().t()) + 1e-30
    err = (got.double() - want).abs()
    worst = float((err / bound).max())
    assert worst <= 1.0, worst


def test_split_join_roundtrip(dev):
    import torch

    x = torch.randn(37, 100, device=dev) * torch.logspace(-20, 20, 100, device=dev)
    s, ld = to_s32(torch, x)
    assert ld == 128 and s.shape == (37, 256)
    hi = s.view(37, 4, 2, 32)[:, :, 0, :]
    assert bool(((hi.view(torch.int32) & 0x1FFF) == 0).all())  # hi is an exact tf32 value
    back = from_s32(torch, s, 37, 100, ld)
    rel = ((back.double() - x.double()).abs() / x.double().abs()).max()
    assert float(rel) <= 2.0 ** -22
    pad = s.view(37, 4, 2, 32)[:, 3, :, 4:]  # logical columns 100..127 are zero
    assert bool((pad == 0).all())


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (37, 200, 784), (300, 64, 128), (129, 64, 1000),
                                   (512, 512, 512), (1, 128, 32), (200, 10, 256)])
def test_tf32x3_shapes(dev, a_mn, b_mn, M, N, K):
    import torch

    a, b, A, lda, B, ldb = operands(torch, dev, M, N, K, a_mn, b_mn)
    got, _ = run(torch, A, a_mn, lda, B, b_mn, ldb, M, N, K)
    check(got, a @ b.t(), a, b)


def test_tf32x3_beats_bf16_and_tf32(dev):
    """The point of the format: error far below a single bf16 or tf32 pass."""
    import torch

    import itertools

    bad = []
    for (M, N, K), (a_mn, b_mn) in itertools.product([(256, 256, 1024), (256, 64, 1024), (300, 128, 4608)],
                                                      [(0, 0), (1, 1)]):
        err, err_f32, err_bf16 = _accuracy_case(torch, dev, M, N, K, a_mn, b_mn)
        # stated bound: the tensor core truncates each in-TMEM accumulation step, so the
        # normwise error grows ~linearly in the steps one main accumulator takes: K / 8
        # with one main (N > 64 tiles double-buffered while 4 ceil(K / 32) <= 288, i.e.
        # K <= 2304), else K / 16 (2 [main | correction] pairs round-robin); <= 2.5e-8 per
        # step, i.e. <= 7.2e-6 at most (measured 1.2e-6 at K = 1024 with two mains, 2.4e-6
        # with one, 5.5e-6 at 4608; cuBLAS fp32 2.7e-7..5.7e-7), >= 300x below bf16 operands
        steps = K // 8 if (N > 64 and 4 * ((K + 31) // 32) <= 288) else K // 16
        if not (err < 2.5e-8 * steps and err < err_bf16 / 300):
            bad.append((M, N, K, a_mn, b_mn, err, err_f32))
    assert not bad, bad


def _accuracy_case(torch, dev, M, N, K, a_mn, b_mn):
    a, b, A, lda, B, ldb = operands(torch, dev, M, N, K, a_mn, b_mn)
    got, _ = run(torch, A, a_mn, lda, B, b_mn, ldb, M, N, K)
    want = a @ b.t()
    err = float((got.double() - want).norm() / want.norm())
    torch.backends.cuda.matmul.allow_tf32 = False
    f32 = (a.float() @ b.float().t()).double()
    err_f32 = float((f32 - want).norm() / want.norm())
    bf = (a.bfloat16().float() @ b.bfloat16().float().t()).double()
    err_bf16 = float((bf - want).norm() / want.norm())
    print(f"{M}x{N}x{K} normwise rel error: 3xTF32 {err:.3g}, cuBLAS fp32 {err_f32:.3g}, bf16 operands {err_bf16:.3g}")
    return err, err_f32, err_bf16


def test_tf32x3_epilogues(dev):
    import torch

    M, N, K = 77, 256, 784
    a, b, A, lda, B, ldb = operands(torch, dev, M, N, K, 0, 0)
    ref = a @ b.t()
    bias = torch.randn(N, device=dev)
    got, _ = run(torch, A, 0, lda, B, 0, ldb, M, N, K, EPI_BIAS_F32, bias=bias)
    check(got, ref + bias.double(), a, b)
    got, s32 = run(torch, A, 0, lda, B, 0, ldb, M, N, K, EPI_BIAS_RELU_S32, bias=bias)
    check(got, torch.relu(ref + bias.double()), a, b)
    # ReLU-backward with the S32 activation as the mask
    got2, _ = run(torch, A, 0, lda, B, 0, ldb, M, N, K, EPI_RELU_GRAD_S32, aux=s32)
    mask = (torch.relu(ref + bias.double()) > 0)
    check(got2, ref * mask, a, b)
    # accumulate and split-K-style atomics
    out = torch.ones(M, N, device=dev)
    got3, _ = run(torch, A, 0, lda, B, 0, ldb, M, N, K, EPI_F32_ACC, out=out)
    check(got3, ref + 1.0, a, b)


def test_tf32x3_ragged_s32_output_zero_pads(dev):
    """An S32 output with N % 32 != 0 zero-fills its pad columns (a later K-major
    operand reads them as K padding)."""
    import torch

    M, N, K = 50, 10, 96
    a, b, A, lda, B, ldb = operands(torch, dev, M, N, K, 0, 0)
    out = torch.full((M, 64), float("nan"), device=dev)
    got, s32 = run(torch, A, 0, lda, B, 0, ldb, M, N, K, EPI_S32, out=out, ldd=32)
    check(got, a @ b.t(), a, b)
    blk = s32.view(M, 2, 32)
    assert bool((blk[:, :, N:] == 0).all())
