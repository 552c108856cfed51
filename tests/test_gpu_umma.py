"""Pin the tcgen05 operand-layout conventions (SWIZZLE_NONE canonical layouts,
K-major, MN-major and 16-byte-shifted "plane" operands; M=64 accumulator lane
mapping) that the CNN kernels are built on."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(M, n, k, a_mode, b_mode, shift):
    import torch
    from paper_2303_01778_b200._lib import lib
    g = torch.Generator().manual_seed(M * n * k + a_mode * 3 + b_mode + shift)
    A = torch.randn(M, k, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(n, k, generator=g).to(torch.bfloat16).cuda()
    want = (A.float() @ B.float().t()).cpu().numpy()
    D = torch.zeros(128, n, device="cuda")
    lib.check(lib.pb_umma_selftest(A.data_ptr(), B.data_ptr(), D.data_ptr(), M, n, k, a_mode,
                                   b_mode, shift, torch.cuda.current_stream().cuda_stream))
    return D.cpu().numpy(), want


@pytest.mark.parametrize("n,k", [(64, 128), (16, 32), (32, 512)])
@pytest.mark.parametrize("a_mode,b_mode", [(0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (2, 1), (2, 2)])
@pytest.mark.parametrize("shift", [0, 5])
def test_umma_m128_layouts(n, k, a_mode, b_mode, shift):
    got, want = _run(128, n, k, a_mode, b_mode, shift)
    assert np.allclose(got, want, rtol=1e-3, atol=1e-2), np.abs(got - want).max()


def test_umma_m64_accumulator_lanes():
    got, want = _run(64, 32, 64, 1, 1, 0)
    lanes = [(r // 16) * 32 + r % 16 for r in range(64)]
    assert np.allclose(got[lanes], want, rtol=1e-3, atol=1e-2)


def _tf32_trunc(x):
    import numpy as np
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def _tf32_rne(x):
    import numpy as np
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0)])
def test_umma_tf32_layouts_and_rounding(a_mn, b_mn):
    """kind::tf32 from fp32 smem operands, K-major (the fc1 kernels' path);
    records whether the hardware truncates or rounds fp32 -> tf32.  (MN-major
    tf32 staging does not follow the bf16 convention; the kernels stage
    transposed K-major tiles instead.)"""
    import torch
    from paper_2303_01778_b200._lib import lib
    g = torch.Generator().manual_seed(7)
    A = torch.randn(128, 64, generator=g).cuda()
    B = torch.randn(32, 64, generator=g).cuda()
    D = torch.zeros(128, 32, device="cuda")
    lib.check(lib.pb_umma_tf32_selftest(A.data_ptr(), B.data_ptr(), D.data_ptr(), 32, 64, a_mn,
                                        b_mn, torch.cuda.current_stream().cuda_stream))
    got = D.cpu().numpy().astype(np.float64)
    a, b = A.cpu().numpy(), B.cpu().numpy()
    exact = a.astype(np.float64) @ b.astype(np.float64).T
    trunc = _tf32_trunc(a).astype(np.float64) @ _tf32_trunc(b).astype(np.float64).T
    rne = _tf32_rne(a).astype(np.float64) @ _tf32_rne(b).astype(np.float64).T
    errs = {k: float(np.abs(got - v).max()) for k, v in
            (("exact", exact), ("trunc", trunc), ("rne", rne))}
    print("tf32 error vs", errs)
    assert min(errs.values()) < 5e-4, errs


@pytest.mark.parametrize("N,K", [(32, 64), (128, 256), (256, 96)])
def test_tma_sw128_tf32_gemm(N, K):
    """TMA-loaded SWIZZLE_128B K-major tf32 tiles (tma.cuh) through tcgen05:
    D = A B^T against torch on the same tf32-truncated operands."""
    import torch
    from paper_2303_01778_b200._lib import lib, ptr
    g = torch.Generator(device="cuda").manual_seed(N + K)
    A = torch.randn(128, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    D = torch.empty(128, N, device="cuda")
    lib.check(lib.pb_tma_tf32_selftest(ptr(A), ptr(B), ptr(D), N, K, torch.cuda.current_stream().cuda_stream))
    trunc = lambda x: (x.view(torch.int32) & -8192).view(torch.float32).double()  # noqa: E731
    ref = trunc(A) @ trunc(B).t()
    assert float((D.double() - ref).norm() / ref.norm()) < 1e-6


@pytest.mark.parametrize("N", [64, 128, 256])
def test_tma_mn_sw128_bf16_gemm(N):
    """MN-major SWIZZLE_128B bf16 tiles loaded by TMA (the ResNet weight
    gradient's operands): LBO = stride between 64-element MN atoms, SBO =
    1024 B (8 K rows) -- measured by tools/tma_mn_probe.py."""
    import torch
    from paper_2303_01778_b200._lib import lib, ptr
    K = 128
    g = torch.Generator(device="cuda").manual_seed(N)
    A = torch.randn(K, 128, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    D = torch.zeros(128, N, device="cuda")
    lib.check(lib.pb_tma_bf16_mn_selftest(ptr(A), ptr(B), ptr(D), N, K, 64 * 128, 1024,
                                          torch.cuda.current_stream().cuda_stream))
    ref = A.double().t() @ B.double()
    assert float((D.double() - ref).norm() / ref.norm()) < 1e-6
