"""k_rn_conv (csrc/resnet.cu) -- the tcgen05 implicit-GEMM convolution of
the ResNet-18 path -- against torch fp32 on the same bf16 operands, every
mode and geometry class the network uses (3x3 stride 1/2, 1x1 stride 2,
the 8-channel stem, partial batches, split-K wgrad)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # BS, cnt, Cinp, Cout, H, R, stride
    (4, 3, 8, 64, 32, 3, 1),
    (3, 3, 64, 64, 32, 3, 1),
    (4, 2, 64, 128, 32, 3, 2),
    (4, 4, 64, 128, 32, 1, 2),
    (5, 5, 128, 256, 8, 3, 1),
    (6, 5, 256, 512, 8, 3, 2),
    (7, 7, 512, 512, 4, 3, 1),
]


def _run(mode, BS, cnt, Cinp, Cout, H, R, stride, x, w, dz):
    import torch
    from paper_2303_01778_b200._lib import lib, ptr
    Ho = H // stride
    if mode == 0:
        out = torch.empty(cnt * Ho * Ho * Cout, device="cuda")
    elif mode == 1:
        out = torch.empty(cnt * H * H * Cinp, device="cuda")
    else:
        nsplit = -(-BS * Ho * Ho // 1024)
        out = torch.empty(nsplit * R * R * Cinp * Cout, device="cuda")
    lib.check(lib.pb_rn_conv_selftest(mode, BS, cnt, Cinp, Cout, H, R, stride, ptr(x), ptr(w), ptr(dz),
                                      ptr(out), torch.cuda.current_stream().cuda_stream))
    return out


@pytest.mark.parametrize("case", CASES, ids=[f"c{i}" for i in range(len(CASES))])
def test_rn_conv_modes_match_torch(case):
    import torch
    import torch.nn.functional as F
    BS, cnt, Cinp, Cout, H, R, stride = case
    Ho = H // stride
    pad = (R - 1) // 2
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(BS, H, H, Cinp, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(Cout, R, R, Cinp, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    dz = torch.randn(BS, Ho, Ho, Cout, device="cuda", generator=g).to(torch.bfloat16)
    xs, ws, dzs = (x[:cnt].float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2),
                   dz[:cnt].float().permute(0, 3, 1, 2))
    # forward
    z = _run(0, BS, cnt, Cinp, Cout, H, R, stride, x, w, dz).view(cnt, Ho, Ho, Cout)
    ref = F.conv2d(xs.double(), ws.double(), stride=stride, padding=pad).permute(0, 2, 3, 1)
    assert float((z.double() - ref).norm() / ref.norm()) < 1e-5
    # dgrad (the network never back-propagates into the 8-channel stem input)
    if Cinp < 16:
        return
    dx = _run(1, BS, cnt, Cinp, Cout, H, R, stride, x, w, dz).view(cnt, H, H, Cinp)
    ref = torch.nn.grad.conv2d_input((cnt, Cinp, H, H), ws.double(), dzs.double(), stride=stride,
                                     padding=pad).permute(0, 2, 3, 1)
    assert float((dx.double() - ref).norm() / ref.norm()) < 1e-5
    # wgrad (split partials summed here)
    parts = _run(2, BS, cnt, Cinp, Cout, H, R, stride, x, w, dz).view(-1, Cout, R * R * Cinp)
    dw = parts.double().sum(0).view(Cout, R, R, Cinp)
    ref = torch.nn.grad.conv2d_weight(xs.double(), (Cout, Cinp, R, R), dzs.double(), stride=stride,
                                      padding=pad).permute(0, 2, 3, 1)
    assert float((dw - ref).norm() / ref.norm()) < 1e-5
