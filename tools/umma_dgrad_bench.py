"""tcgen05 cost of the k_bwd_conv dgrad MMA shapes on resident smem operands
(pb_umma_bench2): cycles per MMA, first issue to completion, 8 K steps per
accumulator.  A: the dz2 planes (K-major, no swizzle, K cores one plane =
5392 B apart); B: the conv2 weights (MN-major, N cores 1024 B apart)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2303_01778_b200._lib import lib  # noqa: E402

KP = 337 * 16
cases = [
    # name, M, N, a_mn, b_mn, a_lbo, a_sbo, b_lbo, b_sbo, kstep(A), b_kstep
    ("dgrad N=128", 128, 128, 0, 1, KP, 128, 128, 1024, 2 * KP, 256),
    ("dgrad N=32", 128, 32, 0, 1, KP, 128, 128, 1024, 2 * KP, 256),
    ("dgrad N=64", 128, 64, 0, 1, KP, 128, 128, 1024, 2 * KP, 256),
    ("dgrad N=256", 128, 256, 0, 1, KP, 128, 128, 1024, 2 * KP, 256),
    ("packed K-major N=128", 128, 128, 0, 0, 128, 256, 128, 256, 256, 256),
    ("packed K-major N=32", 128, 32, 0, 0, 128, 256, 128, 256, 256, 256),
    ("A packed, B MN N=128", 128, 128, 0, 1, 128, 256, 128, 1024, 256, 256),
    ("A planes, B K N=128", 128, 128, 0, 0, KP, 128, 128, 256, 2 * KP, 256),
]
iters = 400
for grid in (1, 148):
    for name, M, N, amn, bmn, albo, asbo, blbo, bsbo, ks, bks in cases:
        cyc = torch.zeros(grid, dtype=torch.int64, device="cuda")
        lib.check(lib.pb_umma_bench2(M, N, amn, bmn, albo, asbo, blbo, bsbo, ks, 1, 0, iters, grid, cyc.data_ptr(),
                                     bks, 0))
        torch.cuda.synchronize()
        c = cyc.double().max().item() / (iters * 8)
        print(f"grid={grid:3d} {name:24s}: {c:6.1f} cyc/MMA  {2 * M * N * 16 / c:7.0f} flop/cyc", flush=True)
