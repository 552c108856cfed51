"""MMA issue cost of the conv kernels' operand patterns (pb_umma_bench2):
cycles per MMA on resident smem operands, 1 CTA/SM, grid 148."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2303_01778_b200._lib import lib

cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
ITERS = 200
cases = [
    # name, M, N, a_mn, b_mn, a_lbo, a_sbo, b_lbo, b_sbo, kstep, ngroups, a_goff
    ("wgrad new  M128 N64 MN/MN sbo2704/2064", 128, 64, 1, 1, 128, 2704, 128, 2064, 256, 5, 16 * 18),
    ("wgrad new  same, groups at +64 B", 128, 64, 1, 1, 128, 2704, 128, 2064, 256, 5, 64),
    ("MN/MN sbo 128 (contig cores)", 128, 64, 1, 1, 16 * 128, 128, 8 * 128, 128, 2 * 16 * 128, 5, 0),
    ("MN/MN sbo2688/2048 (0 mod 128)", 128, 64, 1, 1, 128, 2688, 128, 2048, 256, 5, 16 * 18),
    ("wgrad old  M64 N64 MN/MN sbo5392", 64, 64, 1, 1, 128, 5392, 128, 5392, 256, 5, 16 * 18),
    ("fwd  M128 N64 K/K plane", 128, 64, 0, 0, 5392, 128, 1024, 128, 32, 5, 16),
    ("K/K contiguous M128 N64", 128, 64, 0, 0, 128, 1024, 128, 1024, 256, 5, 0),
    ("K/K contiguous M128 N128", 128, 128, 0, 0, 128, 1024, 128, 1024, 256, 4, 0),
    ("K/K contiguous M128 N256", 128, 256, 0, 0, 128, 1024, 128, 1024, 256, 2, 0),
    ("dgrad M128 N32 K/MN", 128, 32, 0, 1, 5392, 128, 128, 1024, 32, 5, 16),
    ("dgrad new N128 K/MN (kstep A 2 planes, B 256)", 128, 128, 0, 1, 5392, 128, 128, 1024, 10784, 4, 16 * 18, 256),
    ("dgrad new N32  K/MN", 128, 32, 0, 1, 5392, 128, 128, 1024, 10784, 4, 16 * 18, 256),
    ("N128 K/K A plane-strided, B contiguous", 128, 128, 0, 0, 5392, 128, 128, 1024, 10784, 4, 16 * 18, 256),
    ("N128 K/MN A contiguous", 128, 128, 0, 1, 128, 1024, 128, 1024, 256, 4, 0, 256),
    ("N128 MN/MN", 128, 128, 1, 1, 128, 1024, 128, 1024, 256, 4, 0, 256),
    ("N256 K/MN A plane-strided", 128, 256, 0, 1, 5392, 128, 128, 1024, 10784, 2, 16 * 18, 256),
]
for case in cases:
    name, M, N, amn, bmn, al, asb, bl, bsb, ks, ng, goff = case[:12]
    bks = case[12] if len(case) > 12 else 0
    lib.check(lib.pb_umma_bench2(M, N, amn, bmn, al, asb, bl, bsb, ks, ng, goff, ITERS, 148, cyc.data_ptr(), bks, 0))
    torch.cuda.synchronize()
    n = ITERS * ng * 8
    c = cyc.double().max().item() / n
    print(f"{name:40s}: {c:6.1f} cyc/MMA  {2 * M * N * 16 / c:6.0f} flop/cyc/SM", flush=True)

# TMEM -> registers: bytes per cycle per SM
sink = torch.zeros(148 * 512, device="cuda")
for warps in (4, 8, 16):
    for cols in (128, 512):
        c1 = torch.zeros(1, dtype=torch.int64, device="cuda")
        lib.check(lib.pb_tmem_ld_bench(warps, cols, 100, c1.data_ptr(), sink.data_ptr(), 0))
        torch.cuda.synchronize()
        byts = 100 * cols * 128 * 4
        print(f"tmem ld: {warps:2d} warps, {cols} cols x 128 lanes x100: {c1.item():8d} cyc -> {byts / c1.item():6.1f} B/cyc/SM",
              flush=True)
