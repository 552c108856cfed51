import sys
sys.path.insert(0, ".")
import torch
from paper_2303_01778_b200._lib import lib
KP = 337 * 16
iters = 400
for N in (128, 160):
    for goff in (1024, 16, 32, 64, 96):
        cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
        lib.check(lib.pb_umma_bench2(128, N, 0, 1, KP, 128, 128, 1024, 2 * KP, 2, goff, iters, 1, cyc.data_ptr(), 256, 0))
        torch.cuda.synchronize()
        c = cyc.double().max().item() / (iters * 16)
        print(f"N={N} group-1 A offset {goff:5d} B: {c:6.1f} cyc/MMA (avg of aligned + offset group)", flush=True)
