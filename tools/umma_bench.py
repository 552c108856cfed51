"""tcgen05 issue throughput per shape and number of independent accumulators."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2303_01778_b200._lib import lib
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for M, N in [(128, 256), (128, 128), (128, 64), (128, 32), (64, 32), (64, 64), (64, 128)]:
    for nacc in (1, 2, 4, 8):
        if nacc * N > 256:
            continue
        lib.check(lib.pb_umma_bench(M, N, 2, 1, 2000, nacc, out.data_ptr(), 0))
        torch.cuda.synchronize()
        c = out.item() / 2000
        print(f"M={M:3d} N={N:3d} accum={nacc}: {c:6.1f} cyc/MMA {2 * M * N * 16 / c:6.0f} flop/cyc", flush=True)

# several CTAs per SM: is the small-N issue floor per CTA or per SM?
import collections
for M, N in [(128, 32), (128, 64), (64, 64), (128, 256)]:
    for grid in (148, 296, 592):
        cyc = torch.zeros(grid, dtype=torch.int64, device="cuda")
        sm = torch.zeros(grid, dtype=torch.int32, device="cuda")
        lib.check(lib.pb_umma_bench_multi(M, N, 4000, grid, cyc.data_ptr(), sm.data_ptr(), 0))
        torch.cuda.synchronize()
        per_sm = collections.Counter(sm.tolist())
        c = cyc.double().max().item() / 4000
        k = max(per_sm.values())
        print(f"M={M:3d} N={N:3d} grid={grid}: up to {k} CTAs/SM, {c:6.1f} cyc per MMA per CTA -> "
              f"{k * 2 * M * N * 16 / c:6.0f} flop/cyc/SM", flush=True)
