"""cProfile of C1 rounds through SimulationEngine.run_round (FedAvg LR, 10 of
100 clients, SP, eval every round): where the host time of a small round goes.

    python tools/c1_profile.py
"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402

ev, c1, c3 = bench._lr_worlds(pb)
e1, _ = bench._c13_engines(pb, ev, c1, c3, 60, pb.StateStore())
for r in range(5):
    e1.run_round(r)
torch.cuda.synchronize()
t0 = time.perf_counter()
for r in range(5, 25):
    e1.run_round(r)
torch.cuda.synchronize()
print(f"{20 / (time.perf_counter() - t0):.1f} rounds/s")
pr = cProfile.Profile()
pr.enable()
for r in range(25, 45):
    e1.run_round(r)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
