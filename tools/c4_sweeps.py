"""Per-sweep device time of C4 rounds (ResNet-18-GN, 100 of 1000 clients)
from the library's globaltimer sweep stamps: where the round goes between
the dense first sweeps and the long tail of the Dirichlet sizes.

    ROUNDS=2 python tools/c4_sweeps.py
"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_01778_b200.resnet as rn  # noqa: E402
from paper_2303_01778_b200.cnn import sweep_plan  # noqa: E402

rounds = int(os.environ.get("ROUNDS", "2"))
dev = torch.device("cuda", 0)
eng = bench.c4_engine(dev, rounds + 2)
captured = []
orig = rn.resnet_train_group


def traced(*a, **kw):
    _, _, _, active = sweep_plan(a[3], kw["batch_size"], kw["epochs"])
    tl = torch.zeros(len(active) + 1, dtype=torch.int64, device=dev)
    kw["timeline"] = tl
    captured.append((active, tl))
    return orig(*a, **kw)


eng.run_round(0)
rn.resnet_train_group = traced
for r in range(1, rounds + 1):
    captured.clear()
    eng.run_round(r)
    torch.cuda.synchronize()
    active, tl = captured[-1]
    us = np.diff(tl.cpu().numpy().astype(np.float64)) / 1e3
    print(f"round {r}: {len(us)} sweeps, {us.sum() / 1e3:.2f} ms of training")
    edges = [0, 1, 2, 4, 8, 16, 32, 64, 10 ** 9]
    for lo, hi in zip(edges, edges[1:]):
        sel = (active >= lo) & (active < hi)
        if sel.any():
            print(f"  active [{lo}, {hi}): {int(sel.sum())} sweeps, {us[sel].sum() / 1e3:.2f} ms, "
                  f"{us[sel].mean():.0f} us per sweep")
