"""Per-sweep device time of C2 rounds (bench workload, 1000 clients/round),
from the library's globaltimer stamps (k_slots stamps each sweep's start):
where the round's time goes between the dense head and the sparse tail.

    ROUNDS=3 python tools/sweep_times.py
"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
import paper_2303_01778_b200.cnn as cnn  # noqa: E402

rounds = int(os.environ.get("ROUNDS", "3"))
dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=rounds + 2, warmup_rounds=1, seed=0, scheme="PARROT")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data)
captured = []
orig = cnn.cnn_train_group


def traced(*a, **kw):
    n = a[3]
    _, total, _, active = cnn.sweep_plan(n, kw["batch_size"], kw["epochs"])
    tl = torch.zeros(len(active) + 1, dtype=torch.int64, device=dev)
    kw["timeline"] = tl
    captured.append((active, tl))
    return orig(*a, **kw)


eng.run_round(0)
cnn.cnn_train_group = traced
acc = None
for r in range(1, rounds + 1):
    captured.clear()
    eng.run_round(r)
    torch.cuda.synchronize()
    active, tl = captured[-1]
    t = tl.cpu().numpy().astype(np.float64)
    us = np.diff(t) / 1e3
    acc = us if acc is None or len(acc) != len(us) else acc + us
    print(f"round {r}: {len(us)} sweeps, {us.sum() / 1e3:.2f} ms of training")
us = acc / rounds
print("sweep active   us   (mean over rounds)")
for i, (a, u) in enumerate(zip(active, us)):
    print(f"{i:5d} {a:6d} {u:8.1f}")
for lo, hi in ((0, 12), (12, 24), (24, 48), (48, len(us))):
    print(f"sweeps {lo}-{hi}: {us[lo:hi].sum() / 1e3:.2f} ms")
