"""Where the device-timed C2 round spends the time outside the 72 training
sweeps: CUDA events at execute_round entry, just before and just after the
pb_cnn_train_group launch sequence, and at execute_round exit, over rounds
run back to back as in bench.py (prepared inputs, sync=False).

    ROUNDS=4 python tools/round_gaps.py
"""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
import paper_2303_01778_b200._lib as L  # noqa: E402

rounds = int(os.environ.get("ROUNDS", "4"))
dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=rounds + 3, warmup_rounds=1, seed=0, scheme="PARROT")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data)
eng.run_round(0)
eng.run_round(1)
marks = []
host = []
real = L.lib.pb_cnn_train_group


def traced(*a):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks[-1]["pre"] = e
    host[-1]["launch0"] = time.perf_counter()
    rc = real(*a)
    e2 = torch.cuda.Event(enable_timing=True)
    e2.record()
    marks[-1]["post"] = e2
    host[-1]["launch1"] = time.perf_counter()
    return rc


L.lib.pb_cnn_train_group = traced
prepared = [eng.prepare_round(2 + i) for i in range(rounds)]
for p in prepared:
    p.upload()
torch.cuda.synchronize()
for p in prepared:
    m = {"in": torch.cuda.Event(enable_timing=True), "out": torch.cuda.Event(enable_timing=True)}
    marks.append(m)
    host.append({"in": time.perf_counter()})
    m["in"].record()
    eng.execute_round(p, sync=False)
    m["out"].record()
    host[-1]["out"] = time.perf_counter()
torch.cuda.synchronize()
for i, (m, h) in enumerate(zip(marks, host)):
    pre = m["in"].elapsed_time(m["pre"])
    train = m["pre"].elapsed_time(m["post"])
    post = m["post"].elapsed_time(m["out"])
    gap = marks[i - 1]["out"].elapsed_time(m["in"]) if i else float("nan")
    print(f"round {i}: device in->train {pre:.2f} ms, train(+enqueue) {train:.2f}, after {post:.2f}, "
          f"gap from previous round {gap:.2f}; host in->launch0 {1e3 * (h['launch0'] - h['in']):.2f}, "
          f"launch seq {1e3 * (h['launch1'] - h['launch0']):.2f}, total host {1e3 * (h['out'] - h['in']):.2f} ms")
