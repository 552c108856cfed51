"""Per-round end-to-end vs device time of the C2 bench workload through
SimulationEngine.run_round (host prep prefetched, per-round sync)."""
import sys
import time
sys.path.insert(0, ".")
import bench  # noqa: E402
import numpy as np  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
import torch  # noqa: E402

dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=30, warmup_rounds=1, seed=0, scheme="PARROT", scheduling="time-window")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data, init_seed=0)
for r in range(3):
    eng.run_round(r)
for r in range(3, 13):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    oc = eng.run_round(r)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    print(f"round {r}: wall {wall:.1f} ms  events {e0.elapsed_time(e1):.1f} ms  train-launch {oc.device_seconds * 1e3:.1f} ms", flush=True)
# same rounds' work device-timed back to back

# host-side profile of run_round (the device work dominates cumulative time of
# the blocking sync; the rest is the per-round host overhead)
import cProfile  # noqa: E402
import pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for r in range(13, 16):
    eng.run_round(r)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
