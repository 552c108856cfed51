"""Host-side prepare_round time of the C2 bench workload (selection, fits,
greedy schedule, minibatch orders, pinned staging)."""
import sys
import time
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
import torch  # noqa: E402

dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=12, warmup_rounds=1, seed=0, scheme="PARROT", scheduling="time-window")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data, init_seed=0)
import cProfile, pstats  # noqa: E402
for r in range(10):
    t0 = time.perf_counter()
    inp = eng.prepare_round(r)
    t1 = time.perf_counter()
    print(f"round {r}: prepare {1e3 * (t1 - t0):.1f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
eng.prepare_round(10)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
