"""Run ROUNDS rounds of the bench workload (C2: 1000 clients/round, CNN) --
a short command for ncu captures."""
import os
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
import torch  # noqa: E402

rounds = int(os.environ.get("ROUNDS", "1"))
dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=rounds + 1, warmup_rounds=1, seed=0, scheme="PARROT")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data)
for r in range(rounds):
    oc = eng.run_round(r)
    print("round", r, "device_s", oc.device_seconds, flush=True)
