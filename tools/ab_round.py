"""A/B check of two builds of libparrot_b200.so on the bench workload (C2):
run ROUNDS rounds through SimulationEngine and print a SHA-256 of the global
model's bytes after each round plus the device time.  Run once per build
(PB_LIB selects the library) and compare the hashes: a change meant to keep
the arithmetic identical must print the same ones.

    PB_LIB=paper_2303_01778_b200/libparrot_b200_base.so python tools/ab_round.py
    python tools/ab_round.py
"""
import hashlib
import os
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
import torch  # noqa: E402

rounds = int(os.environ.get("ROUNDS", "3"))
dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=rounds + 1, warmup_rounds=1, seed=0, scheme="PARROT")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data)
for r in range(rounds):
    oc = eng.run_round(r)
    flat = torch.cat([t.detach().reshape(-1).float() for t in (e.tensor for e in oc.new_global.entries.values())]).cpu()
    h = hashlib.sha256(flat.numpy().tobytes()).hexdigest()[:16]
    print(f"round {r} sha {h} device_ms {1e3 * oc.device_seconds:.2f} loss {oc.loss}", flush=True)
