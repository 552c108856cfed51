"""Per-kernel-class ms per C2 round (library CUDA events around every
launch), for A/B runs of kernel variants selected by environment knobs:

    ROUNDS=2 python tools/kprobe.py [class ...]
"""
import os
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
import torch  # noqa: E402
from paper_2303_01778_b200._lib import lib, prof_collect  # noqa: E402

rounds = int(os.environ.get("ROUNDS", "2"))
dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=rounds + 2, warmup_rounds=1, seed=0, scheme="PARROT")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data)
eng.run_round(0)
torch.cuda.synchronize()
prof_collect()
lib.pb_prof_enable(1)
for r in range(1, rounds + 1):
    eng.run_round(r)
torch.cuda.synchronize()
lib.pb_prof_enable(0)
k = prof_collect()
want = sys.argv[1:]
tag = os.environ.get("TAG", "")
print(tag, " ".join(f"{n}={ms / rounds:.3f}" for n, (ms, c) in sorted(k.items(), key=lambda x: -x[1][0])
                    if c and (not want or n in want)), flush=True)
