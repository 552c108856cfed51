import sys, time
sys.path.insert(0, ".")
import torch, numpy as np
import bench, paper_2303_01778_b200 as pb
from paper_2303_01778_b200._lib import lib, prof_collect
dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
K, W = 5, 3
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=W + 3 * K + 2, warmup_rounds=1, seed=0, scheme="PARROT", scheduling="time-window")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data, init_seed=0)
r = 0
for _ in range(W):
    eng.run_round(r); r += 1
for rep in range(2):
    prepared = [eng.prepare_round(r + i) for i in range(K)]
    for p in prepared: p.upload()
    torch.cuda.synchronize()
    for p in prepared: eng.execute_round(p, sync=False)
    torch.cuda.synchronize()
    r += K
bench.quiesce_host()
orig_exec = eng.execute_round
for i in range(K):
    ms0 = torch.cuda.memory_stats()
    seg0 = {(x["address"], x["total_size"]) for x in torch.cuda.memory_snapshot()}
    t0 = time.perf_counter()
    inp = eng.prepare_round(r + i)
    t1 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    oc = eng.execute_round(inp)
    e1.record(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    ms1 = torch.cuda.memory_stats()
    seg1 = {(x["address"], x["total_size"]) for x in torch.cuda.memory_snapshot()}
    new = sorted(sz for _, sz in seg1 - seg0)
    if new:
        print("  new segments (bytes):", new, flush=True)
    print(f"round {r+i}: prepare {1e3*(t1-t0):.1f} ms, execute wall {1e3*(t2-t1):.1f} ms, gpu {e0.elapsed_time(e1):.1f} ms, train {oc.device_seconds*1e3:.1f} ms, "
          f"cudaMalloc +{ms1.get('num_device_alloc', 0) - ms0.get('num_device_alloc', 0)}, retries +{ms1.get('num_alloc_retries', 0) - ms0.get('num_alloc_retries', 0)}, reserved {ms1.get('reserved_bytes.all.current', 0) / 1e9:.1f} GB", flush=True)
