"""Benchmark: FL rounds/sec, 1000 clients per round, FEMNIST-shaped CNN
(BASELINE.json metric, config 2 at the headline M_p = 1000), plus the
aggregation microbench (config 5) as a secondary measurement.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

A "step" is one Parrot round: select 1000 of 3400 clients, heterogeneity-
aware schedule over the N GPUs (K = N devices, one per rank), every client's
full local SGD run (E=1, bs=20, lr=0.05), hierarchical fold, NCCL reduction
of the per-GPU partials, FedAvg server update.

* ``value``  device-timed rounds/s with the round's inputs (plan, minibatch
  row ids, global model) already in HBM: CUDA events around K rounds,
  barrier + synchronize on both sides, max over ranks;
* ``e2e``    the same rounds through the public API
  (``SimulationEngine.run_round``): host selection/schedule/permutations,
  host->device copies of the round inputs and the device->host read of the
  round's loss/step results inside the timed region;
* ``roofline`` for the dominant kernel (per-kernel CUDA events recorded by
  the library on the launching stream over the timed rounds);
* ``cpu_baseline``: the CPU oracle port (torch, all host threads) on a
  bounded sample of the same round, extrapolated to 1000 clients.

Data: synthetic FEMNIST-shaped (28x28, 62 classes) Gaussian class mixture of
fedsim.data.generate's form, generated on the device (768,400 samples, 2.4
GB fp32; client sizes from the reference's Dirichlet(1.0) partition rule,
bit-exact); inputs exceed L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

M_TOTAL, M_ROUND, N_CLASSES, BS, LR, EPOCHS = 3400, 1000, 62, 20, 0.05, 1
N_SAMPLES = 768_400
PEAKS = {"hbm_gbs": 6542.1, "bf16_tflops": 1668.8, "bf16_tflops_sustained": 1366.7}
# algorithmic work: CNN training 73.8 MFLOP/sample at P = 1,690,046
FLOP_CONV2_PER_SAMPLE = 3 * 2 * 14 * 14 * 64 * 800   # fwd + dgrad + wgrad of conv2
FLOP_TRAIN_PER_SAMPLE = 73.8e6


def load_peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {k: d.get(k, v) for k, v in PEAKS.items()}, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def client_sizes():
    from paper_2303_01778_b200.core import STREAM_PARTITION, stream_rng
    from paper_2303_01778_b200.data import PartitionSpec, client_sizes as sizes_fn
    return sizes_fn(N_SAMPLES, M_TOTAL, PartitionSpec(quantity_skew=1.0, min_samples_per_client=10),
                    stream_rng(0, STREAM_PARTITION))


def build_device_data(device):
    """FEMNIST-shaped Gaussian mixture on the device (same construction as
    fedsim.data.generate: unit-norm class means * 3.0 + N(0,1) noise)."""
    import torch
    from paper_2303_01778_b200.trainer import ClientData
    g = torch.Generator(device=device).manual_seed(0)
    means = torch.randn(N_CLASSES, 784, generator=g, device=device)
    means *= 3.0 / means.norm(dim=1, keepdim=True)
    labels = torch.randint(0, N_CLASSES, (N_SAMPLES,), generator=g, device=device, dtype=torch.int64)
    X = torch.empty(N_SAMPLES, 784, device=device)
    chunk = 1 << 17
    for lo in range(0, N_SAMPLES, chunk):
        hi = min(N_SAMPLES, lo + chunk)
        X[lo:hi] = means[labels[lo:hi]] + torch.randn(hi - lo, 784, generator=g, device=device)
    sizes = client_sizes()
    base = np.zeros(M_TOTAL, dtype=np.int64)
    base[1:] = np.cumsum(sizes)[:-1]
    return ClientData(X, labels.to(torch.int32), base, sizes.astype(np.int64), 784, N_CLASSES), sizes


def light_profiles(sizes):
    """ClientProfiles carrying only sample counts (the data lives on the GPU)."""
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    feat = np.zeros((1, 784), dtype=np.float32)
    out = []
    for cid, n in enumerate(sizes):
        n = int(n)
        out.append(ClientProfile(cid, n, DataSlice(np.broadcast_to(feat, (n, 784)),
                                                   np.zeros(n, dtype=np.int64), np.arange(n))))
    return out


# ---------------------------------------------------------------------------
# clocks sampling
# ---------------------------------------------------------------------------

def quiesce_host() -> None:
    """Benchmark hygiene before a timed window: collect the set-up garbage and
    freeze the surviving objects, so a full cyclic-GC pass over the whole
    heap (tens of ms) does not land inside the window by chance."""
    import gc
    gc.collect()
    gc.freeze()


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        # NVML directly (a query takes microseconds: many samples even in a
        # sub-second timed region); nvidia-smi as the fallback
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            try:   # the CUDA device's own GPU (NVML indices ignore CUDA_VISIBLE_DEVICES)
                pr = torch.cuda.get_device_properties(self.index)
                h = pynvml.nvmlDeviceGetHandleByPciBusId(
                    f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = (0x8, 0x40, 0x20, 0x4)   # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in bits])
                self._stop.wait(0.02)
            return
        except Exception:
            self.rows.clear()
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=5)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------

def dist_setup(gpus: int):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(v: float, world: int) -> float:
    import torch
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def round_selection(r: int) -> list[int]:
    from paper_2303_01778_b200.core import SimConfig, select_clients
    cfg = SimConfig(total_clients=M_TOTAL, concurrent_clients=M_ROUND, num_devices=1,
                    total_rounds=r + 2, seed=0, scheme="PARROT")
    return [int(m) for m in select_clients(cfg, r).selected]


def cpu_sample_rounds_per_s(sizes, selected, stride: int, offset: int = 0, threads: int | None = None):
    """Oracle port (torch CPU fp32, all host threads) on a stratified sample
    of one round: the round's clients sorted by sample count, every
    `stride`-th from `offset` (so the sample spans the size distribution),
    each running its full local schedule on FEMNIST-shaped Gaussian-mixture
    data; rounds/s = 1 / (measured seconds per sample x the round's samples)."""
    import torch
    from oracle import cnn_oracle
    from paper_2303_01778_b200.models import cnn_init, cnn_spec
    if threads:
        torch.set_num_threads(threads)
    spec = cnn_spec(N_CLASSES)
    w0 = cnn_init(spec, seed=0)
    ranked = sorted(selected, key=lambda m: (int(sizes[m]), m))
    picks = ranked[offset::stride]
    rng = np.random.default_rng(100 + offset)
    means = rng.standard_normal((N_CLASSES, 784)).astype(np.float32)
    means *= 3.0 / np.linalg.norm(means, axis=1, keepdims=True)
    samples, secs = 0, 0.0
    for m in picks:
        n = int(sizes[m])
        y = rng.integers(0, N_CLASSES, n)
        X = means[y] + rng.standard_normal((n, 784), dtype=np.float32)
        t0 = time.perf_counter()
        cnn_oracle.client_train(w0, X, y, int(m), 0, 0, EPOCHS, BS, LR, N_CLASSES, dtype=torch.float32)
        secs += time.perf_counter() - t0
        samples += n
    round_samples = int(sum(int(sizes[m]) for m in selected))
    return samples / secs / round_samples, {
        "clients": len(picks), "samples": samples, "seconds": secs, "round_samples": round_samples,
        "threads": torch.get_num_threads()}


def run_b200(args) -> dict:
    import torch
    import paper_2303_01778_b200 as pb
    from paper_2303_01778_b200._lib import KERNEL_CLASSES, lib, prof_collect
    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    data, sizes = build_device_data(dev)
    profiles = light_profiles(sizes)
    total_rounds = args.warmup + 3 * args.steps + 2
    cfg = pb.SimConfig(total_clients=M_TOTAL, concurrent_clients=M_ROUND, num_devices=world,
                       total_rounds=total_rounds, warmup_rounds=1, seed=0, scheme="PARROT",
                       scheduling="time-window")
    eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=LR, batch_size=BS), profiles,
                              pb.make_device_models(world), model="cnn", client_data=data,
                              init_seed=0)
    r = 0
    for _ in range(args.warmup):
        eng.run_round(r)
        r += 1
    # ---- profiled rounds: CUDA events around every launch (the per-kernel
    # breakdown).  The events cost ~4 ms per round, so the timed rounds below
    # record only the dominant kernel. ----
    prepared = [eng.prepare_round(r + i) for i in range(args.steps)]
    prof_samples = sum(int(np.sum(p.group.n)) for p in prepared if p.group)
    prof_steps = sum(int(np.sum((p.group.n + BS - 1) // BS)) for p in prepared if p.group)
    for p in prepared:
        p.upload()
    torch.cuda.synchronize()
    prof_collect()
    lib.pb_prof_select(~0 & 0xFFFFFFFFFFFFFFFF)
    lib.pb_prof_enable(1)
    for p in prepared:
        eng.execute_round(p, sync=False)
    torch.cuda.synchronize()
    lib.pb_prof_enable(0)
    kernels = prof_collect()
    r += args.steps
    dom_name = max(kernels.items(), key=lambda kv: kv[1][0])[0] if kernels else None
    # ---- device-timed rounds (inputs prepared and resident before timing) ----
    prepared = [eng.prepare_round(r + i) for i in range(args.steps)]
    # algorithmic work of the timed rounds: client-steps (fc1 streams) and samples
    client_steps = sum(int(np.sum((p.group.n + BS - 1) // BS)) for p in prepared if p.group)
    samples_timed = sum(int(np.sum(p.group.n)) for p in prepared if p.group)
    for p in prepared:
        p.upload()
    if dom_name is not None:
        lib.pb_prof_select(1 << KERNEL_CLASSES.index(dom_name))
        lib.pb_prof_enable(1)
    prof_collect()
    quiesce_host()
    barrier(world)
    launches0 = lib.pb_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record()
        for p in prepared:
            eng.execute_round(p, sync=False)
        e1.record()
        barrier(world)
    launches = lib.pb_launch_count() - launches0
    lib.pb_prof_enable(0)
    lib.pb_prof_select(~0 & 0xFFFFFFFFFFFFFFFF)
    live = prof_collect()
    dev_ms = max_over_ranks(e0.elapsed_time(e1), world)
    r += args.steps
    # ---- end-to-end rounds through the public API ----
    # one untimed round first: it starts run_round's pipeline (the next
    # round's host preparation overlaps this one) and pays the first-use
    # host allocations of the e2e path
    eng.run_round(r)
    r += 1
    quiesce_host()
    barrier(world)
    h2d0, d2h0 = eng.io_bytes()
    t0 = time.perf_counter()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record()
    e2e_rounds_ms = []
    for i in range(args.steps):
        t_r = time.perf_counter()
        eng.run_round(r + i)
        e2e_rounds_ms.append(round((time.perf_counter() - t_r) * 1e3, 2))
    e3.record()
    barrier(world)
    e2e_ms = max_over_ranks(max(e2.elapsed_time(e3), (time.perf_counter() - t0) * 1e3), world)
    h2d1, d2h1 = eng.io_bytes()

    # ---- aggregation microbench (config 5), bounded ----
    agg = aggregation_microbench(world, dev) if args.agg else None
    state = state_microbench(dev) if args.agg and world == 1 else None
    # ---- config 4 (ResNet-18-GN) rounds, 1 GPU, secondary ----
    c4 = resnet_round_bench(dev) if args.c4 and world == 1 else None
    # ---- configs 1 and 3 (LR) next to the reference engine itself ----
    c13 = lr_configs_bench(dev) if args.c13 and world == 1 and rank == 0 else None

    peaks, peak_src = load_peaks()
    samples_round = float(np.sum(sizes)) / M_TOTAL * M_ROUND
    ms_round = dev_ms / args.steps
    # dominant kernel: timed live (events around its launches only) over the timed rounds
    dom_ms = live.get(dom_name, (0.0, 0))[0] if dom_name else 0.0
    roof = roofline(dom_name or "none", dom_ms, live, samples_timed, client_steps, peaks, peak_src)
    roof["measured"] = "CUDA events around each launch of this kernel inside the timed rounds"
    all_roofs = {k: roofline(k, v[0], kernels, prof_samples, prof_steps, peaks, peak_src)
                 for k, v in kernels.items() if k.startswith("cnn_") and k != "cnn_slots"}
    out = {
        "metric": "FL rounds/sec (1000 clients, FEMNIST-CNN)",
        "value": args.steps / (dev_ms / 1e3),
        "unit": "rounds/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_round,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16 (tcgen05 operands of conv1 incl. its weight gradient, conv2 and the low-rank fc1: "
                 "its X/dH history and W0 copy) / fp32 (master weights, TMEM accumulation, fc2, loss)",
        "data": "synthetic FEMNIST-shaped: fedsim.data.generate's construction (unit class means x 3 "
                "+ N(0,1)) drawn from torch's device RNG instead of the reference's NumPy stream (the "
                "values do not change the work); per-client sample counts Dirichlet(1.0), min 10, "
                "bit-exact with fedsim.partition",
        "config": {"workload": "C2: FedAvg 2-layer CNN (P=1,690,046), 3400 clients, 1000 per round, "
                               "bs=20, E=1, lr=0.05, PARROT greedy schedule over the GPUs",
                   "clients_per_round": M_ROUND, "total_clients": M_TOTAL,
                   "samples_per_round": samples_round, "parallelism": f"clients across {world} GPU(s)",
                   "l2": "inputs exceed L2 (2.4 GB data, 6.8 GB client parameters per round)"},
        "e2e": {"value": args.steps / (e2e_ms / 1e3), "unit": "rounds/s", "round_ms": e2e_rounds_ms,
                "h2d_bytes_per_step": int((h2d1 - h2d0) / args.steps),
                "d2h_bytes_per_step": int((d2h1 - d2h0) / args.steps)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernels_ms_per_round": {k: round(v[0] / args.steps, 3) for k, v in kernels.items()},
        "kernels_source": f"{args.steps} profiled rounds before the timed ones (CUDA events around "
                          "every launch; they add ~4 ms per round, so the timed rounds record only "
                          "the dominant kernel)",
        "kernels_roofline_frac": {k: (round(v["frac"], 4) if v.get("frac") is not None else None)
                                  for k, v in all_roofs.items()},
        "round_roofline": {"bound": "tensor",
                           "achieved": CNN_TRAIN_FLOP * samples_timed / (dev_ms / 1e3) / 1e12,
                           "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                           "frac": CNN_TRAIN_FLOP * samples_timed / (dev_ms / 1e3) / 1e12
                           / peaks["bf16_tflops_sustained"],
                           "work": f"{CNN_TRAIN_FLOP:.3g} FLOP/sample x {samples_timed} samples "
                                   f"(whole round, all kernels)"},
        "clocks": clocks.summary(),
    }
    if agg is not None:
        out["aggregation"] = agg
    if state is not None:
        out["state_store"] = state
    if c4 is not None:
        out["c4_resnet"] = c4
    if c13 is not None:
        out["c1_c3_lr"] = c13
    if rank == 0 and args.cpu_baseline and world == 1:
        sel = round_selection(0)
        v, info = cpu_sample_rounds_per_s(sizes, sel, stride=4)
        out["cpu_baseline"] = {"value": v, "unit": "rounds/s", "cores": info["threads"],
                               "kind": "port",
                               "sample": f"stratified quarter of round 0: every 4th of its 1000 clients "
                                         f"by sample count ({info['clients']} clients, {info['samples']} of "
                                         f"{info['round_samples']} samples, full local runs, "
                                         f"{info['seconds']:.1f} s), torch CPU fp32 oracle port (the "
                                         f"reference has no CNN), scaled by the round's samples"}
    return out if rank == 0 else None


# fc1 (per-client weights, 512 x 3136 fp32): the forward streams W1 once,
# the fused backward reads it once and writes it once (SGD update).
FC1_BYTES = {"cnn_fc1_fwd": 4 * 512 * 3136, "cnn_fc1_bwd": 8 * 512 * 3136}
# conv2 implicit-GEMM FLOPs per sample and pass (fwd, dgrad, wgrad)
CONV2_FLOP = 2 * 14 * 14 * 64 * 800
# fc1 FLOPs per sample and pass
FC1_FLOP = 2 * 512 * 3136
# whole CNN training step per sample: 73.8 MFLOP
CNN_TRAIN_FLOP = 73.8e6


_TRAFFIC = None


def measured_traffic(name):
    """DRAM bytes per launch of a kernel class (mean over one C2 round's
    launches) from the newest committed ncu capture profiles/r*_traffic.json
    (tools/traffic_summary.py), or None."""
    global _TRAFFIC
    if _TRAFFIC is None:
        _TRAFFIC = {}
        for name_ in ("r2_traffic.json", "r1_traffic.json"):
            try:
                with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name_)) as fh:
                    _TRAFFIC = json.load(fh)["kernels"]
                break
            except (OSError, ValueError, KeyError):
                continue
    k = _TRAFFIC.get(name)
    return None if k is None else k["dram_bytes_per_launch"]


def roofline(name, ms, kernels, samples_timed, client_steps, peaks, peak_src) -> dict:
    """A kernel vs its roofline: ALGORITHMIC work of the timed rounds divided by
    the kernel's total device time over those rounds (CUDA events recorded by
    the library around each launch, on the launching stream).  `traffic` is
    the measured DRAM bytes per launch (ncu, profiles/r1_traffic.json)."""
    out = _roofline(name, ms, kernels, samples_timed, client_steps, peaks, peak_src)
    out["traffic"] = measured_traffic(name)
    if out["traffic"] is not None:
        out["traffic_unit"] = "DRAM bytes per launch (ncu dram__bytes_read+write, mean over a round)"
    return out


def _roofline(name, ms, kernels, samples_timed, client_steps, peaks, peak_src) -> dict:
    if ms <= 0:
        return {"kernel": name, "bound": None, "achieved": None, "peak": None, "unit": None,
                "frac": None, "traffic": None}
    if name in FC1_BYTES:
        gbs = FC1_BYTES[name] * client_steps / (ms / 1e3) / 1e9
        return {"kernel": name, "bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"], "traffic": None,
                "peak_source": f"{peak_src} HBM copy bandwidth",
                "work": f"{FC1_BYTES[name]} B per client-step x {client_steps} client-steps"}
    if name in ("cnn_fwd", "cnn_bwd_conv", "cnn_wgrad"):
        tf = CONV2_FLOP * samples_timed / (ms / 1e3) / 1e12
        peak = peaks["bf16_tflops_sustained"]
        return {"kernel": name, "bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                "frac": tf / peak, "traffic": None, "peak_source": f"{peak_src} bf16 sustained",
                "work": f"conv2 implicit GEMM {CONV2_FLOP} FLOP/sample x {samples_timed} samples"}
    if name in ("cnn_lz_fwd", "cnn_lz_bwd"):
        # the shared W0 GEMM of the low-rank fc1 (forward / dgrad): 2*512*3136
        # FLOP per sample on tf32 tensor cores (tf32 peak = half the bf16 peak)
        tf = FC1_FLOP * samples_timed / (ms / 1e3) / 1e12
        peak = peaks["bf16_tflops_sustained"] / 2
        return {"kernel": name, "bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                "frac": tf / peak, "traffic": None,
                "peak_source": f"{peak_src} bf16 sustained / 2 (tf32)",
                "work": f"fc1 {FC1_FLOP} FLOP/sample x {samples_timed} samples (history corrections extra)"}
    if name == "cnn_head":
        return {"kernel": name, "bound": "latency", "achieved": None, "peak": None, "unit": None,
                "frac": None, "traffic": None}
    return {"kernel": name, "bound": None, "achieved": None, "peak": None, "unit": None,
            "frac": None, "traffic": None}


def aggregation_microbench(world: int, dev) -> dict:
    """Config 5: weighted sum of 1000 client updates of an 11.17M-param model,
    1000/N clients per GPU, fp32, one fold_group pass + one all-reduce."""
    import torch
    from paper_2303_01778_b200 import _kernels as K
    P = 11_173_962
    g = M_ROUND // world
    xs = torch.empty(g, P, device=dev)
    gen = torch.Generator(device=dev).manual_seed(5)
    for lo in range(0, g, 50):
        xs[lo:lo + 50].normal_(generator=gen)
    w = torch.from_numpy(client_sizes()[:g].astype(np.float32)).to(dev)
    acc = torch.zeros(P, device=dev)
    for _ in range(2):
        acc.zero_()
        K.fold_group(acc, xs, None, w)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        acc.zero_()
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.fold_group(acc, xs, None, w)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ms = max_over_ranks(min(times), world)
    red_ms = None
    if world > 1:
        import torch.distributed as dist
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dist.all_reduce(acc)
        b.record()
        torch.cuda.synchronize()
        red_ms = max_over_ranks(a.elapsed_time(b), world)
    peaks, src = load_peaks()
    alg_bytes = 4.0 * g * P + 8.0 * P  # each client row read once, acc read+written once
    gbs = alg_bytes / (ms / 1e3) / 1e9
    out = {"clients_per_gpu": g, "params": P, "fold_ms": ms, "achieved_gbs": gbs,
           "peak_gbs": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"],
           "algorithmic_bytes": "4*P per client + 8*P per launch (acc read+write)",
           "clients_per_s": g * world / (ms / 1e3)}
    if red_ms is not None:
        out["allreduce_ms"] = red_ms
    del xs
    torch.cuda.empty_cache()
    return out


def state_microbench(dev, P: int = 11_173_962, slots: int = 1000, clients: int = 100) -> dict:
    """Config 3's client-state manager at ResNet size: gather `clients` rows
    of a [slots, P] fp32 HBM store into the working buffer and scatter them
    back (pb_state_gather / pb_state_scatter, SCAFFOLD control variates).
    Algorithmic bytes: 16 per parameter per client (read + write, both ways)."""
    import torch
    from paper_2303_01778_b200 import _kernels as K
    pad = (P + 3) // 4 * 4  # rows 16-byte aligned, as the StateStore lays them out
    store = torch.empty(slots, pad, device=dev)[:, :P]
    work = torch.empty(clients, pad, device=dev)[:, :P]
    gen = torch.Generator(device=dev).manual_seed(9)
    store.normal_(generator=gen)
    rows = np.random.default_rng(3).choice(slots, clients, replace=False).astype(np.int32)
    slot = torch.from_numpy(rows).to(dev)
    for _ in range(2):
        K.state_gather(work, store, slot)
        K.state_scatter(store, work, slot)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.state_gather(work, store, slot)
        K.state_scatter(store, work, slot)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    ok = bool(torch.equal(store[torch.from_numpy(rows).long().to(dev)], work))
    peaks, src = load_peaks()
    gbs = 16.0 * clients * P / (best / 1e3) / 1e9
    del store
    # the StateStore's pinned host tier (clients beyond the HBM budget): the
    # same kernels read / write the device-mapped rows over the host link
    hc = 8
    host = torch.empty(hc, pad, pin_memory=True)[:, :P]
    host.normal_()
    hslot = torch.arange(hc, dtype=torch.int32, device=dev)
    hwork = work[:hc]
    K.state_gather(hwork, host, hslot)
    K.state_scatter(host, hwork, hslot)
    torch.cuda.synchronize()
    hbest = float("inf")
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.state_gather(hwork, host, hslot)
        K.state_scatter(host, hwork, hslot)
        b.record()
        torch.cuda.synchronize()
        hbest = min(hbest, a.elapsed_time(b))
    host_ok = bool(torch.equal(host.to(dev), hwork))
    del work, host
    torch.cuda.empty_cache()
    return {"params": P, "store_slots": slots, "clients": clients, "gather_scatter_ms": best,
            "achieved_gbs": gbs, "peak_gbs": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"],
            "algorithmic_bytes": "16 B per parameter per client (gather read+write, scatter read+write)",
            "round_trip_exact": ok,
            "host_tier": {"clients": hc, "gather_scatter_ms": hbest,
                          "link_gbs": 8.0 * hc * P / (hbest / 1e3) / 1e9,
                          "link_bytes": "8 B per parameter per client over the host link (read + write)",
                          "round_trip_exact": host_ok}}


# ---------------------------------------------------------------------------
# config 4: ResNet-18 (GroupNorm) FedAvg rounds (secondary measurement)
# ---------------------------------------------------------------------------
C4_TOTAL, C4_ROUND, C4_SAMPLES, C4_CLASSES = 1000, 100, 50_000, 10
# ResNet-18 CIFAR training FLOPs per sample: 0.556 GMAC fwd x 2 x 3
C4_FLOP_PER_SAMPLE = 3.34e9


def c4_engine(dev, total_rounds: int):
    """C4's engine: 1000 clients with the reference's Dirichlet size rule
    (label skew 0.5, quantity skew 0.1, min 5 samples), 100 per round, bs 20,
    E 1, lr 0.05 on one GPU; synthetic CIFAR-shaped data generated on the
    device."""
    import torch
    import paper_2303_01778_b200 as pb
    from paper_2303_01778_b200.core import STREAM_PARTITION, ClientProfile, DataSlice, stream_rng
    from paper_2303_01778_b200.data import PartitionSpec, client_sizes as sizes_fn
    from paper_2303_01778_b200.trainer import ClientData
    sizes = sizes_fn(C4_SAMPLES, C4_TOTAL, PartitionSpec(label_skew=0.5, quantity_skew=0.1,
                                                         min_samples_per_client=5),
                     stream_rng(0, STREAM_PARTITION))
    g = torch.Generator(device=dev).manual_seed(4)
    means = torch.randn(C4_CLASSES, 3072, generator=g, device=dev)
    means *= 3.0 / means.norm(dim=1, keepdim=True)
    labels = torch.randint(0, C4_CLASSES, (C4_SAMPLES,), generator=g, device=dev, dtype=torch.int64)
    X = means[labels] + torch.randn(C4_SAMPLES, 3072, generator=g, device=dev)
    base = np.zeros(C4_TOTAL, dtype=np.int64)
    base[1:] = np.cumsum(sizes)[:-1]
    data = ClientData(X, labels.to(torch.int32), base, sizes.astype(np.int64), 3072, C4_CLASSES)
    feat = np.zeros((1, 3072), dtype=np.float32)
    profiles = [ClientProfile(c, int(n), DataSlice(np.broadcast_to(feat, (int(n), 3072)),
                                                  np.zeros(int(n), dtype=np.int64), np.arange(int(n))))
                for c, n in enumerate(sizes)]
    cfg = pb.SimConfig(total_clients=C4_TOTAL, concurrent_clients=C4_ROUND, num_devices=1,
                       total_rounds=total_rounds, warmup_rounds=1, seed=0, scheme="PARROT")
    return pb.SimulationEngine(cfg, pb.FedAvg(lr=LR, batch_size=BS), profiles, pb.make_device_models(1),
                               model="resnet", client_data=data, init_seed=0)


def resnet_round_bench(dev, steps: int = 2, warmup: int = 1) -> dict:
    """C4 rounds (c4_engine): a profiled pass for the per-kernel breakdown,
    then device-timed rounds."""
    import torch
    from paper_2303_01778_b200._lib import lib, prof_collect
    eng = c4_engine(dev, warmup + 2 * steps + 1)
    for r in range(warmup):
        eng.run_round(r)
    # profiled rounds (events around every launch) for the per-kernel breakdown
    prepared = [eng.prepare_round(warmup + i) for i in range(steps)]
    prof_samples = sum(int(np.sum(p.group.n)) for p in prepared if p.group)
    for p in prepared:
        p.upload()
    torch.cuda.synchronize()
    prof_collect()
    lib.pb_prof_enable(1)
    for p in prepared:
        eng.execute_round(p, sync=False)
    torch.cuda.synchronize()
    lib.pb_prof_enable(0)
    kernels = prof_collect()
    # timed rounds, no per-launch events
    prepared = [eng.prepare_round(warmup + steps + i) for i in range(steps)]
    samples = sum(int(np.sum(p.group.n)) for p in prepared if p.group)
    for p in prepared:
        p.upload()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for p in prepared:
        eng.execute_round(p, sync=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    peaks, src = load_peaks()
    tf = C4_FLOP_PER_SAMPLE * samples / (ms / 1e3) / 1e12
    conv_ms = sum(v[0] for k, v in kernels.items() if k.startswith("rn_conv"))
    conv_tf = C4_FLOP_PER_SAMPLE * prof_samples / (conv_ms / 1e3) / 1e12 if conv_ms > 0 else None
    del eng
    torch.cuda.empty_cache()
    return {"workload": "C4: FedAvg ResNet-18-GN (P=11,173,962), 1000 clients (Dirichlet sizes, "
                        "quantity skew 0.1), 100 per round, bs=20, E=1, lr=0.05, 1 GPU",
            "rounds_per_s": steps / (ms / 1e3), "ms_per_round": ms / steps,
            "samples_per_round": samples / steps,
            "roofline": {"bound": "tensor", "achieved": tf, "peak": peaks["bf16_tflops_sustained"],
                         "unit": "TFLOP/s", "frac": tf / peaks["bf16_tflops_sustained"],
                         "peak_source": f"{src} bf16 sustained",
                         "work": f"{C4_FLOP_PER_SAMPLE:.3g} FLOP/sample x {samples} samples, whole round"},
            "conv_kernels_tflops": conv_tf,
            "kernels_ms_per_round": {k: round(v[0] / steps, 3) for k, v in kernels.items()}}


# ---------------------------------------------------------------------------
# configs 1 and 3 (the reference's own LR model): GPU rounds next to the
# REFERENCE package itself (fedsim 0.1.0 installed under baseline/_ref) timed
# on this box's host cores in a child process
# ---------------------------------------------------------------------------
C13_ROUNDS = 12


def _lr_worlds(mod):
    """C1 and C3 inputs from a package exposing the fedsim API (the reference
    itself, or this package, whose generate/partition are bit-exact with it:
    tests/test_host_parity.py)."""
    ds = mod.generate(60000, 784, 10, seed=0)
    ev = mod.generate(10000, 784, 10, seed=0, sample_set=1)
    c1 = mod.partition(ds, 100, mod.PartitionSpec(), seed=0)
    c3 = mod.partition(ds, 1000, mod.PartitionSpec(quantity_skew=0.5, min_samples_per_client=5), seed=0)
    return ev, c1, c3


def _c13_engines(mod, ev, c1, c3, rounds, store):
    cfg1 = mod.SimConfig(total_clients=100, concurrent_clients=10, num_devices=1, total_rounds=rounds,
                         seed=0, scheme="SP")
    cfg3 = mod.SimConfig(total_clients=1000, concurrent_clients=100, num_devices=8, total_rounds=rounds,
                         seed=0, scheme="PARROT")
    hetero = [0.1 * k for k in range(8)]
    e1 = mod.SimulationEngine(cfg1, mod.FedAvg(lr=0.1, batch_size=20), c1, mod.make_device_models(1),
                              eval_data=ev)
    e3 = mod.SimulationEngine(cfg3, mod.Scaffold(lr=0.05, batch_size=20, client_fraction=0.1), c3,
                              mod.make_device_models(8, hetero=hetero), store=store, eval_data=ev)
    return e1, e3


def reference_c13_child() -> None:
    """Child process (OPENBLAS_NUM_THREADS=1, NUMBA_CACHE_DIR set): the
    reference engine on C1 (SP, K=1) and C3 (PARROT, K=8 device threads,
    SCAFFOLD with its fsynced file StateStore); median of 3 x C13_ROUNDS
    rounds after 2 warm-up rounds and warm_jit."""
    import tempfile
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    import fedsim
    from fedsim.schedule import warm_jit
    warm_jit()
    ev, c1, c3 = _lr_worlds(fedsim)
    out = {"fedsim": fedsim.__file__, "cores": os.cpu_count()}
    with tempfile.TemporaryDirectory() as root:
        e1, e3 = _c13_engines(fedsim, ev, c1, c3, 2 + 3 * C13_ROUNDS, fedsim.StateStore(root))
        for name, eng in (("c1", e1), ("c3", e3)):
            eng.run(2)
            rates = []
            for _ in range(3):
                t0 = time.perf_counter()
                eng.run(C13_ROUNDS)
                rates.append(C13_ROUNDS / (time.perf_counter() - t0))
            out[name] = float(np.median(rates))
    print(json.dumps(out), flush=True)


def reference_c13() -> dict:
    ref = ROOT / "baseline" / "_ref" / "fedsim"
    if not ref.exists():
        return {"unavailable": "baseline/_ref (the reference package) is not installed"}
    import tempfile
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMBA_CACHE_DIR=tempfile.mkdtemp(prefix="numba_"))
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--_ref_c13"], capture_output=True,
                         text=True, env=env, timeout=900)
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    if res.returncode != 0 or not lines:
        return {"unavailable": f"reference child failed rc={res.returncode}: {res.stderr[-300:]}"}
    return json.loads(lines[-1])


def _time_lr_engine(eng, r0: int, rounds: int) -> dict:
    """Device-timed rounds (inputs prepared and resident) and end-to-end
    rounds through run_round (host preparation, copies, result reads)."""
    import torch
    for r in range(r0, r0 + 2):
        eng.run_round(r)
    r0 += 2
    prepared = [eng.prepare_round(r0 + i) for i in range(rounds)]
    for p in prepared:
        p.upload()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for p in prepared:
        eng.execute_round(p, sync=False)
    b.record()
    torch.cuda.synchronize()
    dev_ms = a.elapsed_time(b)
    r0 += rounds
    eng.run_round(r0)
    r0 += 1
    h0, d0 = eng.io_bytes()
    t0 = time.perf_counter()
    for i in range(rounds):
        eng.run_round(r0 + i)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    h1, d1 = eng.io_bytes()
    return {"rounds_per_s": rounds / (dev_ms / 1e3), "e2e_rounds_per_s": rounds / e2e_s,
            "h2d_bytes_per_round": int((h1 - h0) / rounds), "d2h_bytes_per_round": int((d1 - d0) / rounds)}


def lr_configs_bench(dev) -> dict:
    """C1 (FedAvg LR, 100 clients, 10 per round, SP K=1) and C3 (SCAFFOLD LR,
    1000 clients, 100 per round, PARROT over 8 simulated devices, HBM state
    store) on one GPU, with the evaluation of every round as in the
    reference, beside the reference engine itself on the host cores."""
    import paper_2303_01778_b200 as pb
    ev, c1, c3 = _lr_worlds(pb)
    rounds = 6 + 2 * C13_ROUNDS
    e1, e3 = _c13_engines(pb, ev, c1, c3, rounds, pb.StateStore())
    out = {"c1": {"workload": "C1: FedAvg LR 784x10, 100 clients, 10 per round, bs 20, E 1, "
                              "lr 0.1, SP K=1, eval 10k every round", **_time_lr_engine(e1, 0, C13_ROUNDS)},
           "c3": {"workload": "C3: SCAFFOLD LR 784x10, 1000 clients (quantity skew 0.5), 100 per round, "
                              "bs 20, lr 0.05, PARROT K=8 simulated devices (hetero 0..0.7) on one GPU, "
                              "HBM state store (reference: fsynced files), eval every round",
                  **_time_lr_engine(e3, 0, C13_ROUNDS)}}
    ref = reference_c13()
    out["reference"] = ref
    for k in ("c1", "c3"):
        if k in ref:
            out[k]["reference_rounds_per_s"] = ref[k]
            out[k]["e2e_vs_reference"] = out[k]["e2e_rounds_per_s"] / ref[k]
    return out


# ---------------------------------------------------------------------------
# the reference (CPU oracle port) arm
# ---------------------------------------------------------------------------

def run_reference(args) -> dict | None:
    """The reference arm: the reference has no CNN and no compiled path, so
    C2's CPU implementation is the torch CPU fp32 oracle port
    (oracle/cnn_oracle.py, a restatement of client_execute) on all host
    threads.  Step i times stratum i mod 32 of round 0's clients sorted by
    sample count (about 31 clients spanning the size distribution, full local
    runs), scaled to the round's samples; value = the median over steps."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import torch
    sizes = client_sizes()
    sel = round_selection(0)
    vals, secs = [], 0.0
    for i in range(args.warmup):
        cpu_sample_rounds_per_s(sizes, sel, stride=32, offset=(7 * i + 3) % 32)
    for i in range(args.steps):
        v, info = cpu_sample_rounds_per_s(sizes, sel, stride=32, offset=i % 32)
        vals.append(v)
        secs += info["seconds"]
    v = float(np.median(vals))
    return {"metric": "FL rounds/sec (1000 clients, FEMNIST-CNN)", "value": v, "unit": "rounds/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic FEMNIST-shaped Gaussian mixture; client sizes = the B200 arm's "
                    "(Dirichlet(1.0), bit-exact with fedsim.partition)",
            "config": {"workload": "C2: FedAvg 2-layer CNN (P=1,690,046), 3400 clients, 1000 per round, "
                                   "bs=20, E=1, lr=0.05"},
            "cpu_baseline": {"value": v, "unit": "rounds/s", "cores": torch.get_num_threads(),
                             "kind": "port",
                             "sample": f"per step: one 1/32 stratum of round 0's 1000 clients by sample "
                                       f"count (~31 clients, full local runs; {secs:.0f} s of CPU work "
                                       f"over the {args.steps} steps), torch CPU fp32 oracle port "
                                       f"(the reference has no CNN), scaled to the round's samples"},
            "e2e": {"value": v, "unit": "rounds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-agg", dest="agg", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-c4", dest="c4", action="store_false")
    ap.add_argument("--no-c13", dest="c13", action="store_false")
    ap.add_argument("--_ref_c13", dest="ref_c13", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ref_c13:
        reference_c13_child()
        return
    out = run_reference(args) if args.impl == "reference" else run_b200(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
