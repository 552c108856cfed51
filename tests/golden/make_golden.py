"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
(FedML Parrot ``fedsim`` 0.1.0 at /root/reference/pkg/src) in this container.

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden.py [seam]

The reference tree is read-only and absent on the GPU box, so its outputs are
committed here as small fixtures; nothing at test time reads /root/reference.
Every fixture records which reference entry point produced it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
sys.path.insert(0, "/root/reference/pkg/src")

from fedsim.aggregate import DevicePartial, global_fold, local_fold  # noqa: E402
from fedsim.core import ClientProfile, ClientSelection, DataSlice, SimConfig, select_clients  # noqa: E402
from fedsim.data import PartitionSpec, _client_sizes, generate, partition  # noqa: E402
from fedsim.engine import (DeviceModel, SimulationEngine, make_device_models,  # noqa: E402
                           report_time, virtual_task_seconds)
from fedsim.estimate import TimingHistory, TimingRecord, WorkloadFit, fit_device  # noqa: E402
from fedsim.schedule import greedy_assign, uniform_division  # noqa: E402
from fedsim.statestore import StateStore, encode_tensor_map  # noqa: E402
from fedsim.trainer import (AggOp, FedAvg, FedDyn, FedNova, FedProx, ModelParams,  # noqa: E402
                            ParamBundle, Scaffold, client_execute)
from fedsim.statestore import ClientState  # noqa: E402
from fedsim.core import stream_rng  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# --------------------------------------------------------------------------
# trainer: client_execute per plugin (fedsim/trainer.py:427-477)
# --------------------------------------------------------------------------

def trainer_cases() -> dict:
    out = {}
    rng = np.random.default_rng(2024)
    n, f, c = 37, 6, 3
    X = rng.standard_normal((n, f))
    y = rng.integers(0, c, n)
    y[:c] = np.arange(c)
    W0 = 0.3 * rng.standard_normal((c, f))
    b0 = 0.3 * rng.standard_normal(c)
    ctrl_g = (0.05 * rng.standard_normal((c, f)), 0.05 * rng.standard_normal(c))
    st_a = (0.05 * rng.standard_normal((c, f)), 0.05 * rng.standard_normal(c))
    out["X"], out["y"], out["W0"], out["b0"] = X, y, W0, b0
    out["ctrl_gw"], out["ctrl_gb"] = ctrl_g
    out["state_w"], out["state_b"] = st_a
    prof = ClientProfile(5, n, DataSlice(X, y, np.arange(n)))
    plugins = {
        "fedavg": FedAvg(lr=0.1, batch_size=8, collect_local_loss=True),
        "fedprox": FedProx(mu=0.3, lr=0.1, batch_size=8, collect_local_loss=True),
        "fednova": FedNova(lr=0.1, batch_size=8),
        "scaffold": Scaffold(lr=0.1, batch_size=8, client_fraction=0.5),
        "feddyn": FedDyn(alpha=0.2, lr=0.1, batch_size=8),
    }
    for name, plug in plugins.items():
        g = plug.init_global(ModelParams(W0, b0))
        state = None
        if name == "scaffold":
            g = g.replaced(server_ctrl_weights=ctrl_g[0], server_ctrl_bias=ctrl_g[1])
            state = ClientState(5, 0, {"ctrl_weights": st_a[0], "ctrl_bias": st_a[1]})
        if name == "feddyn":
            state = ClientState(5, 0, {"grad_corr_weights": st_a[0], "grad_corr_bias": st_a[1]})
        rep = client_execute(plug, prof, g, state, epochs=2, batch_size=8, lr=0.1,
                             seed=9, round_num=3)
        for en, e in rep.client_result.entries.items():
            out[f"{name}/res/{en}"] = e.tensor
            out[f"{name}/w/{en}"] = np.array([e.weight])
        if rep.new_state is not None:
            for k, v in rep.new_state.payload.items():
                out[f"{name}/state/{k}"] = v
    return out


# --------------------------------------------------------------------------
# end-to-end engine runs (fedsim/engine.py:748-828)
# --------------------------------------------------------------------------

def engine_run(tag, out, cfg, plugin, profiles, devices, store=None, eval_ds=None):
    eng = SimulationEngine(cfg, plugin, profiles, devices, store=store, eval_data=eval_ds)
    outcomes = eng.run()
    for oc in outcomes:
        r = oc.round
        for name, e in oc.new_global.entries.items():
            out[f"{tag}/r{r}/{name}"] = e.tensor
        out[f"{tag}/r{r}/loads"] = np.array([oc.device_loads[k] for k in sorted(oc.device_loads)])
        out[f"{tag}/r{r}/acc_loss"] = np.array([oc.accuracy, oc.loss])
        recs = eng.history.round_records(r)
        out[f"{tag}/r{r}/records"] = np.array(
            [[rec.device_id, rec.client_id, rec.sample_count, rec.reported_seconds] for rec in recs])
        out[f"{tag}/r{r}/mode"] = np.array([oc.scheduling_mode])
        out[f"{tag}/r{r}/costs"] = np.array([oc.costs.trips_up, oc.costs.trips_down,
                                             oc.costs.bytes_avg_params,
                                             oc.costs.bytes_special_params])
    return eng


def engine_cases() -> dict:
    out = {}
    # c02-style: SP and PARROT K=4, FedAvg (tests/test_acceptance.py:96-116)
    ds = generate(1200, 6, 4, seed=11)
    profiles = partition(ds, 40, PartitionSpec(), seed=11)
    for scheme, k in (("SP", 1), ("PARROT", 4)):
        cfg = SimConfig(total_clients=40, concurrent_clients=20, num_devices=k,
                        total_rounds=6, seed=11, scheme=scheme)
        engine_run(f"c02_{scheme}", out, cfg, FedAvg(lr=0.1), profiles, make_device_models(k))

    # hetero PARROT with greedy schedule and noise (bit-exact plans + loads)
    ds = generate(3000, 4, 2, seed=3)
    profiles = partition(ds, 100, PartitionSpec(quantity_skew=0.3), seed=3)
    cfg = SimConfig(total_clients=100, concurrent_clients=40, num_devices=3,
                    total_rounds=6, seed=3, scheme="PARROT", scheduling="time-window",
                    time_window=3)
    engine_run("hetero", out, cfg, FedAvg(lr=0.1, batch_size=10), profiles,
               make_device_models(3, hetero=[0.0, 0.5, 1.0], noise=0.05, b_true=0.01))

    # stateful + other plugins on a small world (tests/test_engine.py:39-43)
    ds = generate(240, 4, 3, seed=5)
    profiles = partition(ds, 12, PartitionSpec(), seed=5)
    eval_ds = generate(120, 4, 3, seed=5, sample_set=1)
    plugs = {"fedprox": FedProx(mu=0.1, lr=0.1, batch_size=5),
             "fednova": FedNova(lr=0.1, batch_size=7),
             "scaffold": Scaffold(lr=0.1, batch_size=5, client_fraction=0.5),
             "feddyn": FedDyn(alpha=0.1, lr=0.1, batch_size=5)}
    for name, plug in plugs.items():
        cfg = SimConfig(total_clients=12, concurrent_clients=6, num_devices=2,
                        total_rounds=4, local_epochs=2, seed=5, scheme="PARROT")
        store = StateStore(tempfile.mkdtemp(prefix="gold_")) if plug.is_stateful else None
        engine_run(f"small_{name}", out, cfg, plug, profiles, make_device_models(2),
                   store=store, eval_ds=eval_ds)
    return out


def c1_c3_cases() -> dict:
    """BASELINE configs 1 and 3 at their real shapes, few rounds."""
    out = {}
    ds = generate(60000, 784, 10, seed=0)
    eval_ds = generate(10000, 784, 10, seed=0, sample_set=1)
    out["c1/features_sha"] = np.array([sha(ds.features)])
    out["c1/labels_sha"] = np.array([sha(ds.labels)])
    out["c1/eval_features_sha"] = np.array([sha(eval_ds.features)])
    profiles = partition(ds, 100, PartitionSpec(), seed=0)
    out["c1/partition_sha"] = np.array([sha(np.concatenate([p.data_partition.indices
                                                             for p in profiles]))])
    cfg = SimConfig(total_clients=100, concurrent_clients=10, num_devices=1,
                    total_rounds=3, seed=0, scheme="SP")
    engine_run("c1", out, cfg, FedAvg(lr=0.1, batch_size=20), profiles,
               make_device_models(1), eval_ds=eval_ds)

    profiles3 = partition(ds, 1000, PartitionSpec(quantity_skew=0.5, min_samples_per_client=5),
                          seed=0)
    out["c3/sizes"] = np.array([p.sample_count for p in profiles3])
    out["c3/partition_sha"] = np.array([sha(np.concatenate([p.data_partition.indices
                                                             for p in profiles3]))])
    cfg = SimConfig(total_clients=1000, concurrent_clients=100, num_devices=8,
                    total_rounds=3, seed=0, scheme="PARROT")
    store = StateStore(tempfile.mkdtemp(prefix="gold_c3_"))
    engine_run("c3", out, cfg, Scaffold(lr=0.05, batch_size=20, client_fraction=0.1),
               profiles3, make_device_models(8, hetero=[0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7]),
               store=store, eval_ds=eval_ds)
    # one stored client state file, byte for byte (fedsim/statestore.py:181-210)
    files = sorted(Path(store.root).glob("client_*.state"))
    out["c3/state_file_name"] = np.array([files[0].name])
    out["c3/state_file_bytes"] = np.frombuffer(files[0].read_bytes(), dtype=np.uint8)
    return out


# --------------------------------------------------------------------------
# host-side bit-exact pieces: selection, partition sizes, schedule, fits,
# device time model, state codec
# --------------------------------------------------------------------------

def host_cases() -> dict:
    out: dict = {}
    sel = {}
    for seed, m, mp, r in [(0, 100, 10, 0), (0, 100, 10, 1), (7, 3400, 1000, 5),
                           (11, 40, 20, 9), (0, 1000, 100, 2), (2 ** 63 + 5, 50, 50, 3)]:
        cfg = SimConfig(total_clients=m, concurrent_clients=mp, num_devices=1,
                        total_rounds=r + 2, seed=seed, scheme="SP")
        sel[f"{seed}/{m}/{mp}/{r}"] = list(select_clients(cfg, r).selected)
    out["selection"] = sel

    sizes = {}
    for tag, n, m, spec in [("c2", 768_400, 3400, PartitionSpec(quantity_skew=1.0,
                                                                min_samples_per_client=10)),
                            ("c4", 50_000, 1000, PartitionSpec(label_skew=0.5, quantity_skew=0.1,
                                                               min_samples_per_client=5))]:
        sizes[tag] = [int(v) for v in _client_sizes(n, m, spec, stream_rng(0, 3))]
    out["partition_sizes"] = sizes

    perms = {}
    for seed, cid, r, n in [(0, 5, 3, 37), (9, 5, 3, 37), (0, 999, 12, 1840), (0, 1, 0, 1),
                            (123456789, 77, 4, 600)]:
        g = stream_rng(seed, 6, cid, r)
        perms[f"{seed}/{cid}/{r}/{n}"] = [[int(v) for v in g.permutation(n)] for _ in range(2)]
    out["minibatch_perms"] = perms

    greedy = []
    rng = np.random.default_rng(77)
    for trial in range(60):
        n = int(rng.integers(1, 80))
        k = int(rng.integers(1, 9))
        ids = [int(v) for v in rng.choice(500, size=n, replace=False)]
        sz = {m: int(rng.integers(1, 60)) for m in ids}
        t = rng.uniform(0.01, 2.0, k)
        b = rng.uniform(-0.5, 0.5, k) if trial % 3 == 0 else rng.uniform(0, 0.2, k)
        fits = {j: WorkloadFit(j, float(t[j]), float(b[j]), 2, "all-history") for j in range(k)}
        plan = greedy_assign(4, ClientSelection(4, tuple(ids)), fits, sz, k)
        greedy.append({"ids": ids, "sizes": [sz[m] for m in ids], "t": t.tolist(),
                       "b": b.tolist(),
                       "assign": {str(d): v for d, v in plan.assignments.items()},
                       "loads": [plan.predicted_loads[j] for j in range(k)]})
    out["greedy"] = greedy
    uni = uniform_division(0, ClientSelection(0, tuple(range(10, 21))), 4)
    out["uniform_11_4"] = {str(k): v for k, v in uni.assignments.items()}

    fits = []
    rng = np.random.default_rng(5)
    for trial in range(10):
        hist = TimingHistory()
        for i in range(40):
            n = int(rng.integers(5, 200)) if trial != 3 else 50
            hist.add(TimingRecord(0, i, i % 8, n, n * 3e-4 * (1 + 0.05 * rng.standard_normal()) + 0.01))
        win = "all-history" if trial % 2 else 3
        f = fit_device(hist, 0, win, 8)
        fits.append({"records": [[r.client_id, r.round, r.sample_count, r.reported_seconds]
                                 for r in hist.device_records(0, 0, 100)],
                     "window": win, "t": f.t_sample, "b": f.b, "used": f.records_used,
                     "degenerate": f.degenerate})
    out["fits"] = fits

    times = []
    for dev in [DeviceModel(0), DeviceModel(2, hetero_ratio=0.4, dynamic=True, t_true=2e-4,
                                            b_true=0.01, noise=0.05)]:
        for r in range(4):
            for cid in (0, 17):
                v = virtual_task_seconds(dev, 123, 42, r, cid)
                times.append([dev.device_id, r, cid, v, report_time(v, dev, r, 10)])
    out["device_times"] = times

    payload = {"ctrl_weights": np.array([[np.pi, -0.0], [1e-300, np.finfo(np.float64).max]]),
               "ctrl_bias": np.array([2.5, -1.25])}
    out["fsst_payload_hex"] = encode_tensor_map(payload).hex()
    return out


# --------------------------------------------------------------------------
# the device seam: DeviceWorker.execute_clients (fedsim/engine.py:470-503)
# --------------------------------------------------------------------------

def seam_cases() -> dict:
    """One DeviceWorker driven directly (no engine) over two rounds, on a
    FRESH StateStore: the partial (acc, weight sum, count, Collect items,
    fold order) and the timing records it returns."""
    from fedsim.engine import DeviceWorker
    from fedsim.metrics import ReplicaGauge
    out = {}
    ds = generate(240, 4, 3, seed=5)
    profiles = partition(ds, 12, PartitionSpec(), seed=5)
    rng = np.random.default_rng(31)
    W0, b0 = 0.2 * rng.standard_normal((3, 4)), 0.2 * rng.standard_normal(3)
    cg = (0.05 * rng.standard_normal((3, 4)), 0.05 * rng.standard_normal(3))
    out["W0"], out["b0"], out["ctrl_gw"], out["ctrl_gb"] = W0, b0, cg[0], cg[1]
    cfg = SimConfig(total_clients=12, concurrent_clients=6, num_devices=2, total_rounds=4,
                    local_epochs=2, seed=5, scheme="PARROT")
    dev = DeviceModel(1, hetero_ratio=0.3, noise=0.05, t_true=2e-4, b_true=0.01)
    rounds = [(0, [3, 7, 1]), (1, [7, 2, 3])]
    out["rounds"] = np.array([[r] + c for r, c in rounds])
    for name, plug in (("fedavg", FedAvg(lr=0.1, batch_size=5, collect_local_loss=True)),
                       ("scaffold", Scaffold(lr=0.1, batch_size=5, client_fraction=0.5))):
        store = StateStore(tempfile.mkdtemp(prefix="gold_seam_")) if plug.is_stateful else None
        worker = DeviceWorker(dev, cfg, plug, profiles, store, ReplicaGauge())
        glob = plug.init_global(ModelParams(W0, b0))
        if name == "scaffold":
            glob = glob.replaced(server_ctrl_weights=cg[0], server_ctrl_bias=cg[1])
        for r, clients in rounds:
            part, timings = worker.execute_clients(glob, clients, r)
            tag = f"{name}/r{r}"
            out[f"{tag}/folded"] = np.array(part.clients_folded)
            out[f"{tag}/records"] = np.array([[t.device_id, t.client_id, t.round, t.sample_count,
                                               t.reported_seconds] for t in timings])
            for en, pe in part.entries.items():
                out[f"{tag}/op/{en}"] = np.array([pe.op.value])
                out[f"{tag}/count/{en}"] = np.array([pe.count])
                if pe.op is AggOp.COLLECT:
                    out[f"{tag}/collect_ids/{en}"] = np.array([c for c, _ in pe.collected])
                    out[f"{tag}/collect/{en}"] = np.stack([np.asarray(t) for _, t in pe.collected])
                else:
                    out[f"{tag}/acc/{en}"] = pe.acc
                    out[f"{tag}/wsum/{en}"] = np.array([pe.weight_sum])
    return out


def main() -> None:
    if sys.argv[1:] == ["seam"]:
        np.savez_compressed(OUT / "seam.npz", **seam_cases())
        return
    np.savez_compressed(OUT / "seam.npz", **seam_cases())
    np.savez_compressed(OUT / "trainer.npz", **trainer_cases())
    np.savez_compressed(OUT / "engine.npz", **engine_cases())
    np.savez_compressed(OUT / "configs.npz", **c1_c3_cases())
    (OUT / "host.json").write_text(json.dumps(host_cases(), indent=0))
    for p in sorted(OUT.glob("*")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
