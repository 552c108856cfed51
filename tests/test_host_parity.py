"""Host-side product code vs the reference's own outputs: bit-exact selection,
data generation, partitions, minibatch orders (native PCG64 restatement),
greedy plans (native core), fits, device time model, FSST codec.  CPU only."""

import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

import importlib

from paper_2303_01778_b200 import core, data, estimate, metrics
from paper_2303_01778_b200.core import ClientSelection, ConfigError, SimConfig

ROOT = Path(__file__).resolve().parents[1]
# the package re-exports the schedule() function under the module's name
schedule = importlib.import_module("paper_2303_01778_b200.schedule")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_selection_bit_exact(golden_host):
    for key, want in golden_host["selection"].items():
        seed, m, mp, r = map(int, key.split("/"))
        cfg = SimConfig(total_clients=m, concurrent_clients=mp, num_devices=1,
                        total_rounds=r + 2, seed=seed, scheme="SP")
        assert list(core.select_clients(cfg, r).selected) == want


def test_partition_sizes_bit_exact(golden_host):
    specs = {"c2": (768_400, 3400, data.PartitionSpec(quantity_skew=1.0, min_samples_per_client=10)),
             "c4": (50_000, 1000, data.PartitionSpec(label_skew=0.5, quantity_skew=0.1,
                                                     min_samples_per_client=5))}
    for tag, (n, m, spec) in specs.items():
        got = data.client_sizes(n, m, spec, core.stream_rng(0, core.STREAM_PARTITION))
        assert got.tolist() == golden_host["partition_sizes"][tag]


def test_c1_c3_data_bit_exact(golden_configs):
    ds = data.generate(60000, 784, 10, seed=0)
    assert sha(ds.features) == str(golden_configs["c1/features_sha"][0])
    assert sha(ds.labels) == str(golden_configs["c1/labels_sha"][0])
    ev = data.generate(10000, 784, 10, seed=0, sample_set=1)
    assert sha(ev.features) == str(golden_configs["c1/eval_features_sha"][0])
    prof = data.partition(ds, 100, data.PartitionSpec(), seed=0)
    assert sha(np.concatenate([p.data_partition.indices for p in prof])) == \
        str(golden_configs["c1/partition_sha"][0])
    prof3 = data.partition(ds, 1000, data.PartitionSpec(quantity_skew=0.5, min_samples_per_client=5),
                           seed=0)
    assert [p.sample_count for p in prof3] == golden_configs["c3/sizes"].tolist()
    assert sha(np.concatenate([p.data_partition.indices for p in prof3])) == \
        str(golden_configs["c3/partition_sha"][0])


def test_label_skew_partition_covers():
    ds = data.generate(3000, 4, 5, seed=3)
    prof = data.partition(ds, 50, data.PartitionSpec(label_skew=0.3, quantity_skew=0.5,
                                                     min_samples_per_client=3), seed=3)
    idx = np.sort(np.concatenate([p.data_partition.indices for p in prof]))
    assert np.array_equal(idx, np.arange(3000))
    assert min(p.sample_count for p in prof) >= 3


def test_minibatch_orders_native_bit_exact(golden_host):
    from paper_2303_01778_b200 import _kernels as K
    cases = [tuple(map(int, k.split("/"))) for k in golden_host["minibatch_perms"]]
    keys = np.array([[s, 6, c, r] for s, c, r, _ in cases], dtype=np.uint64)
    n = np.array([c[3] for c in cases])
    base = np.arange(len(cases)) * 10_000
    rows, off = K.minibatch_rows(keys, n, base, epochs=2)
    for i, key in enumerate(golden_host["minibatch_perms"]):
        want = np.concatenate(golden_host["minibatch_perms"][key]) + base[i]
        assert np.array_equal(rows[off[i]: off[i] + 2 * n[i]], want)
    # and against NumPy directly on random keys, including >32-bit seeds
    rng = np.random.default_rng(1)
    keys = np.array([[int(rng.integers(0, 2 ** 63)), 6, int(rng.integers(0, 5000)),
                      int(rng.integers(0, 100))] for _ in range(64)], dtype=np.uint64)
    n = rng.integers(1, 700, 64)
    rows, off = K.minibatch_rows(keys, n, np.zeros(64, np.int64), epochs=3, threads=4)
    for i in range(64):
        g = np.random.default_rng([int(v) for v in keys[i]])
        want = np.concatenate([g.permutation(int(n[i])) for _ in range(3)])
        assert np.array_equal(rows[off[i]: off[i] + 3 * n[i]], want)


def test_greedy_native_and_python_bit_exact(golden_host):
    for case in golden_host["greedy"]:
        sizes = dict(zip(case["ids"], case["sizes"]))
        k = len(case["t"])
        fits = {j: estimate.WorkloadFit(j, case["t"][j], case["b"][j], 2, "all-history")
                for j in range(k)}
        sel = ClientSelection(4, tuple(case["ids"]))
        for jit in (True, False):
            plan = schedule.greedy_assign(4, sel, fits, sizes, k, use_jit=jit)
            assert {str(d): v for d, v in plan.assignments.items()} == case["assign"]
            assert [plan.predicted_loads[j] for j in range(k)] == case["loads"]


def test_greedy_worked_examples_and_opcount():
    fits = {k: estimate.WorkloadFit(k, 1.0, 0.0, 2, "all-history") for k in range(2)}
    sizes = {0: 5, 1: 4, 2: 3, 3: 3, 4: 2}
    plan = schedule.greedy_assign(3, ClientSelection(3, tuple(range(5))), fits, sizes, 2)
    assert plan.assignments == {0: [0, 3], 1: [1, 2, 4]}
    assert plan.predicted_loads == {0: 8.0, 1: 9.0}
    assert schedule.makespan(plan, {0: (1.0, 0.0), 1: (1.0, 0.0)}, sizes) == 9.0
    rng = np.random.default_rng(7)
    for n, k in [(1, 1), (10, 4), (100, 8), (250, 16)]:
        s = -np.sort(-rng.integers(1, 50, size=n).astype(np.float64))
        _, _, ops = schedule.greedy_core_py(s, rng.uniform(0.1, 2.0, k), np.zeros(k))
        assert ops <= 4 * k * n
    clamp = {k: estimate.WorkloadFit(k, 0.001, -10.0, 2, "all-history") for k in range(2)}
    plan = schedule.greedy_assign(2, ClientSelection(2, (0, 1, 2)), clamp, {0: 3, 1: 2, 2: 1}, 2)
    assert plan.assignments == {0: [0, 1, 2], 1: []}


def test_uniform_and_routing(golden_host):
    plan = schedule.uniform_division(0, ClientSelection(0, tuple(range(10, 21))), 4)
    assert {str(k): v for k, v in plan.assignments.items()} == golden_host["uniform_11_4"]
    cfg = SimConfig(total_clients=40, concurrent_clients=12, num_devices=3, total_rounds=10)
    sel = ClientSelection(4, tuple(range(12)))
    fits = {k: estimate.WorkloadFit(k, 1.0, 0.0, 2, "all-history") for k in range(3)}
    sizes = {m: m + 1 for m in range(12)}
    assert schedule.schedule(4, sel, fits, sizes, cfg).mode == schedule.MODE_GREEDY
    assert schedule.schedule(1, sel, fits, sizes, cfg).mode == schedule.MODE_WARMUP
    assert schedule.schedule(4, sel, None, sizes, cfg).mode == schedule.MODE_WARMUP
    partial = dict(fits)
    partial[2] = None
    assert schedule.schedule(4, sel, partial, sizes, cfg).mode == schedule.MODE_WARMUP
    rnd = SimConfig(total_clients=40, concurrent_clients=12, num_devices=3, total_rounds=10,
                    scheduling="random-baseline", seed=9)
    a = schedule.schedule(4, sel, None, sizes, rnd)
    assert a.mode == schedule.MODE_RANDOM and a.assignments == schedule.schedule(4, sel, None, sizes, rnd).assignments


def test_fits_bit_exact(golden_host):
    for case in golden_host["fits"]:
        hist = estimate.TimingHistory()
        for cid, rnd, n, secs in case["records"]:
            hist.add(estimate.TimingRecord(0, int(cid), int(rnd), int(n), float(secs)))
        f = estimate.fit_device(hist, 0, case["window"], 8)
        assert (f.t_sample, f.b, f.records_used, f.degenerate) == \
            (case["t"], case["b"], case["used"], case["degenerate"])
    with pytest.raises(estimate.InsufficientDataError):
        estimate.fit_device(estimate.TimingHistory(), 0, 3, 5)


def test_device_time_model_bit_exact(golden_host):
    from paper_2303_01778_b200.engine import DeviceModel, report_time, virtual_task_seconds
    models = {0: DeviceModel(0), 2: DeviceModel(2, hetero_ratio=0.4, dynamic=True, t_true=2e-4,
                                                b_true=0.01, noise=0.05)}
    for dev, r, cid, v, rep in golden_host["device_times"]:
        d = models[int(dev)]
        got = virtual_task_seconds(d, 123, 42, int(r), int(cid))
        assert got == v and report_time(got, d, int(r), 10) == rep


def test_fsst_codec_bytes(golden_host, golden_configs):
    from paper_2303_01778_b200.statestore import _HEADER, decode_tensor_map, encode_tensor_map
    payload = {"ctrl_weights": np.array([[np.pi, -0.0], [1e-300, np.finfo(np.float64).max]]),
               "ctrl_bias": np.array([2.5, -1.25])}
    blob = encode_tensor_map(payload)
    assert blob.hex() == golden_host["fsst_payload_hex"]
    out, used = decode_tensor_map(blob)
    assert used == len(blob) and np.signbit(out["ctrl_weights"][0, 1])
    # a state file written by the reference decodes here (CRC + header layout)
    raw = golden_configs["c3/state_file_bytes"].tobytes()
    magic, ver, _, cid, rnd, length, crc = _HEADER.unpack(raw[:28])
    import zlib
    assert magic == b"FSST" and ver == 1 and length == len(raw) - 28 and zlib.crc32(raw[28:]) == crc
    dec, _ = decode_tensor_map(raw[28:])
    assert set(dec) == {"ctrl_weights", "ctrl_bias"} and dec["ctrl_weights"].shape == (10, 784)


def test_config_validation():
    base = dict(total_clients=100, concurrent_clients=10, num_devices=4, total_rounds=20, seed=7)
    for bad in [dict(total_clients=0), dict(num_devices=0), dict(warmup_rounds=20), dict(seed=-1),
                dict(seed=2 ** 64), dict(scheme="MPI"), dict(scheduling="greedy"),
                dict(time_window=0), dict(concurrent_clients=101), dict(trip_overhead_seconds=-1)]:
        with pytest.raises(ConfigError):
            SimConfig(**{**base, **bad})
    with pytest.raises(ConfigError, match="max_rounds"):
        SimConfig.from_mapping({**base, "max_rounds": 9})
    with pytest.raises(ConfigError):
        SimConfig(**{**base, "scheme": "SP"})


def test_expected_costs_table():
    want = metrics.expected_costs("PARROT", 100, 10, 4, s_a=80.0)
    assert (want.trips_up, want.bytes_avg_params, want.peak_live_model_replicas) == (4, 320, 4)
    obs = metrics.CostLedger(round=0, scheme="PARROT", trips_up=4, trips_down=4,
                             bytes_avg_params=320)
    assert metrics.reconcile(obs, want).ok


def test_library_exports_every_header_symbol():
    from paper_2303_01778_b200._lib import lib
    header = (ROOT / "include" / "parrot_b200.h").read_text()
    declared = set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    assert declared <= set(lib.exported()), declared - set(lib.exported())
    for name in declared:
        assert hasattr(lib, name)
    assert lib.pb_version() >= 1


def test_abi_struct_layouts_match_bindings():
    """The ctypes argument structs have the C ABI's sizes (a field added on
    one side only would shift every later field)."""
    import ctypes
    from paper_2303_01778_b200._lib import CnnTrainArgs, LazyFoldArgs, LrTrainArgs, ResnetTrainArgs, lib
    out = (ctypes.c_int64 * 4)()
    assert lib.pb_abi_sizes(out, 4) == 4
    want = [ctypes.sizeof(t) for t in (LrTrainArgs, CnnTrainArgs, LazyFoldArgs, ResnetTrainArgs)]
    assert list(out) == want
