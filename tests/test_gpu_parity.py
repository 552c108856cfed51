"""End-to-end parity of the CUDA path (through libparrot_b200's C ABI) with the
reference's own outputs (tests/golden, produced by the reference) and the
CPU oracle.  Tolerances (fp32 device path vs the float64 reference):

* model tensors: max|got - want| / max|want| <= 1e-5 per round for LR
  (SURVEY.md §7 "fp32 vs f64"), 1e-4 for multi-round stateful runs;
* schedules, selections, timing records, device loads: bit-exact;
* eval accuracy: within 1 sample; eval loss: abs <= 1e-5.
"""

import numpy as np
import pytest

from conftest import rel_gap

pytestmark = pytest.mark.gpu

PLUGIN_HYPER = {
    "fedavg": dict(lr=0.1, batch_size=8, collect_local_loss=True),
    "fedprox": dict(mu=0.3, lr=0.1, batch_size=8, collect_local_loss=True),
    "fednova": dict(lr=0.1, batch_size=8),
    "scaffold": dict(lr=0.1, batch_size=8, client_fraction=0.5),
    "feddyn": dict(alpha=0.2, lr=0.1, batch_size=8),
}


@pytest.fixture(scope="module")
def pb():
    import paper_2303_01778_b200 as pkg
    return pkg


@pytest.mark.parametrize("name", sorted(PLUGIN_HYPER))
def test_client_execute_matches_reference(pb, name, golden_trainer):
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    from paper_2303_01778_b200.statestore import ClientState
    g = golden_trainer
    plugin = pb.make_plugin(name, **PLUGIN_HYPER[name])
    glob = plugin.init_global(pb.ModelParams(g["W0"], g["b0"]))
    state = None
    if name == "scaffold":
        glob = glob.replaced(server_ctrl_weights=g["ctrl_gw"], server_ctrl_bias=g["ctrl_gb"])
        state = ClientState(5, 0, {"ctrl_weights": g["state_w"], "ctrl_bias": g["state_b"]})
    if name == "feddyn":
        state = ClientState(5, 0, {"grad_corr_weights": g["state_w"], "grad_corr_bias": g["state_b"]})
    prof = ClientProfile(5, len(g["y"]), DataSlice(g["X"], g["y"], np.arange(len(g["y"]))))
    rep = pb.client_execute(plugin, prof, glob, state, epochs=2, batch_size=8, lr=0.1, seed=9,
                            round_num=3)
    want = {k.split("/")[2] for k in g if k.startswith(f"{name}/res/")}
    assert set(rep.client_result.entries) == want
    for k in want:
        e = rep.client_result.entries[k]
        assert rel_gap(rep.client_result.numpy(k), g[f"{name}/res/{k}"]) <= 1e-5, k
        assert e.weight == pytest.approx(float(g[f"{name}/w/{k}"][0]))
    if rep.new_state is not None:
        assert rep.new_state.round_written == 3
        for k, v in rep.new_state.payload.items():
            assert rel_gap(v.cpu().numpy(), g[f"{name}/state/{k}"]) <= 1e-5, k
    if name == "fedavg":
        assert rep.client_result.entries["local_loss"].client_id == 5
    assert rep.samples_processed == 2 * len(g["y"]) and rep.measured_seconds > 0


def test_fedprox_zero_mu_is_fedavg_bitwise(pb, golden_trainer):
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    g = golden_trainer
    prof = ClientProfile(2, len(g["y"]), DataSlice(g["X"], g["y"], np.arange(len(g["y"]))))
    outs = []
    for plugin in (pb.FedAvg(lr=0.1), pb.FedProx(mu=0.0, lr=0.1)):
        glob = plugin.init_global(pb.ModelParams(g["W0"], g["b0"]))
        outs.append(pb.client_execute(plugin, prof, glob, None, 3, 8, 0.1, 7, 1).client_result)
    for k in ("weights", "bias"):
        assert np.array_equal(outs[0].numpy(k), outs[1].numpy(k))


def test_non_finite_loss_raises(pb):
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    from paper_2303_01778_b200.trainer import NonFiniteLossError
    rng = np.random.default_rng(0)
    X = rng.standard_normal((10, 3))
    X[4, 1] = np.nan
    y = np.array([0, 1, 2, 0, 1, 2, 0, 1, 2, 0])
    plugin = pb.FedAvg(lr=0.1)
    glob = plugin.init_global(pb.ModelParams(np.zeros((3, 3)), np.zeros(3)))
    with pytest.raises(NonFiniteLossError, match="client 0 round 2"):
        pb.client_execute(plugin, pb.ClientProfile(0, 10, pb.DataSlice(X, y, np.arange(10))),
                          glob, None, 1, 0, 0.1, seed=1, round_num=2)


def test_local_and_group_fold_examples(pb):
    from paper_2303_01778_b200.aggregate import EmptyAggregateError, OpMismatchError
    from paper_2303_01778_b200.trainer import AggOp, ParamBundle

    def wa(x, w):
        return ParamBundle().add("x", np.asarray(x, float), AggOp.WEIGHTED_AVERAGE, weight=w)

    p = pb.DevicePartial(0)
    pb.local_fold(p, wa([1.0, 2.0], 1.0), 0)
    pb.local_fold(p, wa([3.0, 4.0], 3.0), 1)
    assert np.allclose(p.entries["x"].acc.cpu().numpy(), [10.0, 14.0])
    assert p.entries["x"].weight_sum == 4.0
    p1 = pb.local_fold(pb.DevicePartial(0), wa([1.0, 2.0], 1.0), 0)
    p2 = pb.local_fold(pb.DevicePartial(1), wa([3.0, 4.0], 3.0), 1)
    agg = pb.global_fold([p1, p2, pb.DevicePartial(2)])
    assert np.allclose(agg.bundle.numpy("x"), [2.5, 3.5]) and agg.clients == (0, 1)
    with pytest.raises(OpMismatchError):
        pb.local_fold(p1, ParamBundle().add("x", np.ones(2), AggOp.SUM), 2)
    with pytest.raises(EmptyAggregateError):
        pb.global_fold([pb.DevicePartial(0)])


def test_hierarchy_invariance_random_groupings(pb):
    from paper_2303_01778_b200.trainer import AggOp, ParamBundle
    rng = np.random.default_rng(101)
    results = []
    for cid in range(100):
        b = ParamBundle()
        b.add("weights", rng.standard_normal((3, 4)), AggOp.WEIGHTED_AVERAGE,
              weight=float(rng.integers(1, 50)))
        b.add("scale", rng.standard_normal(1), AggOp.SUM)
        b.add("ctrl", rng.standard_normal(2), AggOp.SIMPLE_AVERAGE)
        b.add("tag", rng.standard_normal(1), AggOp.COLLECT, client_id=cid)
        results.append((cid, b))
    flat = pb.flat_aggregate(results)
    for groups in range(1, 11):
        partials = []
        for g, chunk in enumerate(np.array_split(np.arange(100), groups)):
            part = pb.DevicePartial(g)
            for i in chunk:
                pb.local_fold(part, results[i][1], results[i][0])
            partials.append(part)
        agg = pb.global_fold(partials)
        for name in ("weights", "scale", "ctrl"):
            assert rel_gap(agg.bundle.numpy(name), flat.bundle.numpy(name)) <= 1e-5
        assert sorted(c for c, _ in agg.collected["tag"]) == list(range(100))


def _engine(pb, scheme, k, profiles, rounds, seed, m_p, plugin, **kw):
    cfg = pb.SimConfig(total_clients=len(profiles), concurrent_clients=m_p, num_devices=k,
                       total_rounds=rounds, seed=seed, scheme=scheme,
                       **{x: kw.pop(x) for x in list(kw) if x in ("local_epochs", "scheduling",
                                                                   "time_window")})
    dev_kw = kw.pop("device_kw", {})
    return pb.SimulationEngine(cfg, plugin, profiles, pb.make_device_models(k, **dev_kw), **kw)


@pytest.mark.parametrize("scheme,k", [("SP", 1), ("PARROT", 4), ("SD_DIST", 20), ("FA_DIST", 4)])
def test_engine_c02_per_round_globals(pb, scheme, k, golden_engine):
    ds = pb.generate(1200, 6, 4, seed=11)
    profiles = pb.partition(ds, 40, pb.PartitionSpec(), seed=11)
    eng = _engine(pb, scheme, k, profiles, 6, 11, 20, pb.FedAvg(lr=0.1))
    outs = eng.run()
    for oc in outs:
        r = oc.round
        for name in ("weights", "bias"):
            assert rel_gap(oc.new_global.numpy(name), golden_engine[f"c02_SP/r{r}/{name}"]) <= 1e-5
        if scheme in ("SP", "PARROT"):
            want_loads = golden_engine[f"c02_{scheme}/r{r}/loads"]
            assert [oc.device_loads[d] for d in sorted(oc.device_loads)] == want_loads.tolist()
            assert oc.scheduling_mode == str(golden_engine[f"c02_{scheme}/r{r}/mode"][0])
            costs = golden_engine[f"c02_{scheme}/r{r}/costs"].tolist()
            assert [oc.costs.trips_up, oc.costs.trips_down, oc.costs.bytes_avg_params,
                    oc.costs.bytes_special_params] == costs


def test_engine_hetero_greedy_bit_exact_schedule(pb, golden_engine):
    ds = pb.generate(3000, 4, 2, seed=3)
    profiles = pb.partition(ds, 100, pb.PartitionSpec(quantity_skew=0.3), seed=3)
    eng = _engine(pb, "PARROT", 3, profiles, 6, 3, 40, pb.FedAvg(lr=0.1, batch_size=10),
                  scheduling="time-window", time_window=3,
                  device_kw=dict(hetero=[0.0, 0.5, 1.0], noise=0.05, b_true=0.01))
    for oc in eng.run():
        r = oc.round
        assert oc.scheduling_mode == str(golden_engine[f"hetero/r{r}/mode"][0])
        assert [oc.device_loads[d] for d in range(3)] == golden_engine[f"hetero/r{r}/loads"].tolist()
        recs = np.array([[x.device_id, x.client_id, x.sample_count, x.reported_seconds]
                         for x in eng.history.round_records(r)])
        assert np.array_equal(recs, golden_engine[f"hetero/r{r}/records"])
        for name in ("weights", "bias"):
            assert rel_gap(oc.new_global.numpy(name), golden_engine[f"hetero/r{r}/{name}"]) <= 1e-5


@pytest.mark.parametrize("name,hyper", [
    ("fedprox", dict(mu=0.1, lr=0.1, batch_size=5)),
    ("fednova", dict(lr=0.1, batch_size=7)),
    ("scaffold", dict(lr=0.1, batch_size=5, client_fraction=0.5)),
    ("feddyn", dict(alpha=0.1, lr=0.1, batch_size=5)),
])
def test_engine_plugins_small_world(pb, name, hyper, golden_engine, tmp_path):
    ds = pb.generate(240, 4, 3, seed=5)
    profiles = pb.partition(ds, 12, pb.PartitionSpec(), seed=5)
    eval_ds = pb.generate(120, 4, 3, seed=5, sample_set=1)
    plugin = pb.make_plugin(name, **hyper)
    store = pb.StateStore(tmp_path / "st") if plugin.is_stateful else None
    eng = _engine(pb, "PARROT", 2, profiles, 4, 5, 6, plugin, local_epochs=2, store=store,
                  eval_data=eval_ds)
    for oc in eng.run():
        r = oc.round
        for entry, e in oc.new_global.entries.items():
            assert rel_gap(oc.new_global.numpy(entry), golden_engine[f"small_{name}/r{r}/{entry}"]) \
                <= 1e-4, (r, entry)
        acc, loss = golden_engine[f"small_{name}/r{r}/acc_loss"]
        assert abs(oc.accuracy - acc) <= 1.0 / 120 + 1e-12 and abs(oc.loss - loss) <= 1e-4
    if store is not None:
        assert store.stats().bytes_on_disk > 0 and store.stats().saves > 0


def test_engine_c1_lr_784x10(pb, golden_configs):
    ds = pb.generate(60000, 784, 10, seed=0)
    ev = pb.generate(10000, 784, 10, seed=0, sample_set=1)
    profiles = pb.partition(ds, 100, pb.PartitionSpec(), seed=0)
    eng = _engine(pb, "SP", 1, profiles, 3, 0, 10, pb.FedAvg(lr=0.1, batch_size=20), eval_data=ev)
    for oc in eng.run():
        r = oc.round
        for name in ("weights", "bias"):
            assert rel_gap(oc.new_global.numpy(name), golden_configs[f"c1/r{r}/{name}"]) <= 1e-5
        acc, loss = golden_configs[f"c1/r{r}/acc_loss"]
        assert abs(oc.accuracy - acc) <= 1.0 / 10000 + 1e-12
        assert abs(oc.loss - loss) <= 1e-5


def test_engine_c3_scaffold_1000_clients_k8(pb, golden_configs, tmp_path):
    ds = pb.generate(60000, 784, 10, seed=0)
    ev = pb.generate(10000, 784, 10, seed=0, sample_set=1)
    profiles = pb.partition(ds, 1000, pb.PartitionSpec(quantity_skew=0.5, min_samples_per_client=5),
                            seed=0)
    store = pb.StateStore(tmp_path / "c3", persist="async")
    eng = _engine(pb, "PARROT", 8, profiles, 3, 0, 100,
                  pb.Scaffold(lr=0.05, batch_size=20, client_fraction=0.1), store=store,
                  eval_data=ev, device_kw=dict(hetero=[0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7]))
    for oc in eng.run():
        r = oc.round
        want_loads = golden_configs[f"c3/r{r}/loads"]
        assert [oc.device_loads[d] for d in range(8)] == want_loads.tolist()
        for name in ("weights", "bias", "server_ctrl_weights", "server_ctrl_bias"):
            assert rel_gap(oc.new_global.numpy(name), golden_configs[f"c3/r{r}/{name}"]) <= 1e-4, name
        acc, _ = golden_configs[f"c3/r{r}/acc_loss"]
        assert abs(oc.accuracy - acc) <= 2.0 / 10000 + 1e-12
    # a state file written here has the reference's layout and round
    name = str(golden_configs["c3/state_file_name"][0])
    raw = (tmp_path / "c3" / name).read_bytes()
    ref = golden_configs["c3/state_file_bytes"].tobytes()
    assert raw[:8] == ref[:8] and raw[8:16] == ref[8:16] and len(raw) == len(ref)
    from paper_2303_01778_b200.statestore import decode_tensor_map
    got, _ = decode_tensor_map(raw[28:])
    want, _ = decode_tensor_map(ref[28:])
    for k in want:
        assert rel_gap(got[k], want[k]) <= 1e-4


def test_engine_bit_reproducible_and_resume(pb):
    ds = pb.generate(240, 4, 3, seed=5)
    profiles = pb.partition(ds, 12, pb.PartitionSpec(), seed=5)
    a = _engine(pb, "PARROT", 3, profiles, 6, 5, 6, pb.FedAvg(lr=0.1))
    b = _engine(pb, "PARROT", 3, profiles, 6, 5, 6, pb.FedAvg(lr=0.1))
    a.run()
    b.run(rounds=3)
    c = pb.SimulationEngine(b.cfg, pb.FedAvg(lr=0.1), profiles, pb.make_device_models(3),
                            start_round=3, initial_global=b.global_bundle, history=b.history)
    c.run()
    for name in ("weights", "bias"):
        assert np.array_equal(a.global_bundle.numpy(name), c.global_bundle.numpy(name))


def test_engine_device_failure(pb):
    ds = pb.generate(240, 4, 3, seed=5)
    profiles = list(pb.partition(ds, 12, pb.PartitionSpec(), seed=5))
    bad = profiles[3].data_partition.features.copy()
    bad[0, 0] = np.nan
    profiles[3] = pb.ClientProfile(3, profiles[3].sample_count,
                                   pb.DataSlice(bad, profiles[3].data_partition.labels,
                                                profiles[3].data_partition.indices))
    from paper_2303_01778_b200.engine import DeviceFailureError
    eng = _engine(pb, "PARROT", 2, profiles, 2, 5, 12, pb.FedAvg(lr=0.1))
    with pytest.raises(DeviceFailureError, match="device .* failed"):
        eng.run()


def test_statestore_device_semantics(pb, tmp_path):
    import torch
    from paper_2303_01778_b200.statestore import CorruptRecordError, StaleWriteError
    st = pb.StateStore(tmp_path)
    assert st.load(3) is None
    d = st.load(3, default_factory=lambda: {"w": np.zeros((3, 4)), "b": np.zeros(3)})
    assert d.round_written == -1
    p = {"w": np.random.default_rng(1).standard_normal((3, 4)).astype(np.float32),
         "b": np.arange(3, dtype=np.float32)}
    st.save(7, 3, p)
    got = st.load(7)
    assert got.round_written == 3 and np.array_equal(got.payload["w"].cpu().numpy(), p["w"])
    with pytest.raises(StaleWriteError):
        st.save(7, 3, p)
    st.save(7, 5, p)
    re = pb.StateStore(tmp_path)
    with pytest.raises(StaleWriteError):
        re.save(7, 5, p)
    assert np.array_equal(re.load(7).payload["w"].cpu().numpy(), p["w"])
    # group gather/scatter with defaults for never-saved clients
    work = torch.full((2, 15), 5.0, device="cuda")
    re.gather([7, 99], work)
    assert np.array_equal(work[0, :12].cpu().numpy().reshape(3, 4), p["w"])
    assert not work[1].any().item()
    path = tmp_path / "client_00000007.state"
    raw = bytearray(path.read_bytes())
    raw[-1] ^= 0xFF
    path.write_bytes(raw)
    with pytest.raises(CorruptRecordError):
        pb.StateStore(tmp_path).load(7)


def test_counters_and_replicas(pb):
    ds = pb.generate(240, 4, 3, seed=5)
    profiles = pb.partition(ds, 12, pb.PartitionSpec(), seed=5)
    eng = _engine(pb, "PARROT", 2, profiles, 3, 5, 6, pb.FedAvg(lr=0.1))
    for oc in eng.run():
        assert oc.costs.trips_up == 2 and oc.costs.trips_down == 2
        assert oc.costs.bytes_avg_params == 2 * 8 * (3 * 4 + 3)
        # one replica per busy simulated device (the reference's Table-1
        # bound, so reconcile() passes); the six clients of the round train
        # concurrently in one batched launch
        assert oc.costs.peak_live_model_replicas == 2
        assert oc.costs.peak_device_batch == 6
        want = pb.expected_costs("PARROT", 12, 6, 2, s_a=8 * 15)
        assert pb.reconcile(oc.costs, want).ok


def test_engine_prefetch_matches_sequential(pb):
    """run_round prepares round r+1 on a helper thread while round r runs:
    globals, loads and the timing history equal the sequential
    prepare/execute path, and an unconsumed prefetch leaves no records."""
    ds = pb.generate(600, 6, 4, seed=9)
    profiles = pb.partition(ds, 30, pb.PartitionSpec(quantity_skew=0.3), seed=9)
    kw = dict(scheduling="time-window", time_window=2,
              device_kw=dict(hetero=[0.0, 0.4, 0.8], noise=0.05))
    a = _engine(pb, "PARROT", 3, profiles, 6, 9, 12, pb.FedAvg(lr=0.1, batch_size=5), **dict(kw))
    b = _engine(pb, "PARROT", 3, profiles, 6, 9, 12, pb.FedAvg(lr=0.1, batch_size=5), **dict(kw))
    outs_a = a.run(rounds=4)
    outs_b = [b.execute_round(b.prepare_round(r)) for r in range(4)]
    for oa, ob in zip(outs_a, outs_b):
        assert oa.device_loads == ob.device_loads and oa.scheduling_mode == ob.scheduling_mode
        for name in ("weights", "bias"):
            assert np.array_equal(oa.new_global.numpy(name), ob.new_global.numpy(name))
    assert a.history.size == b.history.size and not a.history.round_records(4)
    for r in range(4):
        ra = [(x.device_id, x.client_id, x.reported_seconds) for x in a.history.round_records(r)]
        rb = [(x.device_id, x.client_id, x.reported_seconds) for x in b.history.round_records(r)]
        assert ra == rb
