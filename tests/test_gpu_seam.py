"""The drop-in seam: ``DeviceWorker.execute_clients`` (fedsim/engine.py:470-503)
driven directly, as the reference's engine and SP path call it, against the
reference's own outputs (tests/golden/seam.npz, make_golden.py:seam_cases),
plus the reference-style plugin path, failure atomicity of a round and the
real-clock timing records.

Tolerances (fp32 device vs float64 reference): partial sums <= 1e-5 of
max|want|; weight sums, counts, fold order and virtual-clock timing records
bit-exact.
"""

import numpy as np
import pytest

from conftest import GOLDEN, rel_gap

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import paper_2303_01778_b200 as pkg
    return pkg


@pytest.fixture(scope="module")
def golden_seam():
    return dict(np.load(GOLDEN / "seam.npz", allow_pickle=False))


def _world(pb):
    ds = pb.generate(240, 4, 3, seed=5)
    profiles = pb.partition(ds, 12, pb.PartitionSpec(), seed=5)
    cfg = pb.SimConfig(total_clients=12, concurrent_clients=6, num_devices=2, total_rounds=4,
                       local_epochs=2, seed=5, scheme="PARROT")
    return profiles, cfg


def _check_partial(part, timings, g, tag):
    assert part.clients_folded == g[f"{tag}/folded"].tolist()
    recs = np.array([[t.device_id, t.client_id, t.round, t.sample_count, t.reported_seconds]
                     for t in timings])
    assert np.array_equal(recs, g[f"{tag}/records"])     # virtual clock: bit-exact
    names = {k.split("/")[3] for k in g if k.startswith(f"{tag}/op/")}
    assert set(part.entries) == names
    for en in names:
        pe = part.entries[en]
        assert pe.op.value == str(g[f"{tag}/op/{en}"][0])
        assert pe.count == int(g[f"{tag}/count/{en}"][0])
        if pe.op.value == "Collect":
            assert [c for c, _ in pe.collected] == g[f"{tag}/collect_ids/{en}"].tolist()
            got = np.stack([t.cpu().double().numpy() for _, t in pe.collected])
            assert rel_gap(got, g[f"{tag}/collect/{en}"]) <= 1e-5, en
        else:
            assert rel_gap(pe.acc.cpu().double().numpy(), g[f"{tag}/acc/{en}"]) <= 1e-5, en
            assert pe.weight_sum == float(g[f"{tag}/wsum/{en}"][0])


def _run_seam(pb, plugin, g, name, tmp_path):
    from paper_2303_01778_b200.engine import DeviceModel, DeviceWorker
    from paper_2303_01778_b200.metrics import ReplicaGauge
    profiles, cfg = _world(pb)
    store = pb.StateStore(tmp_path) if plugin.is_stateful else None   # fresh, never configured
    dev = DeviceModel(1, hetero_ratio=0.3, noise=0.05, t_true=2e-4, b_true=0.01)
    worker = DeviceWorker(dev, cfg, plugin, profiles, store, ReplicaGauge())
    glob = plugin.init_global(pb.ModelParams(g["W0"], g["b0"]))
    if name == "scaffold":
        glob = glob.replaced(server_ctrl_weights=g["ctrl_gw"], server_ctrl_bias=g["ctrl_gb"])
    for row in g["rounds"]:
        r, clients = int(row[0]), [int(c) for c in row[1:]]
        part, timings = worker.execute_clients(glob, clients, r)
        _check_partial(part, timings, g, f"{name}/r{r}")
    return store


@pytest.mark.parametrize("name", ["fedavg", "scaffold"])
def test_device_worker_seam_matches_reference(pb, golden_seam, name, tmp_path):
    """A bare DeviceWorker on a fresh StateStore: two rounds (round 1
    reloads the states round 0 saved) equal the reference worker's partials
    and timing records."""
    plugin = (pb.FedAvg(lr=0.1, batch_size=5, collect_local_loss=True) if name == "fedavg"
              else pb.Scaffold(lr=0.1, batch_size=5, client_fraction=0.5))
    store = _run_seam(pb, plugin, golden_seam, name, tmp_path)
    if store is not None:   # reference durability: one FSST file per trained client
        files = sorted(p.name for p in tmp_path.glob("client_*.state"))
        assert files == [f"client_{c:08d}.state" for c in (1, 2, 3, 7)]


def _ref_style_plugins(pb):
    """Plugins written against the reference's hook API (fedsim/trainer.py:
    172-234): no fused terms, only local_gradient / finalize / server_update."""
    from paper_2303_01778_b200.trainer import AggOp, AlgorithmPlugin, ParamBundle, loss_and_grad

    class MyAvg(AlgorithmPlugin):
        name = "myavg"

        def local_gradient(self, model, xb, yb, ctx):
            return loss_and_grad(model, xb, yb)

        def finalize(self, end_model, steps, ctx, n_samples):
            out = ParamBundle()
            out.add("weights", end_model.weights, AggOp.WEIGHTED_AVERAGE, weight=n_samples)
            out.add("bias", end_model.bias, AggOp.WEIGHTED_AVERAGE, weight=n_samples)
            return out, None

        def server_update(self, old_global, agg):
            return old_global.replaced(weights=agg.bundle.tensor("weights"),
                                       bias=agg.bundle.tensor("bias"))

    class MyScaffold(pb.Scaffold):   # overrides a hook -> runs through the hooks
        def local_gradient(self, model, xb, yb, ctx):
            return super().local_gradient(model, xb, yb, ctx)

    return MyAvg, MyScaffold


def test_reference_style_plugins_run_through_hooks(pb, golden_seam, tmp_path):
    from paper_2303_01778_b200.trainer import uses_hooks
    MyAvg, MyScaffold = _ref_style_plugins(pb)
    avg = MyAvg(lr=0.1, batch_size=5, collect_local_loss=True)
    assert uses_hooks(avg) and not uses_hooks(pb.FedAvg())
    _run_seam(pb, avg, golden_seam, "fedavg", tmp_path / "a")
    sc = MyScaffold(lr=0.1, batch_size=5, client_fraction=0.5)
    assert uses_hooks(sc)
    _run_seam(pb, sc, golden_seam, "scaffold", tmp_path / "s")


def test_plugin_without_hooks_is_rejected(pb):
    from paper_2303_01778_b200.trainer import AlgorithmPlugin, uses_hooks

    class Empty(AlgorithmPlugin):
        name = "empty"

        def server_update(self, old_global, agg):
            return old_global

    with pytest.raises(pb.ConfigError, match="neither the reference hooks"):
        uses_hooks(Empty())


def test_hook_plugin_engine_rounds_match_builtin(pb):
    """Whole engine rounds with a reference-style plugin equal the fused
    built-in (same selection, schedule and folds)."""
    MyAvg, _ = _ref_style_plugins(pb)
    ds = pb.generate(600, 6, 4, seed=9)
    profiles = pb.partition(ds, 30, pb.PartitionSpec(quantity_skew=0.3), seed=9)
    outs = []
    for plugin in (pb.FedAvg(lr=0.1, batch_size=5), MyAvg(lr=0.1, batch_size=5)):
        cfg = pb.SimConfig(total_clients=30, concurrent_clients=12, num_devices=3, total_rounds=3,
                           seed=9, scheme="PARROT")
        eng = pb.SimulationEngine(cfg, plugin, profiles, pb.make_device_models(3))
        outs.append(eng.run())
    for a, b in zip(*outs):
        assert a.device_loads == b.device_loads
        for name in ("weights", "bias"):
            assert rel_gap(b.new_global.numpy(name), a.new_global.numpy(name)) <= 1e-5


def _poisoned_world(pb, bad_client: int):
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    ds = pb.generate(240, 4, 3, seed=5)
    profiles = pb.partition(ds, 12, pb.PartitionSpec(), seed=5)
    p = profiles[bad_client]
    X = np.array(p.data_partition.features, copy=True)
    X[0, 0] = np.nan
    profiles[bad_client] = ClientProfile(p.client_id, p.sample_count,
                                         DataSlice(X, p.data_partition.labels, p.data_partition.indices))
    return profiles


@pytest.mark.parametrize("stateful", [False, True])
def test_failed_round_leaves_engine_untouched(pb, tmp_path, stateful):
    """A diverged client raises DeviceFailureError (fedsim/engine.py:645-650)
    before anything is committed: global model, timing history and client
    states are those of before the round, so the round can be retried."""
    from paper_2303_01778_b200.engine import DeviceFailureError
    profiles = _poisoned_world(pb, 4)
    cfg = pb.SimConfig(total_clients=12, concurrent_clients=12, num_devices=2, total_rounds=3,
                       seed=5, scheme="PARROT")
    plugin = pb.Scaffold(lr=0.1, batch_size=5) if stateful else pb.FedAvg(lr=0.1, batch_size=5)
    store = pb.StateStore(tmp_path) if stateful else None
    eng = pb.SimulationEngine(cfg, plugin, profiles, pb.make_device_models(2), store=store)
    before = {n: eng.global_bundle.numpy(n) for n in eng.global_bundle.entries}
    with pytest.raises(DeviceFailureError, match="client 4 round 0"):
        eng.run_round(0)
    assert eng.history.size == 0 and not eng.history.round_records(0)
    for n, v in before.items():
        assert np.array_equal(eng.global_bundle.numpy(n), v)
    if stateful:
        assert not list(tmp_path.glob("client_*.state"))
        assert store.stats().saves == 0
    with pytest.raises(DeviceFailureError):   # retrying fails the same way, no StaleWriteError
        eng.run_round(0)


@pytest.mark.parametrize("model", ["lr", "cnn"])
def test_real_clock_records_are_device_measured(pb, model):
    """clock='real': every client's record is its own device-measured task
    time (kernel %globaltimer stamps), so the per-device OLS sees seconds
    that grow with the sample count, and the clients' times add up to the
    group's device time (sweep models)."""
    sizes_seed = 13
    if model == "lr":
        ds = pb.generate(6000, 64, 10, seed=sizes_seed)
        m, mp = 40, 20
    else:
        rng = np.random.default_rng(sizes_seed)
        means = rng.standard_normal((62, 784))
        means *= 3.0 / np.linalg.norm(means, axis=1, keepdims=True)
        labels = np.arange(2400) % 62
        ds = pb.SyntheticDataset(means[labels] + rng.standard_normal((2400, 784)), labels, 62, 784,
                                 3.0, 1.0)
        m, mp = 40, 20
    profiles = pb.partition(ds, m, pb.PartitionSpec(quantity_skew=0.5, min_samples_per_client=5),
                            seed=sizes_seed)
    cfg = pb.SimConfig(total_clients=m, concurrent_clients=mp, num_devices=2, total_rounds=4,
                       seed=sizes_seed, scheme="PARROT", clock="real", scheduling="full-history")
    eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=0.05, batch_size=20), profiles,
                              pb.make_device_models(2, hetero=[0.0, 0.5]), model=model)
    outs = eng.run()
    for oc in outs:
        recs = eng.history.round_records(oc.round)
        n = np.array([r.sample_count for r in recs], dtype=float)
        secs = np.array([r.reported_seconds / (1.5 if r.device_id == 1 else 1.0) for r in recs])
        assert np.corrcoef(n, secs)[0, 1] > 0.5               # time grows with the work
        if model == "lr":   # each client's own CTA span: (nearly) all distinct
            assert len(set(secs.tolist())) > len(secs) // 2
        else:   # sweep shares: a strictly increasing function of the step count
            steps = np.ceil(n / 20).astype(int)
            by_steps = {k: set(np.round(secs[steps == k], 12).tolist()) for k in set(steps.tolist())}
            assert all(len(v) == 1 for v in by_steps.values())
            vals = [by_steps[k].pop() for k in sorted(by_steps)]
            assert all(b > a for a, b in zip(vals, vals[1:]))
            # the sweeps are the group's launch minus its set-up / wind-down
            assert 0.7 * oc.device_seconds <= secs.sum() <= oc.device_seconds
    from paper_2303_01778_b200.estimate import fit_device
    fit = fit_device(eng.history, 0, "all-history", 3)
    assert fit.t_sample > 0 and not fit.degenerate
    assert outs[-1].scheduling_mode == "greedy"
