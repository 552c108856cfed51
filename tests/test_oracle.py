"""Pin the CPU oracle (oracle/fedsim_oracle.py) to the reference's own outputs
(tests/golden/*, produced by tests/golden/make_golden.py from /root/reference).
CPU only."""

import numpy as np
import pytest

from conftest import rel_gap
from oracle import fedsim_oracle as O
from paper_2303_01778_b200.data import PartitionSpec, generate, partition

PLUGINS = {
    "fedavg": dict(lr=0.1, batch_size=8, collect_local_loss=True),
    "fedprox": dict(mu=0.3, lr=0.1, batch_size=8, collect_local_loss=True),
    "fednova": dict(lr=0.1, batch_size=8),
    "scaffold": dict(lr=0.1, batch_size=8, client_fraction=0.5),
    "feddyn": dict(alpha=0.2, lr=0.1, batch_size=8),
}


def _glob_for(algo, g):
    glob = algo.init_global(g["W0"], g["b0"])
    state = None
    if algo.name == "scaffold":
        glob["server_ctrl_weights"] = (g["ctrl_gw"], O.SUM)
        glob["server_ctrl_bias"] = (g["ctrl_gb"], O.SUM)
        state = {"ctrl_weights": g["state_w"], "ctrl_bias": g["state_b"]}
    if algo.name == "feddyn":
        state = {"grad_corr_weights": g["state_w"], "grad_corr_bias": g["state_b"]}
    return glob, state


@pytest.mark.parametrize("name", sorted(PLUGINS))
def test_oracle_client_train_matches_reference(name, golden_trainer):
    g = golden_trainer
    algo = O.Algo(name, **PLUGINS[name])
    glob, state = _glob_for(algo, g)
    res, new_state, steps, _ = O.train_client(algo, g["X"], g["y"], 5, glob, state, epochs=2,
                                              batch_size=8, lr=0.1, seed=9, rnd=3)
    assert steps == 2 * int(np.ceil(len(g["y"]) / 8))
    keys = {k.split("/")[2] for k in g if k.startswith(f"{name}/res/")}
    assert keys == set(res)
    for k in keys:
        assert rel_gap(res[k][0], g[f"{name}/res/{k}"]) <= 1e-12, k
        assert res[k][2] == pytest.approx(float(g[f"{name}/w/{k}"][0]))
    if new_state is not None:
        for k, v in new_state.items():
            assert rel_gap(v, g[f"{name}/state/{k}"]) <= 1e-12, k


def test_oracle_fold_worked_examples():
    # tests/test_aggregate.py:67-73 and :93-100 of the reference
    p = O.new_partial()
    O.fold_into(p, {"x": (np.array([1.0, 2.0]), O.WA, 1.0, None)}, 0)
    O.fold_into(p, {"x": (np.array([3.0, 4.0]), O.WA, 3.0, None)}, 1)
    assert np.allclose(p["entries"]["x"]["acc"], [10.0, 14.0]) and p["entries"]["x"]["wsum"] == 4.0
    p1, p2 = O.new_partial(), O.new_partial()
    O.fold_into(p1, {"x": (np.array([1.0, 2.0]), O.WA, 1.0, None)}, 0)
    O.fold_into(p2, {"x": (np.array([3.0, 4.0]), O.WA, 3.0, None)}, 1)
    t, _, w, _, clients = O.combine([p1, p2])
    assert np.allclose(t["x"], [2.5, 3.5]) and w["x"] == 4.0 and clients == (0, 1)
    a, b = O.new_partial(), O.new_partial()
    O.fold_into(a, {"s": (np.array([2.0]), O.SA, 1.0, None)}, 0)
    O.fold_into(a, {"s": (np.array([4.0]), O.SA, 1.0, None)}, 1)
    O.fold_into(b, {"s": (np.array([9.0]), O.SA, 1.0, None)}, 2)
    assert np.allclose(O.combine([a, b, O.new_partial()])[0]["s"], [5.0])
    with pytest.raises(ValueError):
        O.combine([O.new_partial()])


def test_oracle_greedy_matches_reference(golden_host):
    for case in golden_host["greedy"]:
        sizes = dict(zip(case["ids"], case["sizes"]))
        plan, loads = O.greedy_plan(sizes, case["ids"], case["t"], case["b"])
        assert {str(k): v for k, v in plan.items()} == case["assign"]
        assert loads == case["loads"]


def test_oracle_selection_and_perms(golden_host):
    for key, want in golden_host["selection"].items():
        seed, m, mp, r = map(int, key.split("/"))
        assert O.selection(seed, m, mp, r) == want
    for key, want in golden_host["minibatch_perms"].items():
        seed, cid, r, n = map(int, key.split("/"))
        got = O.minibatch_orders(seed, cid, r, n, 2)
        assert [list(map(int, p)) for p in got] == want


def test_oracle_fits(golden_host):
    for case in golden_host["fits"]:
        recs = np.array(case["records"])
        lo = 0 if case["window"] == "all-history" else 8 - case["window"]
        sel = recs[(recs[:, 1] >= lo) & (recs[:, 1] <= 7)]
        t, b = O.ols_fit(sel[:, 2], sel[:, 3])
        assert t == case["t"] and b == case["b"]


def _run_oracle_rounds(algo, profiles, seed, total, per_round, rounds, epochs):
    data = {p.client_id: (p.data_partition.features, p.data_partition.labels) for p in profiles}
    f = profiles[0].data_partition.features.shape[1]
    c = 1 + max(int(p.data_partition.labels.max()) for p in profiles)
    glob = algo.init_global(np.zeros((c, f)), np.zeros(c))
    states, out = {}, []
    for r in range(rounds):
        glob, _ = O.sp_round(algo, data, glob, states, seed, r, total, per_round, epochs)
        out.append(glob)
    return out


def test_oracle_sp_rounds_match_reference_engine(golden_engine):
    ds = generate(1200, 6, 4, seed=11)
    profiles = partition(ds, 40, PartitionSpec(), seed=11)
    per_round = _run_oracle_rounds(O.Algo("fedavg", lr=0.1), profiles, 11, 40, 20, 6, 1)
    for r, glob in enumerate(per_round):
        for scheme in ("SP", "PARROT"):
            assert rel_gap(glob["weights"][0], golden_engine[f"c02_{scheme}/r{r}/weights"]) <= 1e-12
            assert rel_gap(glob["bias"][0], golden_engine[f"c02_{scheme}/r{r}/bias"]) <= 1e-12


@pytest.mark.parametrize("name,hyper", [
    ("fedprox", dict(mu=0.1, lr=0.1, batch_size=5)),
    ("fednova", dict(lr=0.1, batch_size=7)),
    ("scaffold", dict(lr=0.1, batch_size=5, client_fraction=0.5)),
    ("feddyn", dict(alpha=0.1, lr=0.1, batch_size=5)),
])
def test_oracle_plugin_rounds_match_reference_engine(name, hyper, golden_engine):
    ds = generate(240, 4, 3, seed=5)
    profiles = partition(ds, 12, PartitionSpec(), seed=5)
    per_round = _run_oracle_rounds(O.Algo(name, **hyper), profiles, 5, 12, 6, 4, 2)
    for r, glob in enumerate(per_round):
        for entry, (tensor, _) in glob.items():
            assert rel_gap(tensor, golden_engine[f"small_{name}/r{r}/{entry}"]) <= 1e-10, (r, entry)


def test_resnet_spec_matches_oracle_layout():
    """ResNet-18-GN (config 4): P = 11,173,962 at 10 classes; the product's
    flat layout equals the oracle's; the library's workspace planner agrees
    with the model size (host-only call)."""
    from oracle import resnet_oracle as R
    from paper_2303_01778_b200.models import resnet_init, resnet_spec
    spec = resnet_spec(10)
    assert spec.numel == 11_173_962
    assert [(n, tuple(sh)) for n, _, _, sh in spec.columns()] == [(n, tuple(sh)) for n, sh in R.layout(10)]
    w = resnet_init(spec, 0)
    for n, o, s, _ in spec.columns():
        if "gn" in n:
            assert np.all(w[o:o + s] == (1.0 if n.endswith("_w") else 0.0))
    p = R.unflatten(w, 10)
    assert np.array_equal(R.flatten(p, 10), w.astype(np.float64))


def test_resnet_workspace_plan_host_only():
    from paper_2303_01778_b200.resnet import workspace_sizes
    arena, p16, part, gnp = workspace_sizes(20, 10)
    # bf16 copies: every conv weight with the stem's 3 input channels padded to 8
    assert p16 >= 11_173_962 - 5130 - 2 * 4800  # conv weights only (no fc, no GN affine)
    assert arena > 0 and part > 0 and gnp > 0
