"""World-size-2 gloo tests (CPU) of the multi-GPU round plumbing: device
ownership, the packed all-reduce of device partials, Collect gathering,
that every rank derives the identical plan (host-side, bit-exact), and whole
SimulationEngine rounds across ranks on a mocked device layer
(tests/cpu_device.py), stateful clients included."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _partials_for(rank, world, seed=3):
    """Deterministic per-device partials (device k on rank k % world)."""
    from paper_2303_01778_b200.aggregate import DevicePartial, PartialEntry
    from paper_2303_01778_b200.trainer import AggOp
    rng = np.random.default_rng(seed)
    parts = []
    for k in range(4):
        acc = rng.standard_normal((3, 5)).astype(np.float32)
        sa = rng.standard_normal(2).astype(np.float32)
        loss = [(10 * k + j, torch.tensor([float(k + j)])) for j in range(2)]
        p = DevicePartial(device_id=k, entries={
            "w": PartialEntry(AggOp.WEIGHTED_AVERAGE, torch.from_numpy(acc), weight_sum=7.0 + k, count=2),
            "c": PartialEntry(AggOp.SIMPLE_AVERAGE, torch.from_numpy(sa), count=2),
            "local_loss": PartialEntry(AggOp.COLLECT, collected=loss, count=2)},
            clients_folded=[10 * k, 10 * k + 1])
        parts.append(p)
    from paper_2303_01778_b200.distributed import local_devices
    return [parts[k] for k in local_devices(4, world, rank)], parts


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_01778_b200.distributed import allreduce_partials
        from paper_2303_01778_b200.trainer import AggOp
        mine, _ = _partials_for(rank, world)
        schema = [("w", AggOp.WEIGHTED_AVERAGE, (3, 5)), ("c", AggOp.SIMPLE_AVERAGE, (2,)),
                  ("local_loss", AggOp.COLLECT, (1,))]
        assign = {k: [10 * k, 10 * k + 1] for k in range(4)}
        weights = {10 * k + j: 3.5 + 0.5 * k for k in range(4) for j in range(2)}
        got = allreduce_partials(mine, schema, device=torch.device("cpu"),
                                 fold=lambda acc, x: acc.add_(x), assign=assign, weights=weights)
        res = {"w": got.entries["w"].acc.numpy(), "wsum": got.entries["w"].weight_sum,
               "c": got.entries["c"].acc.numpy(), "cnt": got.entries["c"].count,
               "loss": sorted((c, float(t[0])) for c, t in got.entries["local_loss"].collected),
               "clients": sorted(got.clients_folded)}
        # every rank derives the same plan from (seed, round, history)
        from paper_2303_01778_b200.core import ClientSelection, SimConfig, select_clients
        from paper_2303_01778_b200.estimate import WorkloadFit
        from paper_2303_01778_b200.schedule import schedule
        cfg = SimConfig(total_clients=200, concurrent_clients=60, num_devices=4, total_rounds=5)
        sel = select_clients(cfg, 3)
        fits = {k: WorkloadFit(k, 1e-3 * (k + 1), 0.01, 5, 5) for k in range(4)}
        plan = schedule(3, sel, fits, {m: (m % 17) + 3 for m in sel.selected}, cfg)
        res["plan"] = {k: v for k, v in plan.assignments.items()}
        torch.save(res, os.path.join(out_dir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_allreduce_partials_world2(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r0 = torch.load(tmp_path / "rank0.pt", weights_only=False)
    r1 = torch.load(tmp_path / "rank1.pt", weights_only=False)
    _, parts = _partials_for(0, 1)
    want_w = sum(p.entries["w"].acc.numpy().astype(np.float64) for p in parts)
    want_c = sum(p.entries["c"].acc.numpy().astype(np.float64) for p in parts)
    for r in (r0, r1):
        assert np.allclose(r["w"], want_w, atol=1e-5) and np.allclose(r["c"], want_c, atol=1e-5)
        assert r["wsum"] == sum(7.0 + k for k in range(4)) and r["cnt"] == 8
        assert r["loss"] == sorted((10 * k + j, float(k + j)) for k in range(4) for j in range(2))
        assert r["clients"] == sorted(10 * k + j for k in range(4) for j in range(2))
    assert r0["plan"] == r1["plan"]
    assert np.array_equal(r0["w"], r1["w"])  # replicated result


def test_local_devices_partition():
    from paper_2303_01778_b200.distributed import local_devices
    for k in (1, 2, 3, 8, 13):
        for world in (1, 2, 4, 8):
            owned = [local_devices(k, world, r) for r in range(world)]
            flat = sorted(d for o in owned for d in o)
            assert flat == list(range(k))


# ---------------------------------------------------------------------------
# SimulationEngine end to end across 2 ranks (mocked device layer, gloo)
# ---------------------------------------------------------------------------

def _engine_worker(rank, world, port, out_dir, plugin_name):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import cpu_device
    cpu_device.install()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_01778_b200 as pb
        ds = pb.generate(600, 6, 4, seed=9)
        profiles = pb.partition(ds, 30, pb.PartitionSpec(quantity_skew=0.3), seed=9)
        cfg = pb.SimConfig(total_clients=30, concurrent_clients=12, num_devices=4, total_rounds=4,
                           seed=9, scheme="PARROT", scheduling="time-window", time_window=2)
        devs = pb.make_device_models(4, hetero=[0.0, 0.3, 0.6, 0.9], noise=0.05)
        if plugin_name == "scaffold":
            plugin = pb.Scaffold(lr=0.1, batch_size=5, client_fraction=0.5)
            store = pb.StateStore(device=torch.device("cpu"))
        else:
            plugin, store = pb.FedAvg(lr=0.1, batch_size=5, collect_local_loss=True), None
        eng = pb.SimulationEngine(cfg, plugin, profiles, devs, store=store)
        res = {"globals": [], "plans": [], "records": []}
        for oc in eng.run():
            res["globals"].append({n: e.tensor.clone() for n, e in oc.new_global.entries.items()})
            res["records"].append([(x.device_id, x.client_id, x.reported_seconds)
                                   for x in eng.history.round_records(oc.round)])
            res["modes"] = res.get("modes", []) + [oc.scheduling_mode]
        if store is not None:
            res["state"] = {c: store._rows[s].clone() for c, s in store._slot.items()}
            res["rounds"] = dict(store._last_round)
        torch.save(res, os.path.join(out_dir, f"{plugin_name}_w{world}_r{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("plugin_name", ["fedavg", "scaffold"])
def test_engine_rounds_world2_match_world1(tmp_path, plugin_name):
    """SimulationEngine across 2 ranks (devices k % 2 per rank, ONE packed
    all-reduce per round, Collect values in the same buffer, stateful
    clients owned by rank m % 2 and exchanged with all_to_all) equals the
    single-process run: same plans and records (bit-exact), same globals
    (fp32 reassociation tolerance), and the union of the ranks' stores equals
    the single store."""
    for world in (1, 2):
        mp.spawn(_engine_worker, args=(world, _free_port(), str(tmp_path), plugin_name),
                 nprocs=world, join=True)
    one = torch.load(tmp_path / f"{plugin_name}_w1_r0.pt", weights_only=False)
    two = [torch.load(tmp_path / f"{plugin_name}_w2_r{r}.pt", weights_only=False) for r in (0, 1)]
    assert "greedy" in one["modes"]
    for res in two:
        assert res["records"] == one["records"] and res["modes"] == one["modes"]
        for g1, g2 in zip(one["globals"], res["globals"]):
            assert set(g1) == set(g2)
            for name in g1:
                assert torch.allclose(g1[name], g2[name], atol=1e-6, rtol=1e-5), name
    assert all(torch.equal(two[0]["globals"][-1][n], two[1]["globals"][-1][n])
               for n in two[0]["globals"][-1])   # replicated
    if plugin_name == "scaffold":
        merged = {**two[0]["state"], **two[1]["state"]}
        assert set(two[0]["state"]).isdisjoint(two[1]["state"])
        assert all(c % 2 == r for r in (0, 1) for c in two[r]["state"])   # owner = m % world
        assert set(merged) == set(one["state"])
        for c, row in one["state"].items():
            assert torch.allclose(merged[c], row, atol=1e-6), c
        assert {**two[0]["rounds"], **two[1]["rounds"]} == one["rounds"]
