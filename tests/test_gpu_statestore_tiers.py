"""StateStore capacity tiers: a store whose M x width exceeds
its HBM budget keeps the first clients in the HBM matrix and the rest in a
pinned, device-mapped host tier moved by the same gather/scatter kernels
over the host link.  Semantics are the reference's StateStore
(fedsim/statestore.py:147-210) whatever the tier: rows round-trip bit for
bit, never-saved clients gather the zero default, the FSST files written
from either tier reopen identically, and an engine run is bit-identical to
one with everything in HBM."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import paper_2303_01778_b200 as pb
    return pb


def test_tiers_round_trip_and_disk(pb, tmp_path):
    import torch
    W = 37 * 4 + 2                                   # odd-sized rows (8-byte vector path)
    st = pb.StateStore(tmp_path, persist="none", hbm_bytes=3 * ((W + 3) // 4 * 4) * 4,
                       host_chunk_bytes=4 * ((W + 3) // 4 * 4) * 4)   # 4 rows per host chunk
    st.configure(["a", "b"], [(37, 4), (2,)], capacity=10)
    ids = [11, 3, 42, 7, 19, 5, 23, 8, 1, 30]
    gen = torch.Generator(device="cuda").manual_seed(0)
    work = torch.randn(len(ids), W, generator=gen, device="cuda")
    st.scatter(ids, 0, work)
    assert [st.tier_of(c) for c in ids] == ["hbm"] * 3 + ["host"] * 7
    assert st.hbm_bytes() == 3 * ((W + 3) // 4 * 4) * 4 and st.host_bytes() > 0
    order = [8, 99, 11, 30, 5, 3, 77, 19]            # mixed tiers + never-saved clients
    out = torch.full((len(order), W), 7.0, device="cuda")
    st.gather(order, out)
    want = {c: work[j] for j, c in enumerate(ids)}
    for j, c in enumerate(order):
        exp = want[c] if c in want else torch.zeros(W, device="cuda")
        assert torch.equal(out[j], exp), c
    # reference API on a host-tier client
    got = st.load(30)
    assert got.round_written == 0 and torch.equal(got.payload["a"].reshape(-1), work[9, :148])
    p = {"a": np.full((37, 4), 2.5, dtype=np.float32), "b": np.array([1.0, -1.0], dtype=np.float32)}
    st.save(30, 1, p)
    assert np.array_equal(st.load(30).payload["a"].cpu().numpy(), p["a"])
    # both tiers spill to FSST files that reopen identically
    st.flush_to_disk()
    re = pb.StateStore(tmp_path)
    for j, c in enumerate(ids):
        row = re.load(c)
        flat = np.concatenate([row.payload["a"].cpu().numpy().reshape(-1), row.payload["b"].cpu().numpy()])
        ref = np.concatenate([p["a"].reshape(-1), p["b"]]) if c == 30 else work[j].cpu().numpy()
        assert np.array_equal(flat, ref), c
        assert row.round_written == (1 if c == 30 else 0)


def test_engine_scaffold_tiered_store_bit_identical(pb):
    """C3's shape (SCAFFOLD LR, 1000 clients, 100 per round, K = 8) for three
    rounds with 150 clients' states in HBM and the rest in the host tier vs
    all in HBM: every global tensor bit-identical."""
    ds = pb.generate(60000, 784, 10, seed=0)
    profiles = pb.partition(ds, 1000, pb.PartitionSpec(quantity_skew=0.5, min_samples_per_client=5), seed=0)
    cfg = pb.SimConfig(total_clients=1000, concurrent_clients=100, num_devices=8, total_rounds=3, seed=0,
                       scheme="PARROT")
    outs = []
    for budget in (None, 150 * 7852 * 4):
        store = pb.StateStore(persist="none", hbm_bytes=budget)
        eng = pb.SimulationEngine(cfg, pb.Scaffold(lr=0.05, batch_size=20, client_fraction=0.1), profiles,
                                  pb.make_device_models(8), store=store)
        outs.append(eng.run())
        if budget is not None:
            assert store.host_bytes() > 0 and store.hbm_bytes() <= budget
            tiers = {store.tier_of(c) for c in range(1000)} - {None}
            assert tiers == {"hbm", "host"}
    for a, b in zip(*outs):
        for name in ("weights", "bias", "server_ctrl_weights", "server_ctrl_bias"):
            assert np.array_equal(a.new_global.numpy(name), b.new_global.numpy(name)), (a.round, name)
