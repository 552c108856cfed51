"""CNN path (BASELINE config 2 model) on the GPU vs the torch-CPU float64
restatement (oracle/cnn_oracle.py).  Restatement-pinned: the reference has no
CNN.  The device feeds bf16 operands to its tcgen05 conv2 GEMMs (fp32
accumulation in TMEM; everything else fp32), so parity is checked in two
layers (SURVEY.md §7 "fp32 vs f64"):

1. kernel arithmetic -- against the oracle with the SAME bf16 operand
   rounding (``emulate_bf16``): per-tensor update error
   ||dW_gpu - dW_ref|| / ||dW_ref|| <= 2e-2 and local loss within 1e-3
   relative, over several local steps;
2. training outcome -- against the exact float64 oracle at the FL-round
   level: per-round eval accuracy within 1 point, eval loss within 1 %
   relative, global weights within 5e-3 of ||W|| (bf16 perturbs each local
   update by a few percent; it does not change the curve).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spec():
    from paper_2303_01778_b200.models import cnn_spec
    return cnn_spec(62)


@pytest.fixture(scope="module")
def femnist_like():
    from paper_2303_01778_b200.data import generate
    return generate(4000, 784, 62, seed=0)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("n,bs,epochs", [(20, 20, 1), (57, 20, 2), (7, 20, 1), (45, 16, 1)])
def test_cnn_client_kernel_arithmetic(spec, femnist_like, n, bs, epochs):
    import paper_2303_01778_b200 as pb
    from oracle import cnn_oracle
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    from paper_2303_01778_b200.models import cnn_init
    from paper_2303_01778_b200.trainer import NamedParams
    X, y = femnist_like.features[100:100 + n], femnist_like.labels[100:100 + n]
    w0 = cnn_init(spec, seed=3)
    plugin = pb.FedAvg(lr=0.05, batch_size=bs, collect_local_loss=True)
    glob = plugin.init_global(NamedParams.from_flat(spec, w0))
    rep = pb.client_execute(plugin, ClientProfile(11, n, DataSlice(X, y, np.arange(n))), glob,
                            None, epochs, bs, 0.05, seed=4, round_num=2)
    got = np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names])
    want, steps, loss = cnn_oracle.client_train(w0, X, y, 11, 4, 2, epochs, bs, 0.05, 62,
                                                emulate_bf16=True)
    w0d = w0.astype(np.float64)
    errs = {name: _rel(got[o:o + s] - w0d[o:o + s], want[o:o + s] - w0d[o:o + s])
            for name, o, s, _ in spec.columns()}
    assert max(errs.values()) <= 2e-2, errs
    gl = float(rep.client_result.numpy("local_loss")[0])
    assert abs(gl - loss) / loss <= 1e-3, (gl, loss)


def test_cnn_fl_rounds_match_exact_oracle(spec, femnist_like):
    import paper_2303_01778_b200 as pb
    from oracle import cnn_oracle
    from paper_2303_01778_b200.models import cnn_init
    ds = femnist_like
    train = pb.SyntheticDataset(ds.features[:3200], ds.labels[:3200], 62, 784, 3.0, 1.0) \
        if len(np.unique(ds.labels[:3200])) == 62 else ds
    profiles = pb.partition(train, 40, pb.PartitionSpec(quantity_skew=1.0, min_samples_per_client=10),
                            seed=0)
    data = {p.client_id: (p.data_partition.features, p.data_partition.labels) for p in profiles}
    ev = pb.SyntheticDataset(ds.features[3200:], ds.labels[3200:], 62, 784, 3.0, 1.0) \
        if len(np.unique(ds.labels[3200:])) == 62 else ds
    cfg = pb.SimConfig(total_clients=40, concurrent_clients=12, num_devices=2, total_rounds=3,
                       seed=5, scheme="PARROT")
    eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=0.05, batch_size=20), profiles,
                              pb.make_device_models(2), eval_data=ev, model="cnn", init_seed=3)
    ref = cnn_init(spec, seed=3).astype(np.float64)
    for oc in eng.run():
        sel = pb.select_clients(cfg, oc.round).selected
        ref = cnn_oracle.fedavg_round(ref, data, sel, 5, oc.round, 1, 20, 0.05, 62)
        got = np.concatenate([oc.new_global.numpy(nm).reshape(-1) for nm in spec.names])
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 5e-3, oc.round
        acc, loss = cnn_oracle.evaluate(ref, ev.features, ev.labels, 62)
        assert abs(oc.accuracy - acc) <= 0.01, (oc.round, oc.accuracy, acc)
        assert abs(oc.loss - loss) / loss <= 0.01, (oc.round, oc.loss, loss)


def test_cnn_non_finite_detected(spec, femnist_like):
    import paper_2303_01778_b200 as pb
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    from paper_2303_01778_b200.models import cnn_init
    from paper_2303_01778_b200.trainer import NamedParams, NonFiniteLossError
    X = femnist_like.features[:30].copy()
    y = femnist_like.labels[:30]
    X[17, 5] = np.nan
    plugin = pb.FedAvg(lr=0.05, batch_size=10)
    glob = plugin.init_global(NamedParams.from_flat(spec, cnn_init(spec, 0)))
    with pytest.raises(NonFiniteLossError, match="client 3 round 1"):
        pb.client_execute(plugin, ClientProfile(3, 30, DataSlice(X, y, np.arange(30))), glob, None,
                          1, 10, 0.05, seed=0, round_num=1)
