"""ResNet-18 (GroupNorm) path (BASELINE config 4) on the GPU vs the torch-CPU
float64 restatement (oracle/resnet_oracle.py).  Restatement-pinned: the
reference has no ResNet.

Conditioning: the device keeps activations, conv weights and dL/dz in bf16
(fp32 accumulation).  One SGD step of this network under bf16 rounding is
ill-conditioned: the oracle's own bf16 emulation run in float32 instead of
float64 changes the per-tensor update by ~5e-2 (median over tensors; up to
~0.12 in the stem layers, ~1e-3 for fc).  The device is held to that floor,
measured in the test itself -- and its conv kernels are separately exact to
1e-5 against torch (test_gpu_resnet_conv.py):

1. one step from identical weights: per-tensor update error vs the emulating
   float64 oracle, median <= 1.5x the oracle's fp32-vs-f64 median, fc within
   5e-3, every tensor's update direction cos >= 0.95 vs the exact oracle
   (bf16 itself moves the stem-layer updates by up to ~20% from exact), loss
   within 1e-3 (the forward carries the same bf16 rounding noise, ~1e-4);
2. a local run and a two-round FedAvg engine run: losses, eval accuracy and
   global weights close to the exact oracle (tolerances in the tests);
3. bit-identical results across runs.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def spec():
    from paper_2303_01778_b200.models import resnet_spec
    return resnet_spec(10)


@pytest.fixture(scope="module")
def cifar_like():
    from paper_2303_01778_b200.data import generate
    return generate(400, 3072, 10, seed=0)


def _device(spec, w0, X, y, bs, epochs, lr, sweeps=0, monkeypatch=None):
    import paper_2303_01778_b200 as pb
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    from paper_2303_01778_b200.trainer import NamedParams
    if monkeypatch is not None:
        monkeypatch.setenv("PB_CNN_MAX_SWEEPS", str(sweeps))
    plugin = pb.FedAvg(lr=lr, batch_size=bs, collect_local_loss=True)
    glob = plugin.init_global(NamedParams.from_flat(spec, w0))
    n = len(y)
    rep = pb.client_execute(plugin, ClientProfile(11, n, DataSlice(X, y, np.arange(n))), glob, None,
                            epochs, bs, lr, seed=4, round_num=2)
    return (np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names]),
            float(rep.client_result.numpy("local_loss")[0]))


def _per_tensor(spec, w0, got, ref):
    err, cos = {}, {}
    for nm, o, s, _ in spec.columns():
        d, r = got[o:o + s] - w0[o:o + s], ref[o:o + s] - w0[o:o + s]
        err[nm] = float(np.linalg.norm(d - r) / max(np.linalg.norm(r), 1e-30))
        cos[nm] = float(d @ r / max(np.linalg.norm(d) * np.linalg.norm(r), 1e-30))
    return err, cos


def test_resnet_one_step_vs_oracle(spec, cifar_like):
    import torch
    from oracle import fedsim_oracle, resnet_oracle as R
    from paper_2303_01778_b200.models import resnet_init
    X, y = cifar_like.features[:6], cifar_like.labels[:6]
    w0 = resnet_init(spec, seed=3)
    w0d = w0.astype(np.float64)
    got, loss = _device(spec, w0, X, y, 6, 1, 0.05)
    idx = fedsim_oracle.minibatch_orders(4, 11, 2, 6, 1)[0]
    emu64, l64 = R.step(w0d, X[idx], y[idx], 0.05, 10, emulate_bf16=True)
    emu32, _ = R.step(w0d, X[idx], y[idx], 0.05, 10, emulate_bf16=True, dtype=torch.float32)
    exact, _ = R.step(w0d, X[idx], y[idx], 0.05, 10)
    err, _ = _per_tensor(spec, w0d, got, emu64)
    floor, _ = _per_tensor(spec, w0d, emu32, emu64)
    _, cos = _per_tensor(spec, w0d, got, exact)
    assert np.median(list(err.values())) <= 1.5 * np.median(list(floor.values())), (err, floor)
    assert err["fc_w"] <= 5e-3 and err["fc_b"] <= 5e-3, err
    assert min(cos.values()) >= 0.95, cos
    assert abs(loss - l64) / l64 <= 1e-3, (loss, l64)


def test_resnet_local_run_vs_oracle(spec, cifar_like):
    from oracle import resnet_oracle as R
    from paper_2303_01778_b200.models import resnet_init
    X, y = cifar_like.features[10:28], cifar_like.labels[10:28]
    w0 = resnet_init(spec, seed=5)
    got, loss = _device(spec, w0, X, y, 6, 1, 0.01)
    ref, steps, ref_loss = R.client_train(w0, X, y, 11, 4, 2, 1, 6, 0.01, 10)
    assert steps == 3
    assert abs(loss - ref_loss) / ref_loss <= 2e-3, (loss, ref_loss)
    d, r = got - w0, ref - w0
    assert np.linalg.norm(d - r) / np.linalg.norm(r) <= 0.1
    assert d @ r / (np.linalg.norm(d) * np.linalg.norm(r)) >= 0.995


def test_resnet_deterministic(spec, cifar_like):
    from paper_2303_01778_b200.models import resnet_init
    X, y = cifar_like.features[:13], cifar_like.labels[:13]
    w0 = resnet_init(spec, seed=1)
    a = _device(spec, w0, X, y, 5, 2, 0.02)
    b = _device(spec, w0, X, y, 5, 2, 0.02)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]


def test_resnet_fedavg_rounds_vs_oracle(spec, cifar_like):
    import paper_2303_01778_b200 as pb
    from oracle import resnet_oracle as R
    from paper_2303_01778_b200.models import resnet_init
    ds = cifar_like
    train = pb.SyntheticDataset(ds.features[:48], ds.labels[:48], 10, 3072, 3.0, 1.0)
    profiles = pb.partition(train, 6, pb.PartitionSpec(quantity_skew=1.0, min_samples_per_client=4), seed=0)
    data = {p.client_id: (p.data_partition.features, p.data_partition.labels) for p in profiles}
    ev = pb.SyntheticDataset(ds.features[200:400], ds.labels[200:400], 10, 3072, 3.0, 1.0)
    cfg = pb.SimConfig(total_clients=6, concurrent_clients=3, num_devices=2, total_rounds=2, seed=5,
                       scheme="PARROT")
    eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=0.01, batch_size=8), profiles, pb.make_device_models(2),
                              eval_data=ev, model="resnet", init_seed=3)
    ref = resnet_init(spec, seed=3).astype(np.float64)
    w_init = ref.copy()
    for oc in eng.run():
        sel = pb.select_clients(cfg, oc.round).selected
        ref = R.fedavg_round(ref, data, sel, 5, oc.round, 1, 8, 0.01, 10)
        got = np.concatenate([oc.new_global.numpy(nm).reshape(-1) for nm in spec.names])
        d, r = got - w_init, ref - w_init
        # cumulative weight change after r+1 rounds of bf16 steps vs exact f64
        assert np.linalg.norm(d - r) / np.linalg.norm(r) <= 0.15, oc.round
        acc, loss = R.evaluate(ref, ev.features, ev.labels, 10)
        assert abs(oc.accuracy - acc) <= 0.03, (oc.round, oc.accuracy, acc)
        assert abs(oc.loss - loss) / loss <= 0.01, (oc.round, oc.loss, loss)


def test_resnet_stale_workspace_nan(spec, cifar_like):
    """Workspace memory is reused across groups, tests and other models: a
    partial batch (13 samples, batch 5) trained on a workspace poisoned with
    NaN bit patterns gives the same result as on a clean one (samples past
    the batch must never feed the whole-tile weight gradients)."""
    import paper_2303_01778_b200.resnet as rn
    from paper_2303_01778_b200.models import resnet_init
    X, y = cifar_like.features[:13], cifar_like.labels[:13]
    w0 = resnet_init(spec, seed=1)
    clean = _device(spec, w0, X, y, 5, 1, 0.02)
    for t in rn._WS.buf.values():
        t.view(-1).view(dtype=t.dtype).fill_(float("nan")) if t.is_floating_point() else t.fill_(255)
    poisoned = _device(spec, w0, X, y, 5, 1, 0.02)
    assert np.all(np.isfinite(poisoned[0])) and np.isfinite(poisoned[1])
    assert np.array_equal(clean[0], poisoned[0]) and clean[1] == poisoned[1]


def test_resnet_plugin_terms_exact(spec, cifar_like, monkeypatch):
    """FedProx and SCAFFOLD on the ResNet path (fused into every SGD kernel:
    conv weights with their bf16 copies, GroupNorm, fc; fedsim/trainer.py
    :237-257, :288-348).  The terms are pinned by algebra against the FedAvg
    run on the same data, so no operand rounding enters the comparison:
    * SCAFFOLD, one step from w0: the forward/backward are FedAvg's, so
      w1_scaffold - w1_fedavg = -lr * (c - c_m) (random server and client
      controls) to fp32 rounding;
    * FedProx, two steps: step one equals FedAvg's (w = w0), step two sees
      the same weights and adds mu * (w1 - w0), so
      w2_prox - w2_fedavg = -lr * mu * (w1 - w0)."""
    import torch
    import paper_2303_01778_b200 as pb
    from paper_2303_01778_b200.core import ClientProfile, DataSlice
    from paper_2303_01778_b200.models import init_params
    from paper_2303_01778_b200.trainer import ClientData, NamedParams, train_group
    X, y = cifar_like.features[:40], cifar_like.labels[:40]
    data = ClientData.from_profiles([ClientProfile(0, 40, DataSlice(X, y, np.arange(40)))], n_classes=10)
    lr, mu, P = 0.05, 0.5, spec.numel
    w0 = torch.from_numpy(init_params(spec, 3)).cuda()
    base = w0.cpu().numpy().astype(np.float64)

    def run(plugin, sweeps, glob=None, work=None):
        monkeypatch.setenv("PB_CNN_MAX_SWEEPS", str(sweeps))
        glob = glob if glob is not None else plugin.init_global(NamedParams.from_flat(spec, w0))
        go = train_group(plugin, spec, data, [0], w0, glob, work, 1, 20, lr, 4, 1)
        return go.w_out[0].cpu().numpy().astype(np.float64)

    avg1, avg2 = run(pb.FedAvg(lr=lr, batch_size=20), 1), run(pb.FedAvg(lr=lr, batch_size=20), 2)
    prox2 = run(pb.FedProx(mu=mu, lr=lr, batch_size=20), 2)
    want = -lr * mu * (avg1 - base)
    assert np.linalg.norm(want) > 0
    assert _rel(prox2 - avg2, want) <= 1e-3
    sc = pb.Scaffold(lr=lr, batch_size=20)
    glob = sc.init_global(NamedParams.from_flat(spec, w0))
    gen = torch.Generator(device="cuda").manual_seed(1)
    for nm in spec.names:
        t = glob.tensor("server_ctrl_" + nm)
        t.copy_(1e-2 * torch.randn(t.shape, generator=gen, device="cuda"))
    work = torch.zeros(1, (P + 3) // 4 * 4, device="cuda")[:, :P]
    work.copy_(1e-2 * torch.randn(1, P, generator=gen, device="cuda"))
    sc1 = run(sc, 1, glob, work)
    c = glob.flat(spec, "server_ctrl_").cpu().numpy().astype(np.float64)
    cm = work[0].cpu().numpy().astype(np.float64)
    assert _rel(sc1 - avg1, -lr * (c - cm)) <= 1e-4
    monkeypatch.setenv("PB_CNN_MAX_SWEEPS", "0")
