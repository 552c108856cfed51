"""Parity at the headline configuration (BASELINE config 2 at M_p = 1000):
one group of 1000 clients with C2's Dirichlet(1.0) sample counts (the round-0
selection of 3400 clients), bs 20, E 1, lr 0.05 -- every one of its 72 sweeps
runs the dense-sweep kernel variants the bench runs (8 / 4 / 2 clients per
shared-W0 tile, one-CTA head, 2-way wgrad split) down to the sparse tail, on
the low-rank fc1, and the engine round folds fc1 straight from the history
(pb_cnn_lazy_fold).  The reference has no CNN, so the oracle is the torch-CPU
restatement (oracle/cnn_oracle.py, restatement-pinned).

1. Kernel arithmetic, every local step of eight clients spanning the size
   distribution (1 to 72 steps): the group is re-run stopped after k sweeps
   (PB_CNN_MAX_SWEEPS) and step k of each client is replayed in the
   bf16-emulating oracle from the DEVICE's weights after step k-1, so
   errors cannot compound.  The device's own discrete decisions of that step
   (pool-1 argmax + ReLU bit, pool-2 argmax, ReLU-2 and ReLU-3 signs, read
   from its workspace) are compared with the oracle's: every decision that
   differs must sit within 1e-4 RMS of its boundary (a legitimate fp32-vs-f64
   flip, never a wrong tile or index), and the step's update must match the
   oracle's to 2e-3 (per-tensor relative error, the largest tensor counts)
   unless such a flip happened, when the bound is 5e-2.  Flipped steps must
   stay a minority.
2. The FedAvg fold at full density: the engine round's global (deferred
   low-rank fc1 fold, fold_group) equals the float64 sample-weighted mean of
   the clients' materialised end models to 1e-5 of ||W||.
3. Training outcome vs the exact float64 oracle (no operand rounding), whole
   local runs of the same eight clients from the round-start model: mean
   local loss within 0.1 %, and the relative update error at most 1.5x the
   precision floor measured here on the same client -- the error of the
   oracle's own bf16-emulating run (or of its float32 run) against the exact
   one.  That floor is large: near initialisation (loss ~ ln 62) the update
   is ill-conditioned in the operand rounding, so bf16 conv2 / fc1
   operands alone move a single step by 2-5 % and a 16-72-step run by 40-60 %
   (measured: device 0.40 vs emulating oracle 0.39 at 16 steps, 0.57 vs 0.61
   at 72), while the loss trajectories agree to 2e-4.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BS, LR, SEED, ROUND = 20, 0.05, 0, 0
TIGHT, FLIPPED = 2e-3, 5e-2
# largest boundary margin (x layer RMS) at which a decision may legitimately
# differ between the fp32 device and the f64 oracle fed the same rounded
# operands: pool1 argmax / ReLU1 / pool2 argmax / ReLU2 / ReLU3
MARGINS = (1e-4, 1e-4, 1e-3, 1e-3, 1e-3)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def c2():
    """The round-0 selection of C2 (1000 of 3400 clients, Dirichlet(1.0)
    sizes, min 10) with FEMNIST-shaped Gaussian-mixture data (fedsim.data.
    generate's construction: unit class means x 3 + N(0, 1), fp32)."""
    import torch
    import paper_2303_01778_b200 as pb
    from paper_2303_01778_b200.core import STREAM_PARTITION, ClientProfile, DataSlice, stream_rng
    from paper_2303_01778_b200.data import client_sizes
    from paper_2303_01778_b200.models import cnn_init, cnn_spec
    from paper_2303_01778_b200.trainer import ClientData
    sizes_all = client_sizes(768_400, 3400, pb.PartitionSpec(quantity_skew=1.0, min_samples_per_client=10),
                             stream_rng(SEED, STREAM_PARTITION))
    cfg = pb.SimConfig(total_clients=3400, concurrent_clients=1000, num_devices=1, total_rounds=2,
                       seed=SEED, scheme="PARROT")
    chosen = list(pb.select_clients(cfg, ROUND).selected)
    sizes = np.array([int(sizes_all[c]) for c in chosen], dtype=np.int64)
    g = np.random.default_rng(7)
    means = g.standard_normal((62, 784)).astype(np.float32)
    means *= 3.0 / np.linalg.norm(means, axis=1, keepdims=True)
    profiles, data = [], {}
    for cid, n in enumerate(sizes):   # client ids 0..999 (the chosen clients, renumbered)
        y = g.integers(0, 62, int(n))
        X = means[y] + g.standard_normal((int(n), 784), dtype=np.float32)
        profiles.append(ClientProfile(cid, int(n), DataSlice(X, y, np.arange(int(n)))))
        data[cid] = (X, y)
    spec = cnn_spec(62)
    cd = ClientData.from_profiles(profiles, n_classes=62)
    w0 = torch.from_numpy(cnn_init(spec, seed=3)).cuda()
    steps = -(-sizes // BS)
    order = np.argsort(-steps, kind="stable")
    picks = sorted({int(order[0]), int(order[1]), int(order[int(0.05 * len(order))]),
                    int(order[int(0.25 * len(order))]), int(order[int(0.5 * len(order))]),
                    int(order[int(0.75 * len(order))]), int(order[-1]), int(order[-2])})
    return dict(spec=spec, cd=cd, w0=w0, sizes=sizes, steps=steps, data=data, profiles=profiles,
                picks=picks)


def _group(c2, monkeypatch, sweeps: int):
    """Train the whole 1000-client group, stopped after `sweeps` sweeps (0 =
    all); returns (end-model rows of the picked clients, their decisions of
    the last sweep run)."""
    import torch
    import paper_2303_01778_b200 as pb
    from paper_2303_01778_b200 import cnn
    from paper_2303_01778_b200.trainer import NamedParams, train_group
    monkeypatch.setenv("PB_CNN_MAX_SWEEPS", str(sweeps))
    spec, cd = c2["spec"], c2["cd"]
    plugin = pb.FedAvg(lr=LR, batch_size=BS)
    glob = plugin.init_global(NamedParams.from_flat(spec, c2["w0"]))
    G = len(c2["sizes"])
    go = train_group(plugin, spec, cd, list(range(G)), c2["w0"], glob, None, 1, BS, LR, SEED, ROUND)
    picks = c2["picks"]
    rows = go.w_out[picks].cpu().numpy().astype(np.float64)
    dec = None
    if sweeps > 0:
        _, total, rank, active = cnn.sweep_plan(c2["sizes"], BS, 1)
        slot_of = {int(r): j for j, r in enumerate(rank)}
        hlen, hoff, *_ = cnn.lazy_plan(total, active, BS)
        ws, hx = cnn._WS.buf, cnn._LZ.buf["hx"]
        t = sweeps - 1
        dec = {}
        for c in picks:
            if total[c] <= t:
                continue
            j = slot_of[c]
            cnt = min(BS, int(c2["sizes"][c]) - t * BS)
            sid = j * BS
            am1 = ws["am1"][sid * 6272:(sid + cnt) * 6272].view(cnt, 6272).cpu().numpy()
            am2 = ws["am2"][sid * 3136:(sid + cnt) * 3136].view(cnt, 3136).cpu().numpy()
            h = ws["h"].view(torch.float32)[sid * 512:(sid + cnt) * 512].view(cnt, 512).cpu().numpy()
            if 0 < cnn.lz_switch_step(sweeps) <= t:   # past the switch: direct fc1, p2 in the workspace
                p2 = ws["p2"].view(torch.float32)[sid * 3136:(sid + cnt) * 3136].view(cnt, 3136).cpu().numpy()
            else:
                base = int(hoff[c]) + t * BS
                p2 = hx[base * 3136:(base + cnt) * 3136].view(cnt, 3136).float().cpu().numpy()
            dec[c] = (am1 & 3, am1 >> 2, am2, p2 > 0, h > 0)
    return rows, dec


def _oracle_decisions(params, x, fc1_base):
    """The oracle's discrete decisions of one step in the device's layouts,
    each with its margin to the boundary (relative to the layer's RMS):
    pool-1 argmax and ReLU-1 bit ([B, 14*14*32], pool position-major,
    channel-minor), pool-2 argmax over the ReLU outputs ([B, 7*7*64], first
    max), ReLU-2 of each pool-2 window and ReLU-3 signs."""
    import torch
    import torch.nn.functional as F
    from oracle import cnn_oracle as O
    c1w, c1b, c2w, c2b, f1w, f1b, f2w, f2b = [p.detach() for p in params]
    B = x.shape[0]

    def windows(z):   # [B, C, H, W] -> [B, H/2, W/2, C, 4] (d = dy*2 + dx)
        _, C, H, W = z.shape
        return z.reshape(B, C, H // 2, 2, W // 2, 2).permute(0, 2, 4, 1, 3, 5).reshape(B, H // 2, W // 2, C, 4)

    def first_argmax(w):
        best = w.max(-1, keepdim=True).values
        idx = torch.arange(4).expand_as(w)
        return torch.where(w == best, idx, torch.full_like(idx, 9)).min(-1).values

    def gap(w):
        top = w.topk(2, dim=-1).values
        return top[..., 0] - top[..., 1], top[..., 1]

    with torch.no_grad():
        # conv1 as the device runs it: bf16 image and weights on the tensor cores
        z1 = F.conv2d(O._RoundValue.apply(x.reshape(-1, 1, 28, 28)), O._RoundValue.apply(c1w).permute(0, 3, 1, 2),
                      c1b, padding=2)
        r1 = float(z1.pow(2).mean().sqrt())
        w1 = windows(z1)
        best1 = w1.max(-1).values
        arg1 = (first_argmax(w1).reshape(B, -1), (gap(w1)[0] / r1).reshape(B, -1))
        relu1 = ((best1 > 0).reshape(B, -1), (best1.abs() / r1).reshape(B, -1))
        h = F.max_pool2d(F.relu(z1), 2)
        z2 = F.conv2d(O._RoundValue.apply(h), O._RoundValue.apply(c2w).permute(0, 3, 1, 2), padding=2) \
            + c2b.view(1, -1, 1, 1)
        r2 = float(z2.pow(2).mean().sqrt())
        a2 = F.relu(z2)
        zb = windows(z2).max(-1).values            # pre-ReLU max of each pool-2 window
        g2, second = gap(windows(a2))
        g2 = torch.where(second > 0, g2, torch.full_like(g2, np.inf))   # <= 1 positive: fixed unless it crosses 0
        arg2 = (first_argmax(windows(a2)).reshape(B, -1), (torch.minimum(g2, zb.abs()) / r2).reshape(B, -1))
        relu2 = ((zb > 0).reshape(B, -1), (zb.abs() / r2).reshape(B, -1))
        hp = F.max_pool2d(a2, 2).permute(0, 2, 3, 1).reshape(B, -1)
        if fc1_base is None:   # direct fc1 (after the low-rank switch): tf32 truncation
            z3 = O._tf32(hp) @ O._tf32(f1w).t() + f1b
        else:
            z3 = O._bf16(hp) @ (f1w - fc1_base + O._bf16(fc1_base)).t() + f1b
        relu3 = (z3 > 0, z3.abs() / float(z3.pow(2).mean().sqrt()))
    return [(d.numpy(), m.numpy()) for d, m in (arg1, relu1, arg2, relu2, relu3)]


def test_c2_headline_group_per_step_parity(c2, monkeypatch):
    import torch
    import torch.nn.functional as F
    from oracle import cnn_oracle, fedsim_oracle
    spec, picks, steps = c2["spec"], c2["picks"], c2["steps"]
    assert steps.max() >= 60 and steps.min() == 1 and len(steps) == 1000
    o1, s1 = [(o, s) for nm, o, s, _ in spec.columns() if nm == "fc1_w"][0]
    w0 = c2["w0"].cpu().numpy().astype(np.float64)
    fc1_base = torch.as_tensor(w0[o1:o1 + s1]).view(512, 3136)
    prev = {c: w0.copy() for c in picks}
    report = []
    from paper_2303_01778_b200 import cnn
    switch = cnn.lz_switch_step(int(steps.max()))
    for k in range(1, int(max(steps[c] for c in picks)) + 1):
        rows, dec = _group(c2, monkeypatch, k)
        # steps from the switch sweep on run the direct fc1 (tf32 truncation
        # of the materialised weights) instead of the low-rank form
        base_k = None if 0 < switch <= k - 1 else fc1_base
        for i, c in enumerate(picks):
            if steps[c] < k:
                continue
            X, y = c2["data"][c]
            n = len(y)
            order = fedsim_oracle.minibatch_orders(SEED, c, ROUND, n, 1)[0]
            idx = torch.as_tensor(order[(k - 1) * BS:k * BS])
            xb = torch.as_tensor(X, dtype=torch.float64)[idx]
            params = [p.requires_grad_(True) for p in cnn_oracle.unflatten(prev[c], 62)]
            loss = F.cross_entropy(cnn_oracle.forward(params, xb, True, base_k),
                                   torch.as_tensor(y)[idx])
            grads = torch.autograd.grad(loss, params)
            ref = np.concatenate([(p - LR * g).detach().reshape(-1).numpy() for p, g in zip(params, grads)])
            cur = rows[i]
            err = max(_rel(cur[o:o + s] - prev[c][o:o + s], ref[o:o + s] - prev[c][o:o + s])
                      for _, o, s, _ in spec.columns())
            # decisions: device (workspace) vs oracle, and the margin of every flip
            flips, margins = [], []
            for (want, margin), got in zip(_oracle_decisions(params, xb, base_k), dec[c]):
                diff = np.asarray(got) != np.asarray(want)
                flips.append(int(diff.sum()))
                margins.append(float(margin[diff].max()) if diff.any() else 0.0)
            report.append((c, k, err, flips, margins))
            prev[c] = cur
    kinds = ("pool1-arg", "relu1", "pool2-arg", "relu2", "relu3")
    print(f"\n{len(report)} steps replayed")
    for i, kind in enumerate(kinds):
        f = [r[3][i] for r in report]
        m = [r[4][i] for r in report if r[3][i]]
        print(f"  {kind:9s}: {sum(f)} flips in {sum(1 for v in f if v)} steps, "
              f"largest flipped margin {max(m) if m else 0:.2e} (bound {MARGINS[i]:.0e})")
    clean = [r[2] for r in report if not any(r[3])]
    dirty = [r[2] for r in report if any(r[3])]
    print(f"  step error: clean {len(clean)} steps median {np.median(clean) if clean else 0:.2e} "
          f"max {max(clean) if clean else 0:.2e}; flipped {len(dirty)} steps max {max(dirty) if dirty else 0:.2e}")
    assert len(report) == int(sum(steps[c] for c in picks))
    for c, k, err, flips, margins in report:
        for i, kind in enumerate(kinds):   # every differing decision is a rounding flip
            assert margins[i] <= MARGINS[i], (c, k, kind, margins[i])
        assert err <= (TIGHT if not any(flips) else FLIPPED), (c, k, err, flips)
    assert len(dirty) <= len(report) // 2


def test_c2_headline_round_fold_and_outcome(c2, monkeypatch):
    import torch
    import paper_2303_01778_b200 as pb
    from oracle import cnn_oracle
    spec, sizes, picks = c2["spec"], c2["sizes"], c2["picks"]
    # the engine round: 1000 clients, deferred low-rank fc1 fold
    cfg = pb.SimConfig(total_clients=1000, concurrent_clients=1000, num_devices=1, total_rounds=1,
                       warmup_rounds=0, seed=SEED, scheme="PARROT")
    from paper_2303_01778_b200.trainer import NamedParams
    plugin = pb.FedAvg(lr=LR, batch_size=BS)
    glob0 = plugin.init_global(NamedParams.from_flat(spec, c2["w0"]))
    eng = pb.SimulationEngine(cfg, plugin, c2["profiles"], pb.make_device_models(1),
                              client_data=c2["cd"], initial_global=glob0)
    out = eng.run_round(ROUND)
    got = np.concatenate([out.new_global.numpy(nm).reshape(-1) for nm in spec.names])
    # the same clients' materialised end models (fc1 written by pb_cnn_train_group)
    monkeypatch.setenv("PB_CNN_MAX_SWEEPS", "0")
    from paper_2303_01778_b200.trainer import train_group
    G = len(sizes)
    go = train_group(plugin, spec, c2["cd"], list(range(G)), c2["w0"], glob0, None, 1, BS, LR, SEED, ROUND)
    acc = torch.zeros(spec.numel, dtype=torch.float64, device="cuda")
    for j in range(G):   # plan order does not matter in float64 at this tolerance
        acc += float(sizes[j]) * go.w_out[j].double()
    want = (acc / float(sizes.sum())).cpu().numpy()
    assert _rel(got, want) <= 1e-5
    # whole local runs vs the exact float64 oracle; the float32 oracle and the
    # bf16-emulating oracle measure how far operand precision alone moves them
    w0 = c2["w0"].cpu().numpy().astype(np.float64)
    rows = []
    for c in picks:
        X, y = c2["data"][c]
        ref, st, ref_loss = cnn_oracle.client_train(w0, X, y, c, SEED, ROUND, 1, BS, LR, 62)
        emu, _, _ = cnn_oracle.client_train(w0, X, y, c, SEED, ROUND, 1, BS, LR, 62, emulate_bf16=True)
        e32, _, _ = cnn_oracle.client_train(w0, X, y, c, SEED, ROUND, 1, BS, LR, 62, dtype=torch.float32)
        dev = go.w_out[c].cpu().numpy().astype(np.float64)
        du, dr = dev - w0, ref - w0
        cos = float(du @ dr / (np.linalg.norm(du) * np.linalg.norm(dr)))
        rows.append((c, st, _rel(du, dr), cos, _rel(emu - w0, dr), _rel(e32 - w0, dr),
                     _rel(du, emu - w0), float(go.loss_mean[c]), ref_loss))
        print(f"client {c} steps {st}: dev-vs-exact {rows[-1][2]:.3e} cos {cos:.4f}; emulating-vs-exact "
              f"{rows[-1][4]:.3e}; fp32-vs-exact {rows[-1][5]:.3e}; dev-vs-emulating {rows[-1][6]:.3e}; "
              f"loss {rows[-1][7]:.5f} vs {ref_loss:.5f}")
    for c, st, err, cos, e_emu, e_32, e_de, dl, rl in rows:
        # the device is as close to the exact run as bf16 operands allow
        assert err <= 1.5 * max(e_emu, e_32) + 1e-3, (c, st, err, e_emu, e_32)
        assert abs(dl - rl) <= 1e-3 * rl, (c, dl, rl)
