"""Per-step, per-tensor replay error of the device CNN (lazy and direct fc1)
against the emulating oracle (the arithmetic test of tests/test_gpu_cnn.py,
verbose)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
import torch.nn.functional as F

import paper_2303_01778_b200 as pb
from oracle import cnn_oracle, fedsim_oracle
from paper_2303_01778_b200.core import ClientProfile, DataSlice
from paper_2303_01778_b200.models import cnn_init, cnn_spec
from paper_2303_01778_b200.trainer import NamedParams

ds = pb.generate(4000, 784, 62, seed=0)
spec = cnn_spec(62)
w0 = cnn_init(spec, seed=3)
o1, s1 = [(o, s) for nm, o, s, _ in spec.columns() if nm == "fc1_w"][0]


def device_after(X, y, bs, epochs, sweeps):
    os.environ["PB_CNN_MAX_SWEEPS"] = str(sweeps)
    plugin = pb.FedAvg(lr=0.05, batch_size=bs)
    glob = plugin.init_global(NamedParams.from_flat(spec, w0))
    n = len(y)
    rep = pb.client_execute(plugin, ClientProfile(11, n, DataSlice(X, y, np.arange(n))), glob,
                            None, epochs, bs, 0.05, seed=4, round_num=2)
    return np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names])


for lazy in ("1", "0"):
    os.environ["PB_CNN_LAZY"] = lazy
    base = torch.as_tensor(w0.reshape(-1)[o1:o1 + s1].astype(np.float64)).view(512, 3136) if lazy == "1" else None
    for n, bs, epochs in [(45, 16, 1), (100, 20, 1)]:
        X, y = ds.features[100:100 + n], ds.labels[100:100 + n]
        nb = -(-n // min(bs, n))
        orders = fedsim_oracle.minibatch_orders(4, 11, 2, n, epochs)
        Xt, yt = torch.as_tensor(X), torch.as_tensor(y, dtype=torch.long)
        prev = w0.astype(np.float64)
        for k in range(epochs * nb):
            cur = device_after(X, y, bs, epochs, k + 1)
            e, b = divmod(k, nb)
            idx = torch.as_tensor(orders[e][b * min(bs, n):(b + 1) * min(bs, n)])
            for emu_base in ((base, None) if lazy == "1" else (None,)):
                params = [p.requires_grad_(True) for p in cnn_oracle.unflatten(prev, 62)]
                loss = F.cross_entropy(cnn_oracle.forward(params, Xt[idx], True, emu_base), yt[idx])
                grads = torch.autograd.grad(loss, params)
                ref = np.concatenate([(p - 0.05 * g).detach().reshape(-1).numpy() for p, g in zip(params, grads)])
                errs = {nm: "%.1e" % (np.linalg.norm((cur[o:o + s] - prev[o:o + s]) - (ref[o:o + s] - prev[o:o + s]))
                                      / np.linalg.norm(ref[o:o + s] - prev[o:o + s])) for nm, o, s, _ in spec.columns()}
                print("lazy" if lazy == "1" else "direct", n, bs, "step", k,
                      "emu-base" if emu_base is not None else "emu-plain", errs, flush=True)
            prev = cur.astype(np.float64)
