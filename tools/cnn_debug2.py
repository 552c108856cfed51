"""Replay step 2 in the oracle from the device's own step-1 weights."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2303_01778_b200 as pb
from oracle import cnn_oracle, fedsim_oracle
from paper_2303_01778_b200.core import ClientProfile, DataSlice
from paper_2303_01778_b200.models import cnn_init, cnn_spec
from paper_2303_01778_b200.trainer import NamedParams
import torch, torch.nn.functional as F

ds = pb.generate(4000, 784, 62, seed=0)
spec = cnn_spec(62)
w0 = cnn_init(spec, seed=3)
n, bs = int(os.environ.get("DBG_N", "60")), 20
X, y = ds.features[100:100 + n], ds.labels[100:100 + n]
prof = ClientProfile(11, n, DataSlice(X, y, np.arange(n)))

def device_run(sweeps):
    os.environ["PB_CNN_MAX_SWEEPS"] = str(sweeps)
    plugin = pb.FedAvg(lr=0.05, batch_size=bs)
    glob = plugin.init_global(NamedParams.from_flat(spec, w0))
    rep = pb.client_execute(plugin, prof, glob, None, 1, bs, 0.05, seed=4, round_num=2)
    return np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names])

order = fedsim_oracle.minibatch_orders(4, 11, 2, n, 1)[0]
def oracle_step(w, k):
    params = [p.requires_grad_(True) for p in cnn_oracle.unflatten(w, 62)]
    idx = torch.as_tensor(order[k * bs:(k + 1) * bs])
    Xt = torch.as_tensor(X); yt = torch.as_tensor(y, dtype=torch.long)
    loss = F.cross_entropy(cnn_oracle.forward(params, Xt[idx], True), yt[idx])
    g = torch.autograd.grad(loss, params)
    with torch.no_grad():
        return np.concatenate([(p - 0.05 * gg).reshape(-1).numpy() for p, gg in zip(params, g)])

runs = [w0.astype(np.float64)] + [device_run(k) for k in range(1, n // bs + 1)]
for k, (start, end) in enumerate(zip(runs[:-1], runs[1:])):
    ref = oracle_step(start, k)
    print("step", k + 1, {nm: "%.1e" % (np.linalg.norm((end[o:o+s] - start[o:o+s]) - (ref[o:o+s] - start[o:o+s]))
                                   / np.linalg.norm(ref[o:o+s] - start[o:o+s])) for nm, o, s, _ in spec.columns()}, flush=True)
