"""Per-step, per-tensor replay error of the device ResNet-18-GN against the
bf16-emulating oracle (diagnostic twin of tests/test_gpu_resnet.py)."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2303_01778_b200 as pb
from oracle import fedsim_oracle, resnet_oracle as R
from paper_2303_01778_b200.core import ClientProfile, DataSlice
from paper_2303_01778_b200.models import resnet_init, resnet_spec
from paper_2303_01778_b200.trainer import NamedParams

ds = pb.generate(600, 3072, 10, seed=0)
spec = resnet_spec(10)
w0 = resnet_init(spec, seed=3)


def device_after(X, y, bs, epochs, sweeps):
    os.environ["PB_CNN_MAX_SWEEPS"] = str(sweeps)
    plugin = pb.FedAvg(lr=0.05, batch_size=bs)
    glob = plugin.init_global(NamedParams.from_flat(spec, w0))
    n = len(y)
    rep = pb.client_execute(plugin, ClientProfile(11, n, DataSlice(X, y, np.arange(n))), glob,
                            None, epochs, bs, 0.05, seed=4, round_num=2)
    return np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names])


n, bs, epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 12, 6, 1
X, y = ds.features[:n], ds.labels[:n]
nb = -(-n // bs)
orders = fedsim_oracle.minibatch_orders(4, 11, 2, n, epochs)
prev = w0.astype(np.float64)
for k in range(epochs * nb):
    t = time.time()
    cur = device_after(X, y, bs, epochs, k + 1)
    td = time.time() - t
    e, b = divmod(k, nb)
    idx = orders[e][b * bs:(b + 1) * bs]
    for emu in (True, False):
        ref, loss = R.step(prev, X[idx], y[idx], 0.05, 10, emulate_bf16=emu)
        errs = {}
        for nm, o, s, _ in spec.columns():
            d_ref = ref[o:o + s] - prev[o:o + s]
            errs[nm] = np.linalg.norm((cur[o:o + s] - prev[o:o + s]) - d_ref) / max(np.linalg.norm(d_ref), 1e-30)
        worst = sorted(errs.items(), key=lambda kv: -kv[1])[:6]
        med = float(np.median(list(errs.values())))
        print(f"step {k} emu={emu} loss {loss:.4f} median {med:.2e} worst",
              ", ".join(f"{a} {v:.1e}" for a, v in worst), f"(device {td:.1f}s)", flush=True)
        if k == 0 and emu:
            print("  all:", " ".join(f"{a}:{v:.0e}" for a, v in errs.items()), flush=True)
    prev = cur.astype(np.float64)
