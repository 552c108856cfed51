"""Diagnostic: CNN clients trained in one 200-client group (dense sweeps) vs
one at a time (sparse sweeps); per-client update error after N sweeps."""
import os
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
from paper_2303_01778_b200.core import ClientProfile, DataSlice  # noqa: E402
from paper_2303_01778_b200.data import generate  # noqa: E402
from paper_2303_01778_b200.models import cnn_init, cnn_spec  # noqa: E402
from paper_2303_01778_b200.trainer import ClientData, NamedParams, train_group  # noqa: E402

spec = cnn_spec(62)
ds = generate(4000, 784, 62, seed=0)
G = int(os.environ.get("G", "200"))
sizes = np.random.default_rng(9).integers(11, 28, size=G)
off = np.concatenate([[0], np.cumsum(sizes)])
profiles = [ClientProfile(c, int(sizes[c]), DataSlice(ds.features[off[c]:off[c + 1]], ds.labels[off[c]:off[c + 1]],
                                                      np.arange(sizes[c]))) for c in range(G)]
data = ClientData.from_profiles(profiles, n_classes=62)
plugin = pb.FedAvg(lr=0.05, batch_size=10)
glob = plugin.init_global(NamedParams.from_flat(spec, cnn_init(spec, 2)))
w0 = glob.flat(spec)
base = w0.cpu().numpy().astype(np.float64)
cols = spec.columns()
for sweeps in (1, 2, 4):
    os.environ["PB_CNN_MAX_SWEEPS"] = str(sweeps)
    dense = train_group(plugin, spec, data, list(range(G)), w0, glob, None, 2, 10, 0.05, seed=7,
                        round_num=1).w_out.cpu().numpy().astype(np.float64)
    worst = {}
    errs = []
    for c in range(0, G, 17):
        one = train_group(plugin, spec, data, [c], w0, glob, None, 2, 10, 0.05, seed=7,
                          round_num=1).w_out.cpu().numpy()[0].astype(np.float64)
        d, o = dense[c] - base, one - base
        errs.append(np.linalg.norm(d - o) / np.linalg.norm(o))
        for nm, of, sz, _ in cols:
            e = np.linalg.norm(d[of:of + sz] - o[of:of + sz]) / max(np.linalg.norm(o[of:of + sz]), 1e-30)
            worst[nm] = max(worst.get(nm, 0.0), e)
    print(f"lazy={os.environ.get('PB_CNN_LAZY', '1')} sweeps={sweeps} median={np.median(errs):.2e} "
          f"max={np.max(errs):.2e} per-tensor max: " + " ".join(f"{k}={v:.1e}" for k, v in worst.items()), flush=True)
