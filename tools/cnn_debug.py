"""Per-tensor update error of the device CNN step vs the bf16-emulated oracle."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2303_01778_b200 as pb
from oracle import cnn_oracle
from paper_2303_01778_b200.core import ClientProfile, DataSlice
from paper_2303_01778_b200.models import cnn_init, cnn_spec
from paper_2303_01778_b200.trainer import NamedParams

ds = pb.generate(4000, 784, 62, seed=0)
spec = cnn_spec(62)
w0 = cnn_init(spec, seed=3)
w0d = w0.astype(np.float64)
for n, bs, E in [(20, 20, 1), (40, 20, 1), (60, 20, 1), (20, 20, 3), (8, 8, 1), (1, 1, 1)]:
    X, y = ds.features[100:100 + n], ds.labels[100:100 + n]
    plugin = pb.FedAvg(lr=0.05, batch_size=bs)
    glob = plugin.init_global(NamedParams.from_flat(spec, w0))
    rep = pb.client_execute(plugin, ClientProfile(11, n, DataSlice(X, y, np.arange(n))), glob,
                            None, E, bs, 0.05, seed=4, round_num=2)
    got = np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names])
    want, _, _ = cnn_oracle.client_train(w0, X, y, 11, 4, 2, E, bs, 0.05, 62, emulate_bf16=True)
    errs = {nm: "%.1e" % (np.linalg.norm((got[o:o+s] - w0d[o:o+s]) - (want[o:o+s] - w0d[o:o+s]))
                          / np.linalg.norm(want[o:o+s] - w0d[o:o+s])) for nm, o, s, _ in spec.columns()}
    print(n, bs, E, errs, flush=True)
