"""Debug aid: train one 57-sample client (bs 20, 2 epochs) on the low-rank
fc1 after poisoning the history buffers with a value, per sweep count;
prints whether the result matches the clean run."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2303_01778_b200 as pb
import paper_2303_01778_b200.cnn as cnn
from paper_2303_01778_b200.core import ClientProfile, DataSlice
from paper_2303_01778_b200.models import cnn_init, cnn_spec
from paper_2303_01778_b200.trainer import NamedParams
import os

spec = cnn_spec(62)
ds = pb.generate(4000, 784, 62, seed=0)
X, y = ds.features[:57], ds.labels[:57]
w0 = cnn_init(spec, seed=1)


def run(sweeps):
    os.environ["PB_CNN_MAX_SWEEPS"] = str(sweeps)
    plugin = pb.FedAvg(lr=0.05, batch_size=20, collect_local_loss=True)
    glob = plugin.init_global(NamedParams.from_flat(spec, w0))
    try:
        rep = pb.client_execute(plugin, ClientProfile(11, 57, DataSlice(X, y, np.arange(57))), glob,
                                None, 2, 20, 0.05, seed=4, round_num=2)
    except Exception as e:
        return None, repr(e)[:80]
    return np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names]), ""


run(0)

keys = [k for k in cnn._LZ.buf if k not in cnn._LZ.HISTORY]
cnn._LZ.dirty = True
clean, _ = run(0)
for key in keys:
    for val in (float("nan"), 0.0, 1.0):
        for t in cnn._LZ.buf.values():
            t.zero_()
        cnn._LZ.dirty = False
        cnn._LZ.buf[key].fill_(val)
        got, err = run(0)
        if got is None:
            print(key, val, err)
        else:
            d = np.abs(got - clean)
            print(key, val, [(nm, float(d[o:o + s_].max())) for nm, o, s_, _ in spec.columns() if np.any(d[o:o + s_] != 0)])
