"""Compare CNN client training under different samples-per-CTA settings."""
import os, subprocess, sys
sys.path.insert(0, ".")
import numpy as np
CODE = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2303_01778_b200 as pb
from paper_2303_01778_b200.core import ClientProfile, DataSlice
from paper_2303_01778_b200.models import cnn_init, cnn_spec
from paper_2303_01778_b200.trainer import NamedParams
ds = pb.generate(4000, 784, 62, seed=0)
n = 57
X, y = ds.features[100:100 + n], ds.labels[100:100 + n]
spec = cnn_spec(62)
w0 = cnn_init(spec, seed=3)
plugin = pb.FedAvg(lr=0.05, batch_size=20)
glob = plugin.init_global(NamedParams.from_flat(spec, w0))
rep = pb.client_execute(plugin, ClientProfile(11, n, DataSlice(X, y, np.arange(n))), glob, None, 2, 20, 0.05, seed=4, round_num=2)
got = np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names])
np.save(sys.argv[1], got)
'''
outs = {}
for spb in ("-1", "-10", "-20", "-1"):
    env = dict(os.environ, PB_CNN_SPB=spb)
    f = f"/tmp/spb{spb}.npy"
    r = subprocess.run([sys.executable, "-c", CODE, f], env=env, capture_output=True, text=True)
    if r.returncode:
        print(spb, "ERR", r.stderr[-500:]); continue
    outs.setdefault(spb, []).append(np.load(f))
from paper_2303_01778_b200.models import cnn_spec
spec = cnn_spec(62)
base = outs["-10"][0]
for k, vs in outs.items():
    for v in vs:
        print(k, {n: float(np.abs(v[o:o+s] - base[o:o+s]).max()) for n, o, s, _ in spec.columns()})
