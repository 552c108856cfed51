"""Low-rank (lazy) vs direct fc1: per-tensor difference of one client's local
run, plus the h / dp2 workspaces of the last sweep (diagnostic)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2303_01778_b200 as pb
from paper_2303_01778_b200 import cnn
from paper_2303_01778_b200.core import ClientProfile, DataSlice
from paper_2303_01778_b200.models import cnn_init, cnn_spec
from paper_2303_01778_b200.trainer import NamedParams

ds = pb.generate(4000, 784, 62, seed=0)
spec = cnn_spec(62)
w0 = cnn_init(spec, seed=3)
for n, bs, E, sweeps in [(20, 20, 1, 1), (40, 20, 1, 2), (100, 20, 1, 5), (45, 16, 1, 0), (20, 20, 3, 0)]:
    X, y = ds.features[100:100 + n], ds.labels[100:100 + n]
    out, ws = {}, {}
    for mode in ("0", "1"):
        os.environ["PB_CNN_LAZY"] = mode
        os.environ["PB_CNN_MAX_SWEEPS"] = str(sweeps)
        plugin = pb.FedAvg(lr=0.05, batch_size=bs)
        glob = plugin.init_global(NamedParams.from_flat(spec, w0))
        rep = pb.client_execute(plugin, ClientProfile(11, n, DataSlice(X, y, np.arange(n))), glob,
                                None, E, bs, 0.05, seed=4, round_num=2)
        torch.cuda.synchronize()
        out[mode] = np.concatenate([rep.client_result.numpy(nm).reshape(-1) for nm in spec.names])
        b = min(bs, n)
        ws[mode] = {k: cnn._WS.buf[k].view(torch.float32)[:b * w].cpu().numpy().copy()
                    for k, w in (("h", 512), ("dp2", 3136))}
    rel = {}
    for nm, o, s, _ in spec.columns():
        d0 = out["0"][o:o + s] - w0.reshape(-1)[o:o + s]
        d1 = out["1"][o:o + s] - w0.reshape(-1)[o:o + s]
        rel[nm] = "%.1e" % (np.linalg.norm(d1 - d0) / max(np.linalg.norm(d0), 1e-30))
    wsr = {k: "%.1e" % (np.linalg.norm(ws["1"][k] - ws["0"][k]) / max(np.linalg.norm(ws["0"][k]), 1e-30))
           for k in ws["0"]}
    print(n, bs, E, sweeps, "update diff", rel, "ws", wsr, flush=True)

# one sweep, inspect the fc1 forward inputs/outputs directly
n, bs = 20, 20
X, y = ds.features[100:100 + n], ds.labels[100:100 + n]
res = {}
for mode in ("0", "1"):
    os.environ["PB_CNN_LAZY"] = mode
    os.environ["PB_CNN_MAX_SWEEPS"] = "1"
    plugin = pb.FedAvg(lr=0.05, batch_size=bs)
    glob = plugin.init_global(NamedParams.from_flat(spec, w0))
    pb.client_execute(plugin, ClientProfile(11, n, DataSlice(X, y, np.arange(n))), glob, None, 1, bs,
                      0.05, seed=4, round_num=2)
    torch.cuda.synchronize()
    res[mode] = {"h": cnn._WS.buf["h"].view(torch.float32)[:n * 512].view(n, 512).clone(),
                 "p2": (cnn._WS.buf["p2"].view(torch.float32)[:n * 3136] if mode == "0"
                        else cnn._LZ.buf["hx"][:n * 3136]).view(n, 3136).clone()}
W = torch.as_tensor(w0.reshape(-1), device="cuda")
o = dict((nm, (oo, s, sh)) for nm, oo, s, sh in spec.columns())
W1 = W[o["fc1_w"][0]:o["fc1_w"][0] + o["fc1_w"][1]].view(512, 3136)
b1 = W[o["fc1_b"][0]:o["fc1_b"][0] + 512]
for mode in ("0", "1"):
    p2 = res[mode]["p2"]
    ref = torch.relu(p2.double() @ W1.double().t() + b1.double())
    print(mode, "p2 vs direct p2 %.2e" % float((p2 - res["0"]["p2"]).norm() / res["0"]["p2"].norm()),
          "h vs torch(p2) %.2e" % float((res[mode]["h"].double() - ref).norm() / ref.norm()),
          "h norm %.3e" % float(res[mode]["h"].norm()))
wt = cnn._LZ.buf["w0t"][:3136 * 512].view(3136, 512)
print("w0t vs W1^T %.2e" % float((wt - W1.t()).norm() / W1.norm()))
