"""State gather/scatter bandwidth vs a plain torch copy of the same bytes."""
import sys, json
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
from paper_2303_01778_b200 import _kernels as K

dev = torch.device("cuda", 0)
print(json.dumps(bench.state_microbench(dev))[:200])
print(json.dumps(bench.state_microbench(dev, P=1_690_046))[:200])
P, slots, g = 11_173_962, 1000, 100
store = torch.randn(slots, P + 2, device=dev)[:, :P]
work = torch.empty(g, P + 2, device=dev)[:, :P]
for name, rows in (("random", np.random.default_rng(3).choice(slots, g, replace=False)),
                   ("contiguous", np.arange(g))):
    slot = torch.from_numpy(rows.astype(np.int32)).to(dev)
    for fn, lab in ((lambda: K.state_gather(work, store, slot), "gather"),
                    (lambda: K.state_scatter(store, work, slot), "scatter"),
                    (lambda: work.copy_(store[:g]), "torch copy")):
        fn(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = min(ts)
        print(name, lab, f"{ms:.3f} ms {8.0 * g * P / ms / 1e6:.0f} GB/s")
