"""bench.py with host-side timers on the calls a CNN round makes before its
first kernel (diagnostics for e2e outliers): python tools/bench_trace.py [bench args]"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2303_01778_b200._lib as L
import paper_2303_01778_b200.cnn as cnn
import paper_2303_01778_b200.trainer as tr


def timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        r = fn(*a, **k)
        dt = (time.perf_counter() - t) * 1e3
        if dt > 3.0:
            print(f"    SLOW {name}: {dt:.1f} ms", file=sys.stderr, flush=True)
        return r
    return w


cnn.h2d = timed("h2d", L.h2d)
tr.GroupInputs.upload = timed("GroupInputs.upload", tr.GroupInputs.upload)
tr.GroupInputs.__init__ = timed("GroupInputs.__init__", tr.GroupInputs.__init__)
_orig = L.lib.pb_cnn_train_group
L.lib.pb_cnn_train_group = timed("pb_cnn_train_group", _orig)
cnn._LZ.get = timed("lazy workspace get", cnn._LZ.get)
cnn._WS.get = timed("workspace get", cnn._WS.get)
torch.Tensor.zero_ = timed("zero_", torch.Tensor.zero_)
import bench  # noqa: E402
sys.argv = ["bench.py"] + sys.argv[1:]
bench.main()
