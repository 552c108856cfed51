import sys, time
sys.path.insert(0, ".")
import paper_2303_01778_b200.cnn as cnn
import paper_2303_01778_b200.aggregate as agg
import paper_2303_01778_b200._lib as L
orig_h2d = L.h2d
def traced_h2d(a, device):
    t = time.perf_counter(); r = orig_h2d(a, device); dt = time.perf_counter() - t
    if dt > 2e-3: print(f"    h2d {a.nbytes} B took {dt*1e3:.1f} ms", file=sys.stderr, flush=True)
    return r
cnn.h2d = traced_h2d; agg.h2d = traced_h2d
orig_fold = cnn.LazyFc1.fold
def traced_fold(self, *a, **k):
    t = time.perf_counter(); orig_fold(self, *a, **k); print(f"    lazy fold {1e3*(time.perf_counter()-t):.1f} ms", file=sys.stderr, flush=True)
cnn.LazyFc1.fold = traced_fold
orig_kfold = agg.K.fold_group
def traced_kfold(*a, **k):
    t = time.perf_counter(); orig_kfold(*a, **k); dt = time.perf_counter() - t
    if dt > 2e-3: print(f"    K.fold_group {dt*1e3:.1f} ms", file=sys.stderr, flush=True)
agg.K.fold_group = traced_kfold
exec(open("tools/e2e_diag.py").read())
