"""Phase trace of k_bwd_conv in a C2 round: per-sample timestamps of one CTA
(block (0, 0)) of the first launch after arming -- a dense sweep.  Needs the
trace build (run on the GPU box):

    PB_NVCC_DEFS=-DPB_PHASE_TRACE python -m paper_2303_01778_b200.build --force
    python tools/phase_probe.py

Worker thread 0: 0 start, 1 dz_free, 2 planes built (bias-partial sync;
warps 12-15 read H of sample i-2 first), 3 epilogue start, 4 tile 0 in TMEM,
5 tile-0 halo sync, 6 G free (tile 0), 7 G tile 0 written, 8 G free (tile 1),
9 G tile 1 written, 11 end.  MMA thread: 12 dz_full, 13 dgrad issued, 14
conv1 MMAs of sample i-1 issued, 15 dgrad complete.  Times in us from the
iteration's start (column 0; iteration 0 from its column 12).
"""
import ctypes
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_2303_01778_b200 as pb  # noqa: E402
from paper_2303_01778_b200 import _lib  # noqa: E402
import torch  # noqa: E402

dev = torch.device("cuda", 0)
data, sizes = bench.build_device_data(dev)
profiles = bench.light_profiles(sizes)
cfg = pb.SimConfig(total_clients=bench.M_TOTAL, concurrent_clients=bench.M_ROUND, num_devices=1,
                   total_rounds=4, warmup_rounds=1, seed=0, scheme="PARROT")
eng = pb.SimulationEngine(cfg, pb.FedAvg(lr=bench.LR, batch_size=bench.BS), profiles,
                          pb.make_device_models(1), model="cnn", client_data=data)
eng.run_round(0)
torch.cuda.synchronize()
dll = _lib.lib._dll
if not hasattr(dll, "pb_phase_arm"):
    sys.exit("not a PB_PHASE_TRACE build")
assert dll.pb_phase_arm() == 0
eng.run_round(1)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 64 * 16))()
assert dll.pb_phase_read(buf) == 0
all_ph = np.frombuffer(buf, dtype=np.uint64).reshape(2, 64, 16).astype(np.int64)
tables = {
    "k_bwd_conv": ["start", "dz_free", "built", "epi", "tile0", "halo0", "g_free0", "G0", "g_free1", "G1",
                   "-", "end", "m:dz_full", "m:dgrad", "m:conv1", "m:done"],
    # k_fwd, worker thread 0 of sample i: 0 start, 1 conv1(i) done, 2 A(i+1)
    # built, 3 p1(i) written; conv2 epilogue of i-1: 4 conv2 done, 5/8 half
    # tile in smem, 6/9 pooled; 11 end.  MMA thread: 12 p1 ready, 13 conv2 issued
    "k_fwd": ["start", "c1_done", "A built", "p1 ready", "c2_done", "sZ h0", "pool h0", "-", "sZ h1",
              "pool h1", "-", "end", "m:p1", "m:conv2", "-", "-"],
}
for kern, (name, names) in enumerate(tables.items()):
    ph = all_ph[kern]
    print(name)
    print("iter " + " ".join(f"{n:>9s}" for n in names))
    for it in range(64):
        row = ph[it]
        if not row.any():
            break
        t0 = row[0] if row[0] else row[12]
        print(f"{it:4d} " + " ".join(f"{(v - t0) / 1e3:9.2f}" if v else f"{'-':>9s}" for v in row))
    starts = ph[:, 0][ph[:, 0] > 0]
    if len(starts) > 2:
        print("iteration period us (median):", float(np.median(np.diff(starts))) / 1e3)

# low-rank fc1 kernels: CTA (0,0,0) of the 6th launch of k_lz_fwd / k_lz_bwd
# in a round (sweep 5): per ring chunk the time its operands landed (us from
# the ring start), then ring end and kernel end
if hasattr(dll, "pb_lz_phase_arm"):
    assert dll.pb_lz_phase_arm(5) == 0
    eng.run_round(2)
    torch.cuda.synchronize()
    lbuf = (ctypes.c_ulonglong * (2 * 64 * 4))()
    assert dll.pb_lz_phase_read(lbuf) == 0
    lz = np.frombuffer(lbuf, dtype=np.uint64).reshape(2, 64, 4).astype(np.int64)
    for kern, name in enumerate(("k_lz_fwd", "k_lz_bwd")):
        t0 = lz[kern, 63, 0]
        if not t0:
            continue
        chunks = [(c, (lz[kern, c, 0] - t0) / 1e3) for c in range(63) if lz[kern, c, 0]]
        print(name, "chunks landed (us):", " ".join(f"{c}:{t:.2f}" for c, t in chunks))
        print(name, f"ring end {(lz[kern, 63, 1] - t0) / 1e3:.2f} us, kernel end {(lz[kern, 63, 2] - t0) / 1e3:.2f} us")
