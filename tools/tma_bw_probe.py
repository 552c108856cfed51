"""TMA read bandwidth: 16 KB boxes of 128 rows x 128 B with a row pitch
(the history layouts of the low-rank fc1) vs the same bytes as contiguous
16 KB tiles, per CTA count.  python tools/tma_bw_probe.py"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2303_01778_b200 import _lib  # noqa: E402

lib = _lib.lib
dev = torch.device("cuda", 0)
sink = torch.zeros(4096, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream().cuda_stream
for cols, rows, ctas_list in ((3136, 128 * 148 * 4, (148, 74)), (262144, 128 * 8, (8, 4)),
                              (262144, 128 * 64, (64, 32))):
    buf = torch.zeros(rows * cols, device=dev)
    for ctas in ctas_list:
        rpc = rows // ctas
        nbox = min((rpc // 128) * (cols // 32), 512)
        for mode in (0, 1):
            for _ in range(2):
                assert lib.pb_tma_bw_probe(buf.data_ptr(), mode, rows, cols, ctas, nbox, sink.data_ptr(), st) == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert lib.pb_tma_bw_probe(buf.data_ptr(), mode, rows, cols, ctas, nbox, sink.data_ptr(), st) == 0
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            gb = ctas * nbox * 16384 / 1e9
            print(f"pitch {cols * 4:>8} B  ctas {ctas:3d}  {'blocked' if mode else 'pitched'}: "
                  f"{gb / ms * 1e3:7.0f} GB/s total, {gb / ms * 1e3 / ctas:6.1f} GB/s per CTA ({ms:.3f} ms)",
                  flush=True)
    del buf
