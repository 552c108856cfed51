"""C5 aggregation microbench kernel alone (1000 x 11.17M fp32 fold_group),
for an ncu capture: ncu -k regex:fold_group ... python tools/c5_fold.py"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402

print(bench.aggregation_microbench(1, torch.device("cuda", 0)))
