"""One C4 round (ResNet-18-GN, 100 of 1000 clients) after a warm-up round --
a short command for ncu launch lists of the C4 workload."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda", 0)
eng = bench.c4_engine(dev, 3)
eng.run_round(0)
torch.cuda.synchronize()
eng.run_round(1)
torch.cuda.synchronize()
print("ok")
