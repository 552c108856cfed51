import sys, json; sys.path.insert(0, '.')
import torch, bench
print(json.dumps(bench.resnet_round_bench(torch.device("cuda", 0))))
