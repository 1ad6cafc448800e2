import sys, os, torch
sys.path.insert(0, os.getcwd())
import bench, paper_1905_07622_b200 as hf
dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
print(bench.c5_batched(hf, torch, dev, 1, nsims=2, nsteps=n))
