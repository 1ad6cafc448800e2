"""Median CUDA-event time of the 512^3 operator apply (bench.py's apply_512 leg) a few times."""
import os, sys, statistics
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402
dev = torch.device("cuda:0")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    r = bench.apply_512(hf, torch, dev, 6544.0)
    print(f"apply 512^3: {r['ms']:.4f} ms  {r['achieved']:.0f} GB/s  frac {r['frac']:.3f}", flush=True)
