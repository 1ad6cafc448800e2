"""bench.py's C5 batched leg alone: python tools/c5repro.py [nsteps] [nsims]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402

dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 2
r = bench.c5_batched(hf, torch, dev, 1, nsims=ns, nsteps=n)
print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items() if k != "depths_mm"})
