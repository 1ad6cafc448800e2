"""C5 batched sims throughput (bench.c5_batched) under the current environment (tile height etc.)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402

dev = torch.device("cuda:0")
for prec, rtol in ((64, None), (32, 1e-6)):
    r = bench.c5_batched(hf, torch, dev, 1, nsteps=int(os.environ.get("C5_STEPS", "100")), prec=prec, rtol=rtol)
    print(f"C5 fp{prec} R={os.environ.get('HF_TILE_R', 'default')}: {r['sims_per_s_per_gpu']:.3f} sims/s/GPU, "
          f"{r['ms_per_step']:.3f} ms/step, it/step {r['pcg_iters_per_step']:.1f}", flush=True)
