"""C4 (512^3) time steps: fp64 against mixed precision at several rtol_lo (bench.c4_steps)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402

dev = torch.device("cuda:0")
peak = bench.measured_peaks()[0]
for mixed in [float(v) if v != "none" else None for v in (sys.argv[1:] or ["none", "1e-6"])]:
    r = bench.c4_steps(hf, torch, dev, peak, mixed=mixed)
    print(json.dumps({"mixed": mixed, "ms_per_step": round(r["ms_per_step"], 2), "fp64_iters_per_step": r["pcg_iters_per_step"]}),
          flush=True)
