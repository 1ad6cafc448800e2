"""C5 batched sims: fp64 against mixed precision (fp32 stage to rtol_lo, fp64 finish to 1e-12),
10 sims x argv[1] steps; bench.c5_batched."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402

dev = torch.device("cuda:0")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
for mixed in [float(v) if v != "none" else None for v in (sys.argv[2:] or ["none", "1e-6"])]:
    r = bench.c5_batched(hf, torch, dev, 1, nsims=10, nsteps=steps, mixed=mixed)
    print(json.dumps({"mixed": mixed, "sims_per_s": round(r["sims_per_s"] * steps / 300, 4),
                      "ms_per_system_step": round(r["ms_per_step"], 3), "iters": round(r["pcg_iters_per_step"], 1),
                      "front_max": r["front_face_max_C"]}), flush=True)
