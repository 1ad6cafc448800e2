"""512^3 apply (pairs, material ids, fp32) at the tile height in HF_TILE_R: bench.apply_512."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402

dev = torch.device("cuda:0")
peak = bench.measured_peaks()[0]
for name, kw in (("pairs", {}), ("ids", {"ids": True}), ("fp32", {"prec": 32})):
    r = bench.apply_512(hf, torch, dev, peak, **kw)
    print(json.dumps({"R": os.environ.get("HF_TILE_R", "default"), "coef": name, "ms": r["ms"], "frac": r["frac"]}),
          flush=True)
