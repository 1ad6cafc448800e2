"""512^3 apply: pairs / ids / fp32 at tile heights R = 2 and 4 (HF_TILE_R at context creation)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402

dev = torch.device("cuda:0")
peak = bench.measured_peaks()[0]
for R in ("4", "2"):
    os.environ["HF_TILE_R"] = R
    for kind in ("pairs", "ids", "fp32"):
        if kind == "fp32":
            r = bench.apply_512(hf, torch, dev, peak, prec=32)
        else:
            r = bench.apply_512(hf, torch, dev, peak, ids=(kind == "ids"))
        print(f"R={R} {kind}: {r['ms']:.4f} ms, frac {r['frac']:.3f}", flush=True)
        torch.cuda.empty_cache()
