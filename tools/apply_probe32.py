"""fp32 / fp64 512^3 apply kernel times (bench.py legs), for A/B comparisons of library builds."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402
dev = torch.device("cuda:0")
for prec in (32, 64):
    r = bench.apply_512(hf, torch, dev, 6544.0, prec)
    print(f"fp{prec} apply 512^3: {r['ms']:.4f} ms frac {r['frac']:.3f}", flush=True)
r = bench.variant_c3(hf, torch, dev, 32, 1e-6)
print(f"fp32 C3 rtol 1e-6: {r['ms_per_step']:.3f} ms/step {r['us_per_pcg_iter']:.1f} us/iter", flush=True)
