"""One apply of each ablation implementation (hf_apply_impl 1, 2) at 512^3 nodes, for an ncu
capture of k_ebe_pass1 / k_ebe_pass2 / k_dbd (tools/ablation.py does the timing)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
g = synth.c4_grid(int(sys.argv[1]) if len(sys.argv) > 1 else 512)
gen = torch.Generator(device=dev).manual_seed(0)
k = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) * 121.5 + 1.0
c = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) + 1.0
ctx = hf.hf_create(g, 0)
hf.hf_set_coefficients(ctx, k, c)
del k, c
u = torch.randn(g.n_nodes, dtype=torch.float64, device=dev, generator=gen)
y = torch.empty_like(u)
hf.hf_ablation_prepare(ctx, 0.005, 1.0)
for impl in (1, 2):
    hf.hf_apply_impl(ctx, impl, 0.005, 1.0, 1.0, u, None, y)
torch.cuda.synchronize()
print("ok")
