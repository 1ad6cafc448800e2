"""Kernel-A duration vs z extent at a fixed 100 x 100 cross-section (fixed + per-plane cost)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for nzn in [int(a) for a in (sys.argv[1:] or [13, 25, 50, 100, 200, 400])]:
    g = synth.Grid((99, 99, nzn - 1), (0.2, 0.2, 0.2))
    ids = synth.inclusion_ids(g, seed=0)
    k, c = synth.ids_to_fields(ids)
    ctx = hf.hf_create(g, 0)
    hf.hf_set_coefficients(ctx, torch.tensor(k, device=dev), torch.tensor(c, device=dev))
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = torch.zeros(g.n_nodes, dtype=torch.float64, device=dev)
    st = hf.hf_simulate(ctx, 0.5, 0.01, 3, F, u)
    ka = hf.hf_time_kernel_a(ctx, 200)
    print(f"nz={nzn:4d} nodes={g.n_nodes:8d} kernel A {ka * 1e3:7.2f} us  it/step {st['total_iters'] / 3:.1f}  "
          f"ms/step {st['ms_total'] / 3:.3f}", flush=True)
    del ctx
