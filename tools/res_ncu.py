"""One C3 time step through the on-chip PCG (for ncu captures of k_pcg_res)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
p = synth.c3(n_nodes_axis=n, nsteps=2)
ctx = hf.hf_create(p.grid, 0)
kc, inv = np.unique(np.stack([p.k, p.c], 1), axis=0, return_inverse=True)
hf.hf_set_material_ids(ctx, inv.astype(np.uint8).ravel(), kc[:, 0], kc[:, 1])
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
u = torch.tensor(p.u0, device=dev)
print(hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol), hf.hf_resident_plan(ctx))
