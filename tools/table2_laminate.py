"""Paper Table 2 workload: the laminate [-15,15]^2 x [0,10] mm, f = 1 on
x3 = 0, steel below x3 = 5 / oxide above, 50 CN steps of dt = 0.01, Jacobi-PCG with
relative tolerance 1e-6, C = (30s, 30s, 10s) for s = 1..6 (10.5k .. 2.00M DoF).  Runs both the
paper's element (6 P1 tets per voxel, hf_set_element 1) and the Q1 hexahedron and prints total
PCG iterations and wall time next to the paper's FG DbD column (D700, context only)."""
import json
import os

import numpy as np
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

PAPER = {1: (287, 0.48), 2: (344, 1.7), 3: (567, 2.0), 4: (780, 5.4), 5: (1047, 13.0), 6: (1278, 26.0)}
dev = torch.device("cuda:0")
rows = []
for s in range(1, 7):
    p = synth.laminate(s)
    # the paper's material assignment: per vertex (steel for x3 <= 5), averaged per element
    z = np.repeat(p.grid.origin[2] + np.arange(p.grid.ne[2] + 1) * p.grid.h[2], (p.grid.ne[0] + 1) * (p.grid.ne[1] + 1))
    steel = z <= 5.0 + 1e-9
    kn = np.where(steel, synth.STEEL[1], synth.OXIDE[1])
    cn = np.where(steel, synth.STEEL[0], synth.OXIDE[0])
    for elem in ("tetv", 1, 0):
        ctx = hf.hf_create(p.grid, 0)
        hf.hf_set_element(ctx, 0 if elem == 0 else 1)
        if elem == "tetv":
            hf.hf_set_vertex_coefficients(ctx, torch.tensor(kn, device=dev), torch.tensor(cn, device=dev))
        else:
            hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
        F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
        hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
        u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
        hf.hf_simulate(ctx, p.theta, p.dt, 2, F, u, rtol=p.rtol)      # warm-up (graph build)
        u.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        r = {"s": s, "dofs": p.grid.n_nodes,
             "element": {"tetv": "6 P1 tets, vertex-averaged materials (paper)", 1: "6 P1 tets, per-voxel materials",
                         0: "Q1 hex"}[elem],
             "total_iters": st["total_iters"], "seconds": round(wall, 4), "ms_per_iter": round(wall * 1e3 / st["total_iters"], 4),
             "paper_fg_dbd_iters": PAPER[s][0], "paper_fg_dbd_seconds_D700": PAPER[s][1]}
        rows.append(r)
        print(json.dumps(r), flush=True)
        del ctx
