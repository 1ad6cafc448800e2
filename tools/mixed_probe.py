"""Mixed precision (hf_set_mixed) vs plain fp64 on C3 and on a 256^3 grid: ms/step, iterations."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for n in (100, 256):
    p = synth.c3(n_nodes_axis=n, nsteps=8)
    for mode in ("fp64", "mixed"):
        for rlo in ((1e-6,) if mode == "fp64" else (1e-3, 1e-5)):
            ctx = hf.hf_create(p.grid, 0)
            if mode == "mixed":
                hf.hf_set_mixed(ctx, 1, rlo)
            hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
            F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
            hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
            u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
            up = torch.zeros_like(u)
            hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=p.rtol)
            lo0 = hf.hf_mixed_iters(ctx) if mode == "mixed" else 0
            hf.hf_set_step_flush(ctx, 1)
            st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 5, F, u, up, 3, rtol=p.rtol)
            lo = (hf.hf_mixed_iters(ctx) - lo0) if mode == "mixed" else 0
            print(f"n={n} {mode} rtol_lo={rlo if mode == 'mixed' else '-'}: {st['ms_steps'] / 5:.3f} ms/step, "
                  f"fp64 it/step {st['total_iters'] / 5:.1f}, fp32 it/step {lo / 5:.1f}, |u| {float(u.norm()):.10e}",
                  flush=True)
            del ctx
