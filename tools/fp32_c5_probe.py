"""Convergence of the fp32 variant on C5 (one system): iterations and status per rtol."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1905_07622_b200 as hf  # noqa: E402
dev = torch.device("cuda:0")
p = synth.c5(0, nsteps=300)
for prec in (64, 32):
    for rtol in (1e-5, 1e-6, 1e-7):
        for rep in (50, 0):
            ctx = hf.hf_create(p.grid, 0)
            if prec == 32:
                hf.hf_set_precision(ctx, 32)
            hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
            F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
            hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
            u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
            st = hf.hf_simulate(ctx, p.theta, p.dt, 5, F, u, rtol=rtol, max_iter=3000, replace_every=rep,
                                raise_on_noconv=False)
            print(prec, rtol, "replace", rep, "rc", st["rc"], "iters", st["total_iters"], "failed", st["first_failed_step"],
                  "umax", float(u.max()), flush=True)
