"""Fixed cost of a C3 time step: the step graph at a loose tolerance (PCG stops after 0-2
iterations) vs rtol 1e-12, L2 flushed before every step (bench protocol)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
p = synth.c3(nsteps=20)
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
for flush in (1, 0):
    for rtol in (1e-12, 1e-3, 0.5):
        u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
        up = torch.zeros_like(u)
        hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=1e-12)
        hf.hf_simulate_resume(ctx, p.theta, p.dt, 1, F, u.clone(), up.clone(), 3, rtol=rtol)  # graph for rtol
        hf.hf_set_step_flush(ctx, 1 if flush else 0)
        st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 10, F, u, up, 3, rtol=rtol)
        hf.hf_set_step_flush(ctx, 0)
        ms = (st["ms_steps"] if flush else st["ms_total"]) / 10
        print(f"flush={flush} rtol={rtol:g}: {ms * 1e3:.1f} us/step, {st['total_iters'] / 10:.1f} it/step", flush=True)
