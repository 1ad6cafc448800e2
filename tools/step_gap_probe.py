"""C3 steps back to back: whole-call device time vs the sum of per-step event intervals
(hf_set_step_flush 2: no flush), i.e. the gaps between consecutive step graphs."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
p = synth.c3(nsteps=30)
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
for mode in (0, 2, 1, 2, 0):
    u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=p.rtol)
    hf.hf_set_step_flush(ctx, mode)
    st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 20, F, u, up, 3, rtol=p.rtol)
    hf.hf_set_step_flush(ctx, 0)
    print(f"mode {mode}: call {st['ms_total'] / 20:.4f} ms/step, steps {st['ms_steps'] / 20:.4f} ms/step, "
          f"it/step {st['total_iters'] / 20:.1f}", flush=True)
