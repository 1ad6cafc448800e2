"""A/B timing of the C3 time step for a package tree (argv[1]: directory holding
paper_1905_07622_b200/ and synth/): 10 steps after a 3-step warm-up, L2 flushed per step."""
import sys

root = sys.argv[1]
sys.path.insert(0, root)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

print("package:", hf.__file__)
dev = torch.device("cuda:0")
p = synth.c3(nsteps=13)
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
for rep in range(3):
    u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=p.rtol)
    hf.hf_set_step_flush(ctx, 1)
    st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 10, F, u, up, 3, rtol=p.rtol)
    hf.hf_set_step_flush(ctx, 0)
    ms = st["ms_steps"] / 10
    print(f"rep {rep}: {ms:.4f} ms/step, {1e3 * st['ms_steps'] / st['total_iters']:.2f} us/iter, iters {st['total_iters']}")
    t = hf.hf_time_kernel_a(ctx, 200) if hasattr(hf, "hf_time_kernel_a") else None
    print("   kernel A", t)
