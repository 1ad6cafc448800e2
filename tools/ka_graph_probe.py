"""Kernel A at C3: plain back-to-back replay (hf_time_kernel_a) against the graph chain with the
loop's programmatic edges (hf_time_kernel_a_graph), next to the PCG iteration of the step graph."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
p = synth.c3(nsteps=13)
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
up = torch.zeros_like(u)
hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=p.rtol)
hf.hf_set_step_flush(ctx, 1)
st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 10, F, u, up, 3, rtol=p.rtol)
hf.hf_set_step_flush(ctx, 0)
print(f"iteration {1e3 * st['ms_steps'] / st['total_iters']:.2f} us", flush=True)
for _ in range(3):
    print(f"kernel A plain {hf.hf_time_kernel_a(ctx, 200) * 1e3:.2f} us, graph chain "
          f"{hf.hf_time_kernel_a_graph(ctx, 200) * 1e3:.2f} us", flush=True)
