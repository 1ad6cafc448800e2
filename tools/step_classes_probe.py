"""C3: per-class kernel times of the host-loop profiling driver (each launch between its own event
pair, so absolute values include per-launch event overhead): the per-step kernels (RHS, init,
step end) against the PCG kernels."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
p = synth.c3(nsteps=8)
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
up = torch.zeros_like(u)
hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=p.rtol)
hf.hf_profile(ctx, True)
st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 5, F, u, up, 3, rtol=p.rtol)
prof = hf.hf_profile_read(ctx)
hf.hf_profile(ctx, False)
steps = 5
for k, (ms, n) in prof.items():
    print(f"{k:16s} {n:6d} launches  {ms / max(n, 1) * 1e3:8.2f} us/launch  {ms / steps * 1e3:9.1f} us/step")
print("iterations/step", st["total_iters"] / steps)
