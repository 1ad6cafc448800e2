"""C3 time step on a 1-rank peer-memory slab (transport 1, in-process) against the plain
context: the cost of the mailbox protocol itself (10 steps after 3, L2 flushed per step)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
p = synth.c3(nsteps=13)
grp = hf.hf_local_group_create(1)
for name in ("plain", "slab1", "plain", "slab1"):
    ctx = hf.hf_create(p.grid, 0) if name == "plain" else hf.hf_create_slab(p.grid, 0, 1, grp, transport=1, device=0)
    hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
    F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = torch.zeros(ctx.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=p.rtol)
    hf.hf_set_step_flush(ctx, 1)
    st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 10, F, u, up, 3, rtol=p.rtol)
    hf.hf_set_step_flush(ctx, 0)
    print(f"{name}: {st['ms_steps'] / 10:.3f} ms/step, {1e3 * st['ms_steps'] / st['total_iters']:.2f} us/iter, "
          f"iters {st['total_iters']}", flush=True)
    del ctx
hf.hf_local_group_destroy(grp)
