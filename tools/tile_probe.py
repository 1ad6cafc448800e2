"""C3 time step and kernel A timing for the tile height in HF_TILE_R (and HF_ZCHUNK etc.):
10 steps after a 3-step warm-up, L2 flushed per step; kernel A over 200 back-to-back launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
p = synth.c3(n_nodes_axis=n, nsteps=13)
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
ref = None
for rep in range(2):
    u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=p.rtol)
    hf.hf_set_step_flush(ctx, 1)
    st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 10, F, u, up, 3, rtol=p.rtol)
    hf.hf_set_step_flush(ctx, 0)
    ka = hf.hf_time_kernel_a(ctx, 200)
    print(f"R={os.environ.get('HF_TILE_R', 'default')} zchunk={os.environ.get('HF_ZCHUNK', '-')}: "
          f"{st['ms_steps'] / 10:.4f} ms/step, {1e3 * st['ms_steps'] / st['total_iters']:.2f} us/iter, "
          f"iters {st['total_iters']}, kernel A {ka * 1e3 if ka < 1 else ka:.2f} us", flush=True)
    ref = u.cpu().numpy()
np.save(f"/tmp/u_R{os.environ.get('HF_TILE_R', 'd')}.npy", ref)
