"""Probe of the on-chip PCG plan and a C1/C3 run (development aid)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for name, p in (("c1", synth.c1()), ("c3", synth.c3(nsteps=int(sys.argv[1]) if len(sys.argv) > 1 else 5))):
    ctx = hf.hf_create(p.grid, 0)
    kc, inv = np.unique(np.stack([p.k, p.c], 1), axis=0, return_inverse=True)
    hf.hf_set_material_ids(ctx, inv.astype(np.uint8).ravel(), kc[:, 0], kc[:, 1])
    print(name, hf.hf_resident_plan(ctx), flush=True)
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    for mode in (1, 0):
        hf.hf_set_resident(ctx, mode)
        if mode == 1:
            hf.hf_resident_profile(ctx, 1)
        u = torch.tensor(p.u0, device=dev)
        hf.hf_simulate(ctx, p.theta, p.dt, 1, F, u, rtol=p.rtol)      # warm-up (graph build)
        u = torch.tensor(p.u0, device=dev)
        torch.cuda.synchronize()
        t0 = time.time()
        st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol, raise_on_noconv=False)
        torch.cuda.synchronize()
        t = time.time() - t0
        it = max(st["total_iters"], 1)
        print(f"  mode {mode}: {st}, {1e3 * st['ms_total'] / p.nsteps:.1f} us/step, "
              f"{1e3 * st['ms_total'] / it:.2f} us/iter, |u| {float(u.norm()):.6e}, plan {hf.hf_resident_plan(ctx)['last_used']}",
              flush=True)
        if mode == 1:
            pr = hf.hf_resident_profile(ctx, 0)
            n = max(pr["iters"], 1)
            print("   per iteration (CTA 0):", {k: round(v / n, 3) for k, v in pr.items() if k.endswith("us") and not k.startswith("max")}, flush=True)
            print("   per iteration (max over CTAs):", {k: round(v / n, 3) for k, v in pr.items() if k.endswith("us") and k.startswith("max")}, flush=True)
