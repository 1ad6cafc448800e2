"""A/B of the coefficient layouts (material ids vs fp64 pairs): C3 ms/step and kernel-A time,
512^3 apply time.  HF_TILE_R=2/4 forces the tile height."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
what = sys.argv[1:] or ["c3", "a512"]
if "c3" in what:
    for coef in ("ids", "pairs", "ids", "pairs"):
        r = bench.variant_c3(hf, torch, dev, 64, 1e-12, coef=coef)
        p = synth.c3(nsteps=4)
        ctx = hf.hf_create(p.grid, 0)
        if coef == "ids":
            hf.hf_set_material_ids(ctx, torch.tensor(p.extra["ids"], device=dev), [4.9e8, 4e6], [3.724e6, 1.65e6])
        else:
            hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
        F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
        hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
        u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
        hf.hf_simulate(ctx, p.theta, p.dt, 4, F, u)
        ka = hf.hf_time_kernel_a(ctx, 200)
        print(f"C3 {coef:5s}: {r['ms_per_step']:.4f} ms/step, {r['us_per_pcg_iter']:.2f} us/iter, "
              f"it/step {r['pcg_iters_per_step']:.1f}, kernel A {ka * 1e3:.2f} us", flush=True)
        del ctx
if "a512" in what:
    for ids in (True, False):
        r = bench.apply_512(hf, torch, dev, 6549.8, ids=ids)
        print(f"apply 512^3 {'ids' if ids else 'pairs'} R={os.environ.get('HF_TILE_R', 'default')}: "
              f"{r['ms']:.4f} ms, {r['achieved']:.0f} GB/s, frac {r['frac']:.3f}", flush=True)
