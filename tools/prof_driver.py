"""Small workloads for ncu captures (ncu replays each kernel; keep them short)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
mode = sys.argv[1] if len(sys.argv) > 1 else "sim"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2

if mode == "sim":
    p = synth.c3(nsteps=steps)
    ctx = hf.hf_create(p.grid, 0)
    if os.environ.get("HF_PREC"):
        hf.hf_set_precision(ctx, int(os.environ["HF_PREC"]))
    if os.environ.get("CG_VARIANT"):    # single-reduction PCG (hf_set_cg_variant)
        hf.hf_set_cg_variant(ctx, int(os.environ["CG_VARIANT"]))
    if os.environ.get("HF_IDS"):        # materials by id (stencil variant EL_Q1P)
        hf.hf_set_material_ids(ctx, torch.tensor(p.extra["ids"], device=dev),
                               [m[1] for m in p.extra["materials"]], [m[0] for m in p.extra["materials"]])
    else:
        hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
    st = hf.hf_simulate(ctx, p.theta, p.dt, steps, F, u)
    print(st)
elif mode == "sim512":
    # C4 grid (512^3 nodes), two materials i.i.d. per element as bench.c4_steps, 1 CN step
    g = synth.c4_grid(512)
    gen = torch.Generator(device=dev).manual_seed(3)
    ox = torch.rand(g.n_elems, device=dev, generator=gen) < 0.2
    k = torch.where(ox, synth.OXIDE[1], synth.STEEL[1]).to(torch.float64)
    c = torch.where(ox, synth.OXIDE[0], synth.STEEL[0]).to(torch.float64)
    del ox
    ctx = hf.hf_create(g, 0)
    hf.hf_set_coefficients(ctx, k, c)
    del k, c
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = torch.zeros(g.n_nodes, dtype=torch.float64, device=dev)
    print(hf.hf_simulate(ctx, 0.5, 0.01, steps, F, u))
elif mode.startswith("apply"):
    n = int(mode[5:] or 512)
    g = synth.c4_grid(n)
    gen = torch.Generator(device=dev).manual_seed(0)
    k = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) + 0.5
    c = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) + 0.5
    u = torch.randn(g.n_nodes, dtype=torch.float64, device=dev, generator=gen)
    y = torch.empty_like(u)
    ctx = hf.hf_create(g, 0)
    if os.environ.get("HF_PREC"):
        hf.hf_set_precision(ctx, int(os.environ["HF_PREC"]))
    if os.environ.get("HF_IDS"):
        ids = (torch.rand(g.n_elems, device=dev, generator=gen) < 0.2).to(torch.uint8)
        hf.hf_set_material_ids(ctx, ids, [synth.STEEL[1], synth.OXIDE[1]], [synth.STEEL[0], synth.OXIDE[0]])
    else:
        hf.hf_set_coefficients(ctx, k, c)
    for _ in range(steps):
        hf.hf_apply(ctx, 0.005, 1.0, u, y)
    torch.cuda.synchronize()
