"""Sweep tile height / z-chunk for the C3 apply and CG step (tuning aid)."""
import os, sys, itertools
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa
import synth  # noqa
dev = torch.device("cuda:0")
p = synth.c3(nsteps=10)
k = torch.tensor(p.k, device=dev); c = torch.tensor(p.c, device=dev)
u = torch.randn(p.grid.n_nodes, dtype=torch.float64, device=dev); y = torch.empty_like(u)
combos = [(2, 0), (2, 8), (2, 10), (2, 12), (2, 14), (2, 17), (2, 20), (2, 25), (2, 34), (4, 0), (4, 12), (4, 20)]
if len(sys.argv) > 1:
    combos = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for R, ch in combos:
    os.environ["HF_TILE_R"] = str(R); os.environ["HF_ZCHUNK"] = str(ch)
    ctx = hf.hf_create(p.grid, 0)
    hf.hf_set_coefficients(ctx, k, c)
    F = torch.empty_like(u); hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    for _ in range(5): hf.hf_apply(ctx, 0.005, 1.0, u, y)
    s = torch.cuda.current_stream(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(100): hf.hf_apply(ctx, 0.005, 1.0, u, y)
    e1.record(s); e1.synchronize()
    ap = e0.elapsed_time(e1) / 100 * 1e3
    uu = torch.zeros_like(u)
    hf.hf_simulate(ctx, p.theta, p.dt, 3, F, uu)
    uu.zero_()
    st = hf.hf_simulate(ctx, p.theta, p.dt, 10, F, uu)
    hf.hf_profile(ctx, True)
    uu.zero_()
    hf.hf_simulate(ctx, p.theta, p.dt, 3, F, uu)
    pr = hf.hf_profile_read(ctx)
    hf.hf_profile(ctx, False)
    a_us = pr["stencil_cg_a"][0] / max(1, pr["stencil_cg_a"][1]) * 1e3
    b_us = pr["pointwise_cg_b"][0] / max(1, pr["pointwise_cg_b"][1]) * 1e3
    print(f"R={R} zchunk={ch}: A {a_us:5.1f} us  B {b_us:5.1f} us | apply {ap:6.1f} us   step {st['ms_total']/10:.3f} ms  {st['ms_total']/st['total_iters']*1e3:.1f} us/iter", flush=True)
    del ctx
