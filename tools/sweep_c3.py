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
for R, ch in [(2, 0), (2, 4), (2, 6), (2, 12), (2, 20), (2, 34), (4, 0), (4, 4), (4, 8), (4, 20)]:
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
    print(f"R={R} zchunk={ch}: apply {ap:6.1f} us   step {st['ms_total']/10:.3f} ms  {st['ms_total']/st['total_iters']*1e3:.1f} us/iter", flush=True)
    del ctx
