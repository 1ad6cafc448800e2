"""C4 (512^3 nodes) time steps with Alg. 1's two-kernel PCG (variant 0) and the single-reduction
PCG (variant 1): ms per step / per iteration after one warm-up step, and the difference between
the two solutions."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = synth.c4_grid(n)
gen = torch.Generator(device=dev).manual_seed(3)
ox = torch.rand(g.n_elems, device=dev, generator=gen) < 0.2
k = torch.where(ox, synth.OXIDE[1], synth.STEEL[1]).to(torch.float64)
c = torch.where(ox, synth.OXIDE[0], synth.STEEL[0]).to(torch.float64)
del ox
res = {}
for v in (0, 1, 0, 1):
    ctx = hf.hf_create(g, 0)
    hf.hf_set_cg_variant(ctx, v)
    hf.hf_set_coefficients(ctx, k, c)
    F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = torch.zeros(ctx.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    hf.hf_simulate_resume(ctx, 0.5, 0.01, 1, F, u, up, 0, rtol=1e-12)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = hf.hf_simulate_resume(ctx, 0.5, 0.01, 2, F, u, up, 1, rtol=1e-12)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    it = max(st["total_iters"], 1)
    print(f"n={n} variant {v} (used {hf.hf_cg_variant(ctx)['last_used']}): {ms / 2:.2f} ms/step, "
          f"{ms / it * 1e3:.1f} us/iter, iters {it}", flush=True)
    res[v] = u.clone()
    del ctx, F, u, up
    torch.cuda.empty_cache()
print("variant 1 vs 0 rel diff", float((res[1] - res[0]).norm() / res[0].norm()))
