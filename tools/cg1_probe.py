"""Single-reduction PCG (hf_set_cg_variant 1) against Alg. 1's two-kernel PCG (variant 0):
C1 / C2 vs the oracle, C3 timing (10 steps after a 3-step warm-up, L2 flushed per step) and the
difference between the two variants' solutions."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def run(p, variant, nsteps=None, flush=False):
    ctx = hf.hf_create(p.grid, 0)
    hf.hf_set_cg_variant(ctx, variant)
    hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    u = torch.tensor(p.u0, device=dev)
    n = nsteps or p.nsteps
    if flush:
        up = torch.zeros_like(u)
        hf.hf_simulate_resume(ctx, p.theta, p.dt, 3, F, u, up, 0, rtol=p.rtol)
        hf.hf_set_step_flush(ctx, 1)
        st = hf.hf_simulate_resume(ctx, p.theta, p.dt, n, F, u, up, 3, rtol=p.rtol)
        hf.hf_set_step_flush(ctx, 0)
    else:
        st = hf.hf_simulate(ctx, p.theta, p.dt, n, F, u, rtol=p.rtol)
    torch.cuda.synchronize()
    used = hf.hf_cg_variant(ctx)["last_used"]
    return u.cpu().numpy(), st, used


for name, p in (("c1", synth.c1()), ("c2", synth.c2())):
    o, Fo = oracle.problem_oracle(p)
    uo, sto, it, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
    for v in (0, 1):
        ug, st, used = run(p, v)
        rel = np.linalg.norm(ug - uo) / np.linalg.norm(uo)
        print(f"{name} variant {v} (used {used}): rel-L2 {rel:.2e}, iters {st['total_iters']} (oracle {int(it.sum())})",
              flush=True)

p = synth.c3(nsteps=13)
res = {}
for v in (0, 1, 0, 1):
    t0 = time.time()
    ug, st, used = run(p, v, nsteps=10, flush=True)
    res[v] = ug
    print(f"c3 variant {v} (used {used}): {st['ms_steps'] / 10:.4f} ms/step, "
          f"{1e3 * st['ms_steps'] / max(st['total_iters'], 1):.2f} us/iter, iters {st['total_iters']} "
          f"(wall {time.time() - t0:.1f} s)", flush=True)
print("c3 variant 1 vs 0 rel diff", np.linalg.norm(res[1] - res[0]) / np.linalg.norm(res[0]))
