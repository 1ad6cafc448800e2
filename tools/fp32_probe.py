import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, oracle, paper_1905_07622_b200 as hf
DEV = torch.device("cuda:0")
T = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for name, p in [("c1", synth.c1()), ("c3", synth.c3(nsteps=2))]:
    o, F = oracle.problem_oracle(p)
    uo, _, _, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0, tol=1e-12)
    for prec in (64, 32):
        for rtol in (1e-6, 1e-7, 1e-8, 1e-9):
            ctx = hf.hf_create(p.grid, 0); hf.hf_set_precision(ctx, prec); hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
            Fd = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV); hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, Fd)
            u = T(p.u0)
            st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, Fd, u, rtol=rtol, raise_on_noconv=False)
            torch.cuda.synchronize()
            print(name, prec, rtol, "rc", st["rc"], "iters", st["total_iters"], "rel", rel(u.cpu().numpy(), uo), flush=True)
