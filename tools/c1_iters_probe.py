"""Per-step PCG iteration counts of C1: the GPU (graph and host drivers) against the oracle."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth, paper_1905_07622_b200 as hf
dev = torch.device('cuda:0')
p = synth.c1()
o, Fo = oracle.problem_oracle(p)
uo, sto, it, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
print('oracle per step', list(it))
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
u = torch.tensor(p.u0, device=dev); up = torch.zeros_like(u)
gi = []
for n in range(p.nsteps):
    un = u.clone()
    st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 1, F, u, up, n, rtol=p.rtol)
    gi.append(st['total_iters'])
print('gpu per step   ', gi)
for drv in (1,):
    hf.hf_set_driver(ctx, drv)
    u2 = torch.tensor(p.u0, device=dev)
    st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u2, rtol=p.rtol)
    print('host driver total', st['total_iters'])
