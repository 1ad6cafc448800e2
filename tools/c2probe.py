import sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_1905_07622_b200 as hf, synth
dev = torch.device("cuda:0")
p = synth.c2()
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
hf.hf_set_dirichlet_faces(ctx, p.dirichlet_bits, p.dirichlet_values)
F = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
for drv in (0, 1):
    hf.hf_set_driver(ctx, drv)
    u = torch.tensor(p.u0, device=dev)
    st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol, raise_on_noconv=False)
    print(sys.argv[1], "driver", drv, st)
