import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1905_07622_b200 as hf, synth
dev = torch.device("cuda:0")
p = synth.c3(nsteps=3)
for f in ("0", "1"):
    os.environ["HF_FUSE_AB"] = f
    ctx = hf.hf_create(p.grid, 0)
    hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
    l0 = hf.hf_get_launch_count(ctx)
    st = hf.hf_simulate(ctx, p.theta, p.dt, 3, F, u)
    print(f, "launches", hf.hf_get_launch_count(ctx) - l0, "iters", st["total_iters"], "ms", st["ms_total"])
