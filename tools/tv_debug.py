import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, oracle, paper_1905_07622_b200 as hf
dev = torch.device("cuda:0")
T = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
for g in [synth.Grid((1,1,1),(1.0,1.0,1.0)), synth.Grid((2,2,2),(1.0,1.0,1.0)), synth.Grid((8,8,8),(0.125,)*3)]:
    for mode in ["const", "xlin", "ylin", "zlin", "rand"]:
        x, y, z = [a.ravel() for a in g.node_coords()]
        kn = {"const": np.ones(g.n_nodes), "xlin": 1 + x, "ylin": 1 + y, "zlin": 1 + z, "rand": np.random.default_rng(0).uniform(1, 2, g.n_nodes)}[mode]
        cn = np.ones(g.n_nodes)
        o = oracle.Oracle(g, kn, cn, elem=1, vertex=True)
        ctx = hf.hf_create(g, 0); hf.hf_set_element(ctx, 1); hf.hf_set_vertex_coefficients(ctx, T(kn), T(cn))
        u = np.random.default_rng(1).standard_normal(g.n_nodes)
        y = torch.empty(g.n_nodes, dtype=torch.float64, device=dev)
        for aK, aM in [(1.0, 0.0), (0.0, 1.0)]:
            hf.hf_apply(ctx, aK, aM, T(u), y); yo = o.spmv(aK, aM, u)
            err = np.abs(y.cpu().numpy() - yo).max() / np.abs(yo).max()
            print(g.ne, mode, aK, aM, "err %.3e" % err)
        d = torch.empty_like(y); hf.hf_diag(ctx, 1.0, 0.0, d)
        print("   diag err %.3e" % (np.abs(d.cpu().numpy() - o.diag(1.0, 0.0)).max() / np.abs(o.diag(1.0,0.0)).max()))
