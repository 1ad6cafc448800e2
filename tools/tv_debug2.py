import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, oracle, paper_1905_07622_b200 as hf
dev = torch.device("cuda:0")
T = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
np.set_printoptions(precision=4, suppress=True, linewidth=150)
g = synth.Grid((1, 1, 1), (1.0, 1.0, 1.0))
ctx = hf.hf_create(g, 0); hf.hf_set_element(ctx, 1); hf.hf_set_vertex_coefficients(ctx, T(np.ones(8)), T(np.ones(8)))
ctx2 = hf.hf_create(g, 0); hf.hf_set_element(ctx2, 1); hf.hf_set_coefficients(ctx2, T([1.0]), T([1.0]))
for aK, aM in [(1.0, 0.0), (0.0, 1.0)]:
    A1 = np.zeros((8, 8)); A2 = np.zeros((8, 8))
    for j in range(8):
        e = np.zeros(8); e[j] = 1
        y = torch.empty(8, dtype=torch.float64, device=dev)
        hf.hf_apply(ctx, aK, aM, T(e), y); A1[:, j] = y.cpu().numpy()
        hf.hf_apply(ctx2, aK, aM, T(e), y); A2[:, j] = y.cpu().numpy()
    print("aK", aK, "aM", aM); print(A1); print(A2)
