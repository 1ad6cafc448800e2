"""Kernel A (hf_time_kernel_a, 200 back-to-back launches) on an nx x ny x nz node grid with random
(k, c) fields: sensitivity of the C3 kernel to the tile quantisation (argv: nx ny nz ...)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
a = [int(v) for v in sys.argv[1:]] or [100, 100, 100]
for i in range(0, len(a), 3):
    nx, ny, nz = a[i:i + 3]
    g = synth.Grid((nx - 1, ny - 1, nz - 1), (0.2, 0.2, 0.2))
    k, c = synth.random_fields(g, seed=1)
    ctx = hf.hf_create(g, 0)
    hf.hf_set_coefficients(ctx, torch.tensor(k, device=dev), torch.tensor(c, device=dev))
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = torch.zeros(g.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_simulate(ctx, 0.5, 0.01, 2, F, u)
    t = min(hf.hf_time_kernel_a(ctx, 200) for _ in range(3))
    print(f"{nx}x{ny}x{nz}: kernel A {t * 1e3:.2f} us ({nx * ny * nz / 1e6:.2f}M nodes)", flush=True)
