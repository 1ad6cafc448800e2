"""C5 batched sims: sims/s for batch sizes B with the modelled stack group (HF_BATCH_GROUP unset)
and with fixed groups (argv: B values)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402
from paper_1905_07622_b200 import inverse as inv  # noqa: E402

dev = torch.device("cuda:0")
g = synth.c5_grid(100)
steps = int(os.environ.get("STEPS", "60"))
for B in [int(a) for a in sys.argv[1:]] or [8]:
    depths = synth.c5_depths(B)
    k, c = [], []
    for j, d in enumerate(depths):
        kk, cc = inv.corrosion_fields(g, float(d), 15.0, 12.7)
        k.append(kk)
        c.append(cc)
    kb = torch.tensor(np.concatenate(k), device=dev)
    cb = torch.tensor(np.concatenate(c), device=dev)
    ctx = hf.hf_create(g, 0)
    hf.hf_set_coefficients(ctx, kb[: g.n_elems].contiguous(), cb[: g.n_elems].contiguous())
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, synth.FACE_ZM, 0.0, (inv.BEAM_POWER, 2.0, 0.0, 0.0), F)
    ub = torch.zeros(B * g.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_simulate_batched(ctx, B, kb, cb, 0.5, 10.0 / 300, 2, F, ub, rtol=1e-12)    # warm-up (graphs)
    ub.zero_()
    torch.cuda.synchronize()
    t0 = time.time()
    st = hf.hf_simulate_batched(ctx, B, kb, cb, 0.5, 10.0 / 300, steps, F, ub, rtol=1e-12)
    torch.cuda.synchronize()
    t = time.time() - t0
    it = sum(s["total_iters"] for s in st)
    print(f"B={B} group={os.environ.get('HF_BATCH_GROUP', 'model')}: {t:.2f} s for {steps} steps, "
          f"{B * steps / t:.1f} sim-steps/s, {it / B / steps:.0f} it/step, |u| {float(ub.norm()):.10e}", flush=True)
    del ctx
