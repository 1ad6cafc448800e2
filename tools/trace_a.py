"""Where kernel A's time goes at C3: %globaltimer stamps per block (debug build -DHF_TRACE,
variants/lib_trace.so).  Points: 0 entry, 1 state header, 2 barrier init + TMA issue,
3 partial sums + iteration start, 4 first plane's TMA wait, 5 plane loop done, 6 partials stored."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HF_LIB_VARIANT", os.path.join(ROOT, "variants", "lib_trace.so"))
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
p = synth.c3(nsteps=4)
ctx = hf.hf_create(p.grid, 0)
hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
hf.hf_simulate(ctx, p.theta, p.dt, 4, F, u)
for reps in (1, 50):
    ms = hf.hf_time_kernel_a(ctx, reps)
    nb = 280
    buf = (C.c_ulonglong * (8 * 4096))()
    hf._lib.hf_trace_read(buf, 4096)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8)[:nb].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t[:, :7] - t0) / 1e3
    print(f"reps={reps}: mean launch {ms * 1e3:.2f} us; span of last launch (first entry -> last exit) "
          f"{(t[:, 6].max() - t0) / 1e3:.2f} us; SMs used {len(set(t[:, 7]))}")
    names = ["entry", "header", "tma issued", "iter start", "first plane", "loop done", "exit"]
    for k in range(7):
        print(f"  {names[k]:12s} min {rel[:, k].min():6.2f}  med {np.median(rel[:, k]):6.2f}  max {rel[:, k].max():6.2f} us")
    d = np.diff(rel, axis=1)
    for k in range(6):
        print(f"  {names[k]:>12s} -> {names[k + 1]:12s} med {np.median(d[:, k]):6.2f}  max {d[:, k].max():6.2f}")

# which CTAs are slow: loop time by SM co-residency and by grid position (4 x 7 x 10 at C3)
from collections import Counter
loop = (t[:, 5] - t[:, 4]) / 1e3
start = (t[:, 4] - t0) / 1e3
cnt = Counter(t[:, 7].tolist())
share = np.array([cnt[s] for s in t[:, 7]])
for k in sorted(set(share)):
    m = share == k
    print(f"CTAs on SMs holding {k}: {m.sum():4d}  loop med {np.median(loop[m]):.2f}  max {loop[m].max():.2f}  "
          f"first-plane med {np.median(start[m]):.2f}")
gx, gy = 4, 7
bx, by, bz = np.arange(nb) % gx, (np.arange(nb) // gx) % gy, np.arange(nb) // (gx * gy)
for name, v in (("x", bx), ("y", by), ("z", bz)):
    print(name, " ".join(f"{np.median(loop[v == i]):.2f}" for i in sorted(set(v))))
sl = np.argsort(-loop)[:8]
print("slowest:", [(int(bx[i]), int(by[i]), int(bz[i]), int(t[i, 7]), round(float(loop[i]), 2)) for i in sl])
