"""Where the e2e time goes: the bench's e2e sequence (pinned host k, c, u0, per-step snapshots)
with CUDA-synchronised wall-clock stamps per call."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
K = 30
p = synth.c3(nsteps=K)
g = p.grid
plane = (g.ne[0] + 1) * (g.ne[1] + 1)
kh = torch.tensor(p.k).pin_memory()
ch = torch.tensor(p.c).pin_memory()
uh = torch.zeros(g.n_nodes, dtype=torch.float64).pin_memory()
snap = torch.empty(K * plane, dtype=torch.float64).pin_memory()
ctx = hf.hf_create(g, 0)
Fe = torch.empty(g.n_nodes, dtype=torch.float64, device=dev)
hf.hf_set_coefficients(ctx, kh, ch)
hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, Fe)
hf.hf_simulate(ctx, p.theta, p.dt, K, Fe, uh, 0, snap, rtol=p.rtol)
for rep in range(2):
    uh.zero_()
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    hf.hf_set_coefficients(ctx, kh, ch)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, Fe)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    st = hf.hf_simulate(ctx, p.theta, p.dt, K, Fe, uh, 0, snap, rtol=p.rtol)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"rep {rep}: set_coefficients {d[0]:.2f} ms, face_load {d[1]:.2f} ms, simulate {d[2]:.2f} ms "
          f"(device steps {st['ms_total']:.2f} ms), total {sum(d):.2f} ms = {sum(d) / K:.3f} ms/step", flush=True)
# the same simulate with device u and no snapshots
ud = torch.zeros(g.n_nodes, dtype=torch.float64, device=dev)
hf.hf_simulate(ctx, p.theta, p.dt, K, Fe, ud, rtol=p.rtol)
ud.zero_()
torch.cuda.synchronize()
t0 = time.perf_counter()
st = hf.hf_simulate(ctx, p.theta, p.dt, K, Fe, ud, rtol=p.rtol)
torch.cuda.synchronize()
print(f"device u, no snapshots: {1e3 * (time.perf_counter() - t0):.2f} ms (device {st['ms_total']:.2f})")
