"""Quick device timings used while tuning (not the bench contract; see bench.py)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def ev_time(fn, reps):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def apply_probe(n_axis, tiles, reps=20, chunks=(0,)):
    g = synth.c4_grid(n_axis)
    gen = torch.Generator(device=dev).manual_seed(0)
    k = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) + 0.5
    c = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) + 0.5
    u = torch.randn(g.n_nodes, dtype=torch.float64, device=dev, generator=gen)
    y = torch.empty_like(u)
    for R in tiles:
        for ch in chunks:
            os.environ["HF_TILE_R"] = str(R)
            os.environ["HF_ZCHUNK"] = str(ch)
            ctx = hf.hf_create(g, 0)
            hf.hf_set_coefficients(ctx, k, c)
            for _ in range(3):
                hf.hf_apply(ctx, 0.005, 1.0, u, y)
            ms = ev_time(lambda: hf.hf_apply(ctx, 0.005, 1.0, u, y), reps)
            gbs = 32.0 * g.n_nodes / (ms * 1e-3) / 1e9
            print(f"apply {n_axis}^3 R={R} zchunk={ch}: {ms:.4f} ms  {gbs:.0f} GB/s (algorithmic 32 B/node)", flush=True)
            del ctx
    os.environ.pop("HF_TILE_R", None)
    os.environ.pop("HF_ZCHUNK", None)


def sim_probe(nsteps=20, tiles=(2, 4), drivers=(0, 1), chunks=(0,)):
    p = synth.c3(nsteps=nsteps)
    k = torch.tensor(p.k, device=dev)
    c = torch.tensor(p.c, device=dev)
    for R in tiles:
        for ch in chunks:
            for drv in drivers:
                os.environ["HF_TILE_R"] = str(R)
                os.environ["HF_ZCHUNK"] = str(ch)
                ctx = hf.hf_create(p.grid, 0)
                hf.hf_set_driver(ctx, drv)
                hf.hf_set_coefficients(ctx, k, c)
                F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
                hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
                u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
                hf.hf_simulate(ctx, p.theta, p.dt, 3, F, u)
                u.zero_()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                st = hf.hf_simulate(ctx, p.theta, p.dt, nsteps, F, u)
                wall = (time.perf_counter() - t0) * 1e3
                its = st["total_iters"] / nsteps
                print(f"c3 sim R={R} zchunk={ch} driver={drv}: {st['ms_total'] / nsteps:.3f} ms/step "
                      f"(wall {wall / nsteps:.3f}), {its:.1f} it/step, "
                      f"{st['ms_total'] / st['total_iters'] * 1e3:.1f} us/iter", flush=True)
                if drv == 1:
                    hf.hf_profile(ctx, True)
                    u.zero_()
                    hf.hf_simulate(ctx, p.theta, p.dt, 5, F, u)
                    prof = hf.hf_profile_read(ctx)
                    print("   profile (us/launch, n):",
                          {k: (round(v[0] / max(v[1], 1) * 1e3, 2), v[1]) for k, v in prof.items()}, flush=True)
                del ctx
    os.environ.pop("HF_TILE_R", None)
    os.environ.pop("HF_ZCHUNK", None)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "apply"):
        apply_probe(512, (2, 4))
        apply_probe(100, (2, 4), reps=200, chunks=(0, 8, 16))
    if what in ("all", "sim"):
        sim_probe(chunks=(0, 10))
