"""NEXT row f4: the paper's operator-interpretation comparison (§5.1, Fig. 5 / Table 1)
rerun on one B200 with the three implementations of libheatfem (hf_apply_impl):

  impl 1  flexible DbD, two passes, stored 8x8 element matrices
  impl 2  single-pass FG DbD, one thread per node gathering 27 inputs
  impl 3  the production TMA stencil (sum-factorised; the paper's Implementation 3 role)

Workloads: the §5.1 laminate grids C = (30s, 30s, 10s), s = 1..6 (10.5k .. 2.0M DoF) with the
paper's element (6 P1 tets, one (k, c) per voxel) and with Q1 voxels; C3 (1M DoF inclusion
field, Q1); the 512^3-node grid of C4 (Q1), where every input is far larger than the L2.
Timing: CUDA events around REPS back-to-back applies on the context stream after 3 warm-up
applies (caches warm, as inside a PCG loop).  achieved = algorithmic bytes (read u, write y:
16 B/node; read (k, c): 16 B/element -- the same for every implementation) / time; "design"
bytes = what the implementation moves by construction (impl 1 adds the stored matrices
512 B/element and the contribution round trip 64 B/element + 64 B/node).
Parity of each implementation with the oracle: tests/test_gpu_ablation.py.
Writes one JSON line per (grid, element, impl) to stdout and to gpurun_out/ablation.jsonl."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_07622_b200 as hf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    PEAK = 7672.0


def run(name, g, elem, impls=(1, 2, 3), reps=20):
    gen = torch.Generator(device=dev).manual_seed(0)
    k = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) * 121.5 + 1.0
    c = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) + 1.0
    ctx = hf.hf_create(g, 0)
    hf.hf_set_element(ctx, elem)
    hf.hf_set_coefficients(ctx, k, c)
    del k, c
    u = torch.randn(g.n_nodes, dtype=torch.float64, device=dev, generator=gen)
    y = torch.empty_like(u)
    aK, aM = 0.005, 1.0
    out = []
    s = torch.cuda.current_stream(dev)
    for impl in impls:
        if impl == 1:
            hf.hf_ablation_prepare(ctx, aK, aM)
        for _ in range(3):
            hf.hf_apply_impl(ctx, impl, aK, aM, 1.0, u, None, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            hf.hf_apply_impl(ctx, impl, aK, aM, 1.0, u, None, y)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        alg = 16.0 * g.n_nodes + 16.0 * g.n_elems
        design = alg + (512.0 * g.n_elems + 64.0 * g.n_elems + 64.0 * g.n_nodes if impl == 1 else 0.0)
        r = {"grid": name, "dofs": g.n_nodes, "elements": g.n_elems,
             "element": "6 P1 tets / voxel" if elem == 1 else "Q1 hex", "impl": impl, "ms": round(ms, 5),
             "algorithmic_GBps": round(alg / (ms * 1e-3) / 1e9, 1),
             "design_GBps": round(design / (ms * 1e-3) / 1e9, 1),
             "frac_of_peak_design": round(design / (ms * 1e-3) / 1e9 / PEAK, 3),
             "ns_per_dof": round(ms * 1e6 / g.n_nodes, 4)}
        out.append(r)
        print(json.dumps(r), flush=True)
    del ctx, u, y
    torch.cuda.empty_cache()
    return out


def main():
    rows = []
    for s in range(1, 7):
        g = synth.laminate(s).grid
        for elem in (1, 0):
            rows += run(f"laminate s={s}", g, elem)
    rows += run("C3 100^3", synth.c3(nsteps=1).grid, 0)
    if "--no-512" not in sys.argv:
        rows += run("C4 512^3", synth.c4_grid(512), 0, reps=5)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ablation.jsonl"), "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    # the paper's Table 1 analogue: slope of time vs DoF (largest two laminate sizes), impl 3 / impl k
    for elem in ("6 P1 tets / voxel", "Q1 hex"):
        sl = {}
        for impl in (1, 2, 3):
            pts = sorted((r["dofs"], r["ms"]) for r in rows
                         if r["element"] == elem and r["impl"] == impl and r["grid"].startswith("laminate"))
            (d0, t0), (d1, t1) = pts[-2], pts[-1]
            sl[impl] = (t1 - t0) / (d1 - d0)
        print(json.dumps({"table1_analogue": elem, "ms_per_MDoF_slope": {k: round(v * 1e6, 4) for k, v in sl.items()},
                          "impl3_speedup_over": {k: round(v / sl[3], 2) for k, v in sl.items()}}), flush=True)


if __name__ == "__main__":
    main()
