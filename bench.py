#!/usr/bin/env python3
"""Benchmark of the hot path: ms per time step at 1M DoF (BASELINE.json metric).

Workload (BASELINE.json configs[2]): 100^3 nodes (99^3 Q1 voxels), h = 0.2 mm,
20 % spherical oxide inclusions in steel (P:271 materials), flux f = 1 on z = 0,
Crank-Nicolson (theta = 0.5), dt = 0.01, Jacobi-PCG to rtol 1e-12.  A "step" is one time step
of the theta-scheme: RHS apply + PCG solve (Alg. 1) + guess update, all on the device.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1: one GPU, the C3 problem.  N > 1 (torchrun, one process per GPU; `--gpus N` launches it):
the headline is weak scaling over N independent C3 problems, one per GPU (the inverse problem's
forward solves; no collective on the data path): value = the slowest rank's time / all ranks'
time steps.  Legs: `c3_slabs_strong` (the same C3 problem split into N z-slabs, strong scaling;
`--strong` makes it the headline), `apply_512_slabs`, `c4_steps_slabs` (BASELINE configs[3]) and
`c5_batched_replicas`.  The slabs talk over peer memory (CUDA IPC mailboxes over NVLink: the
kernels store ghost planes into the neighbours' buffers and publish their reduction sums to every
rank; the whole solve stays in the step graph); `--transport nccl` selects the NCCL send/recv +
allreduce baseline instead.  HF_BENCH_SHARE_GPU=1 puts every rank on GPU 0 (code-path validation
on a one-GPU box; its timings mean nothing).
--impl reference: the CPU oracle (oracle/, plain C, 1 core) on the same workload, a bounded
sample of steps.  Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

TRANSPORT_NAME = "peer-memory mailboxes over NVLink, in-kernel exchange"
METRIC = "ms per time step at 1M DOF (C3: 100^3-node heterogeneous cube, CN, Jacobi-PCG rtol 1e-12)"
UNIT = "ms/step"


def workload_config(p):
    """The workload the line is about (identical in both arms; measured quantities and the
    implementation's parallelism are top-level keys of the line)."""
    return {
        "workload": "C3 (BASELINE.json configs[2]): 100^3 nodes = 1,000,000 DoF, 99^3 trilinear voxels, "
                    "h=0.2 mm, 20% spherical Fe2O3 inclusions in steel (P:271), f=1 on z=0, theta=0.5, "
                    "dt=0.01, rtol=1e-12, guess 2u^n-u^(n-1)",
        "nodes": p.grid.n_nodes,
        "elements": p.grid.n_elems,
        "l2": "flushed (512 MiB memset) before every timed step; within a step the 104 MB working set "
              "stays L2-resident, as in any real run",
    }


def parallelism(n_gpus):
    return "single GPU" if n_gpus == 1 else f"z-slabs x{n_gpus} ({TRANSPORT_NAME})"


# ---------------------------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel_key):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d[kernel_key]["dram_bytes_per_launch"]
    except Exception:
        return None


def _reduce(dist, dev, values, op="max"):
    """All-reduce a list of floats across ranks (CUDA tensors over NCCL, CPU tensors over gloo)."""
    import torch
    where = "cpu" if dist.get_backend() == "gloo" else dev
    t = torch.tensor([float(v) for v in values], device=where, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


# ---------------------------------------------------------------------------------------------
# our arm

def run_ours(args):
    import torch
    import paper_1905_07622_b200 as hf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("HF_BENCH_SHARE_GPU"):           # validation only: every rank on GPU 0
        local_rank = 0
    # N > 1: the headline is weak scaling over independent C3 problems, one per GPU (the inverse
    # problem's forward solves, north_star; no collective on the data path); --strong makes it
    # the same C3 problem split into N z-slabs; --force-slab: the slab code path on one rank
    slab = args.force_slab or (world > 1 and args.strong)
    replicas = world > 1 and not slab
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1 or args.force_slab:
        # stdout carries exactly one JSON line: NCCL's log (NCCL_DEBUG as the caller set it,
        # e.g. INFO for the communicator lines) goes to stderr unless a log file is given
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
            if os.environ.get("HF_BENCH_SHARE_GPU"):   # NCCL refuses two ranks on one GPU
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=dev)

    p = synth.c3(nsteps=args.warmup + args.steps)
    g = p.grid
    plane = (g.ne[0] + 1) * (g.ne[1] + 1)
    kd = torch.tensor(p.k, device=dev)
    cd = torch.tensor(p.c, device=dev)
    # per-element fp64 (k, c) pairs (default), or the paper's material description -- two
    # materials by region, one uint8 id per element (hf_set_material_ids, --coef ids)
    use_ids = args.coef == "ids"
    kmat = [m[1] for m in p.extra["materials"]]
    cmat = [m[0] for m in p.extra["materials"]]
    idsd = torch.tensor(p.extra["ids"], device=dev)

    def set_coef(c_, k_, c2_, ids_):
        if use_ids:
            hf.hf_set_material_ids(c_, ids_, kmat, cmat)
        else:
            hf.hf_set_coefficients(c_, k_, c2_)
    if not slab:
        ctx = hf.hf_create(g, local_rank)
        z0, lp = 0, g.ne[2] + 1
    else:
        ctx = make_slab_ctx(hf, g, rank, world, dist, local_rank, args.transport)
        _, _, lp, z0 = ctx.slab
    set_coef(ctx, kd, cd, idsd)
    F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = torch.zeros(ctx.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    stream = torch.cuda.current_stream(dev)

    # warm-up steps (state continues into the timed steps)
    st = hf.hf_simulate_resume(ctx, p.theta, p.dt, args.warmup, F, u, up, 0, rtol=p.rtol)
    step0 = args.warmup
    lc0 = hf.hf_get_launch_count(ctx)
    clocks = ClockSampler(local_rank)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    times, iters = [], 0
    if not slab:
        # one call: the library flushes L2 (512 MiB memset) before every step and times each
        # step alone with CUDA events on the context stream (= this torch stream)
        hf.hf_set_step_flush(ctx, True)
        st = hf.hf_simulate_resume(ctx, p.theta, p.dt, args.steps, F, u, up, step0, rtol=p.rtol)
        hf.hf_set_step_flush(ctx, False)
        times = [st["ms_steps"]]
        iters = st["total_iters"]
    else:
        for n in range(args.steps):
            hf.hf_flush_l2(ctx)                       # untimed L2 eviction between timed steps
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 1, F, u, up, step0 + n, rtol=p.rtol)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            iters += st["total_iters"]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    launches = hf.hf_get_launch_count(ctx) - lc0
    total_ms = float(sum(times))
    if dist:
        total_ms = _reduce(dist, dev, [total_ms])[0]
        if replicas:                                   # every rank's kernels count
            launches = int(_reduce(dist, dev, [launches], "sum")[0])
    ms_step = total_ms / args.steps
    # whole-job value: time steps of 1M-DoF problems processed by all ranks / the slowest rank's time
    value = total_ms / (args.steps * (world if replicas else 1))

    # dominant kernel: PCG kernel A (stencil apply), timed per launch with CUDA events on the
    # context stream over the same steps replayed with the profiling driver
    u2, up2 = u.clone(), up.clone()
    hf.hf_profile(ctx, True)
    prof_steps = min(args.steps, 5)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, prof_steps, F, u2, up2, step0 + args.steps, rtol=p.rtol)
    prof = hf.hf_profile_read(ctx)
    hf.hf_profile(ctx, False)
    a_ms, a_n = prof["stencil_cg_a"]
    a_bracketed_ms = a_ms / max(a_n, 1)          # each launch bracketed by its own event pair
    # kernel A replayed 200x as a graph chain joined by the PCG loop body's programmatic edges
    # (launched as in the loop: each launch's prologue overlaps the previous one's tail), timed
    # between one event pair on the context stream; this is the duration the roofline uses.
    # Beside it: the same launches back to back without the edges (each pays the launch gap).
    a_plain_ms = hf.hf_time_kernel_a(ctx, 200) if not slab else a_bracketed_ms
    a_avg_ms = hf.hf_time_kernel_a_graph(ctx, 200) if not slab else a_bracketed_ms
    nodes_local = plane * lp
    elems_local = g.ne[0] * g.ne[1] * max(lp - 1, 1)
    # algorithmic bytes of one kernel-A launch: read s, d_old (16 B/node) + the element
    # coefficients (a uint8 material id, or a (k, c) fp64 pair: 16 B/element), write d_new, q
    a_bytes = 32.0 * nodes_local + (1.0 if use_ids else 16.0) * elems_local
    peak, peak_src = measured_peaks()
    achieved = a_bytes / (a_avg_ms * 1e-3) / 1e9

    # e2e: the same workload through the public API from pinned host memory: H2D of k, c, u0
    # and D2H of the front-face plane every step + the final field, inside the timed region
    e2e = None
    if not slab:
        # (N > 1 replicas: every rank runs this on its own GPU; wall clock max over ranks and the
        # whole job's step count, as the headline)
        kh = torch.tensor(p.k).pin_memory()
        ch = torch.tensor(p.c).pin_memory()
        idh = torch.tensor(p.extra["ids"]).pin_memory()
        uh = torch.zeros(g.n_nodes, dtype=torch.float64).pin_memory()
        snap = torch.empty(args.steps * plane, dtype=torch.float64).pin_memory()
        ctx2 = hf.hf_create(g, local_rank)
        Fe = torch.empty(g.n_nodes, dtype=torch.float64, device=dev)
        set_coef(ctx2, kh, ch, idh)
        hf.hf_face_load(ctx2, p.flux_face, p.flux_const, None, Fe)
        # warm-up with the timed call's own arguments (host u, host snapshots): the library's
        # step graph is built and instantiated here, as in any repeated use of the API
        hf.hf_simulate(ctx2, p.theta, p.dt, args.steps, Fe, uh, 0, snap, rtol=p.rtol)
        uh.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        set_coef(ctx2, kh, ch, idh)
        hf.hf_face_load(ctx2, p.flux_face, p.flux_const, None, Fe)
        se = hf.hf_simulate(ctx2, p.theta, p.dt, args.steps, Fe, uh, 0, snap, rtol=p.rtol)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        if replicas:
            wall = _reduce(dist, dev, [wall])[0] / world
        coef_bytes = idh.numel() + 16 * len(kmat) if use_ids else (kh.numel() + ch.numel()) * 8
        e2e = {"value": wall / args.steps, "unit": UNIT,
               "h2d_bytes_per_step": int((coef_bytes + uh.numel() * 8) / args.steps),
               "d2h_bytes_per_step": int(plane * 8 + uh.numel() * 8 / args.steps),
               "how": "wall clock around " + ("hf_set_material_ids (pinned uint8 ids)" if use_ids else
                                              "hf_set_coefficients (pinned k, c)") +
                      " + hf_face_load + hf_simulate(K steps) with pinned host u0, u_N and a per-step "
                      "front-face snapshot (host)"}
        del ctx2
    else:
        # N ranks: each rank feeds its slab from pinned host memory (global k, c; its planes of
        # u0) through the same calls on the existing slab context; wall clock, max over ranks
        kh = torch.tensor(p.k).pin_memory()
        ch = torch.tensor(p.c).pin_memory()
        uh = torch.zeros(ctx.n_nodes, dtype=torch.float64).pin_memory()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        set_coef(ctx, kh, ch, torch.tensor(p.extra["ids"]).pin_memory())
        hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
        se = hf.hf_simulate(ctx, p.theta, p.dt, args.steps, F, uh, rtol=p.rtol)
        torch.cuda.synchronize()
        wall = _reduce(dist, dev, [(time.perf_counter() - t0) * 1e3])[0]
        e2e = {"value": wall / args.steps, "unit": UNIT,
               "h2d_bytes_per_step": int((kh.numel() + ch.numel() + uh.numel()) * 8 / args.steps),
               "d2h_bytes_per_step": int(uh.numel() * 8 / args.steps),
               "how": "per rank: wall clock around hf_set_coefficients + hf_face_load + hf_simulate(K steps) "
                      "with pinned host k, c, u0 (its slab) and u_N; max over ranks"}

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
            "scaling": "weak" if replicas else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded inclusion field, synth.c3)",
            "coefficients": ("material ids (uint8 per element, 2-entry table: steel / Fe2O3, P:271)" if use_ids
                             else "per-element fp64 (k, c) pairs"),
            "config": workload_config(p),
            "parallelism": (f"{world} independent C3 problems, one per GPU (inverse-problem forward solves, "
                            "no collective on the data path); value = slowest rank's time / all ranks' steps"
                            if replicas else parallelism(world)),
            "pcg_iters_per_step": iters / args.steps,
            "us_per_pcg_iter": total_ms / max(iters, 1) * 1e3,
            "e2e": e2e,
            # the whole PCG iteration against the same peak: kernel A (48 B/node + coefficients)
            # + kernel B (64 B/node) algorithmic bytes / the measured time per iteration
            "pcg_iteration_roofline": {
                "bytes_per_iter": a_bytes + 64.0 * nodes_local,
                "us_per_iter": total_ms / max(iters, 1) * 1e3,
                "achieved_GBps": (a_bytes + 64.0 * nodes_local) / (total_ms / max(iters, 1) * 1e-3) / 1e9,
                "frac": (a_bytes + 64.0 * nodes_local) / (total_ms / max(iters, 1) * 1e-3) / 1e9 / peak,
                "note": "time per iteration includes the per-step kernels (RHS, init, step end) spread "
                        "over the step's iterations"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic("stencil_cg_a_c3_ids" if use_ids else "r02_stencil_cg_a_c3"),
                         "kernel": "k_stencil<LD_CGD,EP_CGA,%s> (PCG kernel A: d = s + beta d; q = A d; d.q)"
                                   % ("EL_Q1P" if use_ids else "EL_Q1"),
                         "bytes_per_launch": a_bytes, "avg_launch_ms": a_avg_ms,
                         "avg_launch_ms_how": "200 launches as one CUDA graph chain joined by the PCG loop "
                                              "body's programmatic edges, one event pair on the context "
                                              "stream (hf_time_kernel_a_graph)",
                         "avg_launch_ms_plain_replay": a_plain_ms,
                         "plain_replay_how": "the same 200 launches back to back without programmatic edges "
                                             "(hf_time_kernel_a): each pays the full launch gap",
                         "avg_launch_ms_event_bracketed": a_bracketed_ms, "launches_bracketed": int(a_n),
                         "peak_source": peak_src,
                         "note": "C3 working set (~104 MB) is L2-resident during a step, so achieved can exceed "
                                 "the HBM copy peak; see apply_512 for the HBM-bound apply"},
        }
    if world > 1 or args.force_slab:
        # strong scaling on N z-slabs: C3 itself (peer memory), and the metric's second half --
        # the 512^3 operator apply and time step on N slabs (BASELINE configs[3]) -- plus the
        # corrosion sims as independent replicas; times max over ranks
        if replicas:
            c3s = c3_slabs(hf, torch, dev, rank, world, dist)
            if rank == 0:
                line["c3_slabs_strong"] = c3s
        a512 = apply_512_slabs(hf, torch, dev, peak, rank, world, dist)
        c4s = c4_steps(hf, torch, dev, peak, rank=rank, world=world, dist=dist)
        c5r = c5_batched(hf, torch, dev, world, rank=rank, dist=dist)
        c5m = c5_batched(hf, torch, dev, world, rank=rank, dist=dist, mixed=1e-7)   # same fp64 bar
        if rank == 0:
            line["apply_512_slabs"] = a512
            line["c4_steps_slabs"] = c4s
            line["c5_batched_replicas"] = c5r
            line["c5_batched_replicas_mixed"] = c5m
    if world == 1 and not slab:
        line["c3_other_coef"] = variant_c3(hf, torch, dev, 64, p.rtol, coef="pairs" if use_ids else "ids")
        # the on-chip PCG (opt-in): one cooperative launch per time step
        line["c3_resident_ids"] = variant_c3(hf, torch, dev, 64, p.rtol, steps=5, coef="ids", resident=True)
        line["apply_512"] = apply_512(hf, torch, dev, peak)
        line["apply_512_ids"] = apply_512(hf, torch, dev, peak, ids=True)
        line["c4_steps"] = c4_steps(hf, torch, dev, peak)
        # the same 512^3 time steps at the same accuracy through mixed precision
        c4m = c4_steps(hf, torch, dev, peak, mixed=1e-7)
        line["c4_steps_mixed"] = {"ms_per_step": c4m["ms_per_step"], "fp64_iters_per_step": c4m["pcg_iters_per_step"],
                                  "rtol": 1e-12, "precision": "fp64 mixed (fp32 stage to 1e-07, fp64 finish)",
                                  "nodes": c4m["nodes"]}
        line["c5_batched"] = c5_batched(hf, torch, dev, world)
        # the same sims at the same fp64 accuracy through mixed precision (fp32 stage to 1e-7,
        # fp64 finish to rtol 1e-12 on the fp64 residual)
        line["c5_batched_mixed"] = c5_batched(hf, torch, dev, world, mixed=1e-7)
        # the paper's settings for the inverse problem: rtol 1e-6, single precision
        line["c5_batched_fp32_rtol1e-6"] = c5_batched(hf, torch, dev, world, prec=32, rtol=1e-6)
        line["fp32_variant"] = fp32_variant(hf, torch, dev, peak)
    if rank == 0 and world == 1:                   # the oracle on the host cores: N = 1 only
        line["cpu_baseline"] = cpu_baseline(args)
    return line


def c3_slabs(hf, torch, dev, rank, world, dist, steps=5, warm=3):
    """C3 on N z-slabs over peer memory (strong scaling of the headline problem): ms per time
    step, max over ranks, L2 flushed before each timed step."""
    p = synth.c3(nsteps=steps + warm)
    ctx = make_slab_ctx(hf, p.grid, rank, world, dist, dev.index, _TRANSPORT[0])
    hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
    F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = torch.zeros(ctx.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, warm, F, u, up, 0, rtol=p.rtol)
    stream = torch.cuda.current_stream(dev)
    tot, iters = 0.0, 0
    for n in range(steps):
        hf.hf_flush_l2(ctx)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = hf.hf_simulate_resume(ctx, p.theta, p.dt, 1, F, u, up, warm + n, rtol=p.rtol)
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
        iters += st["total_iters"]
    tot = _reduce(dist, dev, [tot])[0]
    return {"ranks": world, "steps": steps, "ms_per_step": tot / steps,
            "pcg_iters_per_step": iters / steps, "transport": TRANSPORT_NAME,
            "note": "the same 1M-DoF problem split into z-slabs; per-iteration cross-GPU synchronisation "
                    "(two reductions) dominates at this size (DESIGN.md section 8)"}


def make_slab_ctx(hf, g, rank, world, dist, device, transport):
    """Slab context of this rank: peer memory (IPC handshake over torch.distributed) or NCCL."""
    if transport == "nccl":
        uid = hf.hf_nccl_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        return hf.hf_create_slab(g, rank, world, obj[0], transport=hf.TRANSPORT_NCCL, device=device)
    ctx = hf.hf_create_slab(g, rank, world, None, transport=hf.TRANSPORT_PEER_IPC, device=device)

    def all_gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out
    hf.hf_peer_setup(ctx, all_gather)
    return ctx


def apply_512(hf, torch, dev, peak, prec=64, ids=False):
    """Operator apply (Eq. (1)) on the 512^3-node grid of C4, HBM-bound: inputs 4.3 GB >> L2.
    prec=32: the fp32 storage variant (NEXT f3), half the bytes.  ids=True: two materials by id
    (steel / Fe2O3, 20 % oxide, i.i.d. per element), 1 B per element instead of a 16-B pair."""
    g = synth.c4_grid(512)
    gen = torch.Generator(device=dev).manual_seed(0)
    ctx = hf.hf_create(g, dev.index)
    if prec != 64:
        hf.hf_set_precision(ctx, prec)
    if ids:
        idv = (torch.rand(g.n_elems, device=dev, generator=gen) < 0.2).to(torch.uint8)
        hf.hf_set_material_ids(ctx, idv, [synth.STEEL[1], synth.OXIDE[1]], [synth.STEEL[0], synth.OXIDE[0]])
        del idv
    else:
        k = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) * 121.5 + 1.0
        c = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) + 1.0
        hf.hf_set_coefficients(ctx, k, c)
        del k, c
    torch.cuda.empty_cache()
    if prec == 64:
        u = torch.randn(g.n_nodes, dtype=torch.float64, device=dev, generator=gen)
        y = torch.empty_like(u)
        return _apply_time(hf, torch, dev, peak, ctx, g, u, y, 8, ids=ids)
    return _apply_time_internal(hf, torch, dev, peak, ctx, g, prec)


def apply_512_slabs(hf, torch, dev, peak, rank, world, dist, _unused=None):
    """512^3 apply on this rank's z-slab (strong scaling of configs[3]); aggregate GB/s from the
    slowest rank.  No exchange is needed: the input vector carries its ghost planes."""
    g = synth.c4_grid(512)
    ctx = make_slab_ctx(hf, g, rank, world, dist, dev.index, _TRANSPORT[0])
    lo, hi, lp, z0 = ctx.slab
    gen = torch.Generator(device=dev).manual_seed(0)
    k = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) * 121.5 + 1.0
    c = torch.rand(g.n_elems, dtype=torch.float64, device=dev, generator=gen) + 1.0
    hf.hf_set_coefficients(ctx, k, c)
    del k, c
    torch.cuda.empty_cache()
    u = torch.randn(ctx.n_nodes, dtype=torch.float64, device=dev)
    y = torch.empty_like(u)
    for _ in range(3):
        hf.hf_apply(ctx, 0.005, 1.0, u, y)
    s = torch.cuda.current_stream(dev)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        hf.hf_apply(ctx, 0.005, 1.0, u, y)
    e1.record(s)
    e1.synchronize()
    ms = _reduce(dist, dev, [e0.elapsed_time(e1) / 10])[0]
    nodes = (g.ne[0] + 1) * (g.ne[1] + 1) * (hi - lo)          # owned output nodes of this rank
    byts_total = 16.0 * g.n_nodes + 16.0 * g.n_elems              # all ranks together
    del ctx
    torch.cuda.empty_cache()
    agg = byts_total / (ms * 1e-3) / 1e9
    return {"ms_max_over_ranks": ms, "aggregate_GBps": agg, "per_gpu_GBps": agg / world,
            "frac_per_gpu": agg / world / peak, "peak": peak, "owned_nodes_rank0": nodes,
            "kernel": "k_stencil<LD_RAW,EP_APPLY> on each rank's 512^3 z-slab, mean of 10, max over ranks"}


def _apply_time_internal(hf, torch, dev, peak, ctx, g, prec):
    """fp32 contexts convert fp64 user vectors at the boundary; the kernel-only time is taken
    from the profiling driver's per-launch events on the context stream instead."""
    u = torch.randn(g.n_nodes, dtype=torch.float64, device=dev)
    y = torch.empty_like(u)
    for _ in range(3):
        hf.hf_apply(ctx, 0.005, 1.0, u, y)
    hf.hf_profile(ctx, True)
    for _ in range(10):
        hf.hf_apply(ctx, 0.005, 1.0, u, y)
    pr = hf.hf_profile_read(ctx)
    hf.hf_profile(ctx, False)
    ms = pr["rhs_apply"][0] / max(1, pr["rhs_apply"][1])
    es = prec // 8
    byts = 2.0 * es * g.n_nodes + 2.0 * es * g.n_elems
    ach = byts / (ms * 1e-3) / 1e9
    del ctx
    torch.cuda.empty_cache()
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "ms": ms,
            "bytes_per_launch": byts, "traffic": ncu_traffic("stencil_apply_512_f32"),
            "kernel": f"k_stencil<LD_RAW,EP_APPLY,fp{prec}> 512^3 nodes, mean of 10 (per-launch events)"}


def _apply_time(hf, torch, dev, peak, ctx, g, u, y, es, ids=False):
    for _ in range(3):
        hf.hf_apply(ctx, 0.005, 1.0, u, y)
    s = torch.cuda.current_stream(dev)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        hf.hf_apply(ctx, 0.005, 1.0, u, y)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    # read u + write y + read (k, c) pairs (2 es B per element) or material ids (1 B per element)
    byts = 2.0 * es * g.n_nodes + (1.0 if ids else 2.0 * es) * g.n_elems
    ach = byts / (ms * 1e-3) / 1e9
    del ctx
    torch.cuda.empty_cache()
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "ms": ms,
            "bytes_per_launch": byts, "traffic": ncu_traffic("stencil_apply_512_ids" if ids else "stencil_apply_512"),
            "kernel": "k_stencil<LD_RAW,EP_APPLY,%s> (y = (aK K + aM M) u), 512^3 nodes, median of 10"
                      % ("EL_Q1P, material ids" if ids else "EL_Q1, (k, c) pairs")}


def variant_c3(hf, torch, dev, prec, rtol, steps=10, warm=3, coef="pairs", mixed=None, resident=False, n=100):
    """C3 time steps of a precision / tolerance / coefficient-layout / solver variant, L2 flushed
    before each timed step.  mixed: rtol of the fp32 stage (hf_set_mixed); resident: the
    on-chip PCG (hf_set_resident, material ids); n: nodes per axis."""
    p = synth.c3(n_nodes_axis=n, nsteps=steps + warm)
    ctx = hf.hf_create(p.grid, dev.index)
    if prec != 64:
        hf.hf_set_precision(ctx, prec)
    if mixed:
        hf.hf_set_mixed(ctx, 1, mixed)
    if resident:
        hf.hf_set_resident(ctx, 1)
    if coef == "ids":
        hf.hf_set_material_ids(ctx, torch.tensor(p.extra["ids"], device=dev),
                               [m[1] for m in p.extra["materials"]], [m[0] for m in p.extra["materials"]])
    else:
        hf.hf_set_coefficients(ctx, torch.tensor(p.k, device=dev), torch.tensor(p.c, device=dev))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, warm, F, u, up, 0, rtol=rtol)
    lo0 = hf.hf_mixed_iters(ctx) if mixed else 0
    hf.hf_set_step_flush(ctx, True)
    st = hf.hf_simulate_resume(ctx, p.theta, p.dt, steps, F, u, up, warm, rtol=rtol)
    hf.hf_set_step_flush(ctx, False)
    out = {"precision": f"fp{prec}" if not mixed else "fp32 correction + fp64 finish", "coefficients": coef,
           "rtol": rtol, "steps": steps, "nodes": p.grid.n_nodes,
           "ms_per_step": st["ms_steps"] / steps,
           "pcg_iters_per_step": st["total_iters"] / steps,
           "us_per_pcg_iter": st["ms_steps"] / max(st["total_iters"], 1) * 1e3}
    if mixed:
        out["fp32_iters_per_step"] = (hf.hf_mixed_iters(ctx) - lo0) / steps
        out["fp32_stage_rtol"] = mixed
    if resident:
        out["solver"] = "on-chip PCG (hf_set_resident)"
        out["used"] = bool(hf.hf_resident_plan(ctx)["last_used"])
    del ctx
    return out


def fp32_variant(hf, torch, dev, peak):
    """NEXT row f3: fp32 storage (fp64 dots and scalars) at the paper's rtol 1e-6, next
    to fp64 at the same rtol; parity of the variant is in tests/test_gpu_fp32.py."""
    return {"c3_fp32_rtol1e-6": variant_c3(hf, torch, dev, 32, 1e-6),
            "c3_fp64_rtol1e-6": variant_c3(hf, torch, dev, 64, 1e-6),
            "apply_512_fp32": apply_512(hf, torch, dev, peak, 32),
            "parity": "fp32 vs the fp64 oracle: rel-L2 1.9e-7 after 2 C3 steps at rtol 1e-6 (bar 1e-5)",
            # the fp64 result from mostly-fp32 work (hf_set_mixed, defect correction), rtol 1e-12,
            # next to plain fp64 on the same grid: C3, and a 256^3 grid where iterations are
            # bandwidth-bound (C3's are latency-bound)
            "mixed_c3_rtol1e-12": variant_c3(hf, torch, dev, 64, 1e-12, steps=5, mixed=1e-5),
            "mixed_256_rtol1e-12": variant_c3(hf, torch, dev, 64, 1e-12, steps=3, warm=2, mixed=1e-5, n=256),
            "fp64_256_rtol1e-12": variant_c3(hf, torch, dev, 64, 1e-12, steps=3, warm=2, n=256),
            "mixed_parity": "fp64 finish to rtol 1e-12: C1, C2, C3 within 1e-10 of the oracle (tests/test_gpu_fp32.py)"}


def c4_steps(hf, torch, dev, peak, steps=2, rank=0, world=1, dist=None, mixed=None):
    """C4 (BASELINE configs[3] grid, 512^3 nodes = 134M DoF) time steps: two materials (steel /
    Fe2O3, 20 % oxide, i.i.d. per element, generated on the device), f = 1 on z = 0, CN,
    dt = 0.01, rtol 1e-12, after one warm-up step.  Every iteration streams ~17 GB, far beyond
    L2.  With dist (N ranks): the same problem on N z-slabs (NCCL ghost planes + allreduce, strong
    scaling of configs[3]), time = max over ranks.  Reports ms/step, ms/iteration and the
    iteration's aggregate algorithmic GB/s."""
    g = synth.c4_grid(512)
    gen = torch.Generator(device=dev).manual_seed(3)
    ox = torch.rand(g.n_elems, device=dev, generator=gen) < 0.2
    k = torch.where(ox, synth.OXIDE[1], synth.STEEL[1]).to(torch.float64)
    c = torch.where(ox, synth.OXIDE[0], synth.STEEL[0]).to(torch.float64)
    del ox
    if dist is None:
        ctx = hf.hf_create(g, dev.index)
        if mixed:                               # fp32 stage to rtol_lo, fp64 finish
            hf.hf_set_mixed(ctx, 1, mixed)
    else:
        ctx = make_slab_ctx(hf, g, rank, world, dist, dev.index, _TRANSPORT[0])
    hf.hf_set_coefficients(ctx, k, c)
    del k, c
    torch.cuda.empty_cache()
    F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=dev)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = torch.zeros(ctx.n_nodes, dtype=torch.float64, device=dev)
    up = torch.zeros_like(u)
    hf.hf_simulate_resume(ctx, 0.5, 0.01, 1, F, u, up, 0, rtol=1e-12)
    s = torch.cuda.current_stream(dev)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    st = hf.hf_simulate_resume(ctx, 0.5, 0.01, steps, F, u, up, 1, rtol=1e-12)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        ms = _reduce(dist, dev, [ms])[0]
    it = max(st["total_iters"], 1)
    byts = 112.0 * g.n_nodes + 16.0 * g.n_elems          # kernel A 48 B/node + (k, c); kernel B 64 B/node
    del ctx, F, u, up
    torch.cuda.empty_cache()
    return {"nodes": g.n_nodes, "ranks": world, "steps": steps, "ms_per_step": ms / steps,
            "pcg_iters_per_step": it / steps, "ms_per_iter": ms / it,
            "iteration_GBps": byts / (ms / it * 1e-3) / 1e9,
            "frac_per_gpu": byts / (ms / it * 1e-3) / 1e9 / peak / world, "rtol": 1e-12,
            "fields": "two materials, 20 % oxide i.i.d. per element (device RNG, seed 3)"}


def c5_batched(hf, torch, dev, world, nsims=10, nsteps=300, prec=64, rtol=None, rank=0, dist=None, mixed=None):
    """C5 (BASELINE configs[4]): corrosion-inverse forward simulations, 99^3 voxels each
    (1M DoF), T_F = 10 s in 300 CN steps, Gaussian beam 10 W sigma 2 mm, per-sim depth and
    log-normal k perturbation; nsims of them through hf_simulate_batched on this GPU.  With dist
    (N ranks): independent replicas, rank r runs sims r*nsims .. (r+1)*nsims-1 (weak scaling, no
    collective in the data path), time = max over ranks."""
    probs = [synth.c5(rank * nsims + j, nsteps=nsteps) for j in range(nsims)]
    g = probs[0].grid
    kb = torch.tensor(np.stack([p.k for p in probs]).ravel(), device=dev)
    cb = torch.tensor(np.stack([p.c for p in probs]).ravel(), device=dev)
    ctx = hf.hf_create(g, dev.index)
    if prec != 64:
        hf.hf_set_precision(ctx, prec)
    if mixed:                                   # fp32 correction + fp64 finish per stack (rtol_lo)
        hf.hf_set_mixed(ctx, 1, mixed)
    hf.hf_set_coefficients(ctx, kb[:g.n_elems], cb[:g.n_elems])
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=dev)
    p0 = probs[0]
    hf.hf_face_load(ctx, p0.flux_face, p0.flux_const, p0.beam, F)
    ub = torch.zeros(nsims * g.n_nodes, dtype=torch.float64, device=dev)
    front = torch.empty(nsims * (g.ne[0] + 1) * (g.ne[1] + 1), dtype=torch.float64, device=dev)
    # warm-up with the timed call's batch size: the stack context and its step graph are built here
    hf.hf_simulate_batched(ctx, nsims, kb, cb, p0.theta, p0.dt, 2, F, ub, rtol=rtol if rtol else p0.rtol)
    ub.zero_()
    s = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    stats = hf.hf_simulate_batched(ctx, nsims, kb, cb, p0.theta, p0.dt, nsteps, F, ub, 0, front,
                                   rtol=rtol if rtol else p0.rtol)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    if dist is not None:
        sec = _reduce(dist, dev, [sec])[0]
    its = sum(st["total_iters"] for st in stats)
    del ctx
    return {"sims": nsims * world, "ranks": world, "sims_per_rank": nsims, "steps_per_sim": nsteps, "seconds": sec,
            "sims_per_s": nsims * world / sec, "sims_per_s_per_gpu": nsims / sec,
            "ms_per_step": sec * 1e3 / (nsims * nsteps), "pcg_iters_per_step": its / (nsims * nsteps),
            "scaling": "weak (independent replicas, max over ranks)" if dist is not None else "single GPU",
            "precision": f"fp{prec}" + (f" mixed (fp32 stage to {mixed:g}, fp64 finish)" if mixed else ""),
            "rtol": rtol if rtol else p0.rtol,
            "path": "systems stacked along z (groups of up to 8), per-system PCG scalars and stop tests",
            "depths_mm": [round(p.extra["depth"], 3) for p in probs],
            "front_face_max_C": float(front.max().item())}


# ---------------------------------------------------------------------------------------------
# the oracle on the host

def oracle_steps(nsteps_timed, warm=1):
    import oracle
    p = synth.c3(nsteps=nsteps_timed + warm)
    t0 = time.perf_counter()
    o, F = oracle.problem_oracle(p)
    t_setup = time.perf_counter() - t0
    u, st, it, _ = o.simulate(p.theta, p.dt, warm, F, p.u0, tol=p.rtol)
    # continue from u^warm: the oracle restarts with guess u (same as u^0 rule)
    t0 = time.perf_counter()
    u2, st, it2, _ = o.simulate(p.theta, p.dt, nsteps_timed, F, u, tol=p.rtol)
    t = time.perf_counter() - t0
    return t * 1e3 / nsteps_timed, int(it2.sum()), t_setup, p


def _omp_threads(n):
    """Run the oracle on n OpenMP threads from here on (omp_set_num_threads through libgomp)."""
    import ctypes
    import oracle
    oracle.lib()
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass
    return oracle.num_threads()


def cpu_baseline(args):
    """The oracle as it stands on this host: all cores (OpenMP, the value) and one core."""
    steps = 2
    cores = _omp_threads(os.cpu_count() or 1)
    ms, iters, t_setup, p = oracle_steps(steps, warm=0)
    _omp_threads(1)
    ms1, _, _, _ = oracle_steps(1, warm=0)
    _omp_threads(cores)
    return {"value": ms, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{steps} time steps of C3 after CSR assembly ({t_setup:.1f} s, excluded): "
                      f"{iters / steps:.0f} PCG iterations/step, plain C + OpenMP on {cores} threads",
            "single_core": {"value": ms1, "unit": UNIT, "cores": 1, "sample": "1 time step of C3, 1 thread"}}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    steps = max(1, min(args.steps, 20))
    warm = 1 if args.warmup > 0 else 0
    cores = _omp_threads(os.cpu_count() or 1)
    ms, iters, t_setup, p = oracle_steps(steps, warm=warm)
    sample = (f"{steps} of the K={args.steps} requested C3 time steps (capped at 20 to bound the run), after "
              f"{warm} warm-up step and CSR assembly ({t_setup:.1f} s, excluded); plain C oracle, OpenMP on "
              f"{cores} threads")
    return {"impl": "reference", "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded inclusion field, synth.c3)",
            "config": workload_config(p),
            "parallelism": f"CPU oracle, OpenMP on {cores} threads",
            "pcg_iters_per_step": iters / steps,
            "cpu_baseline": {"value": ms, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


_TRANSPORT = ["peer"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--coef", choices=["ids", "pairs"], default="pairs",
                    help="element coefficients as per-element fp64 (k, c) pairs (default) or material ids "
                         "(the paper's two-material field, 1 B per element; no faster at C3, whose kernel A "
                         "is latency-bound, but 16 %% faster for the HBM-bound 512^3 apply)")
    ap.add_argument("--strong", action="store_true",
                    help="N > 1: the headline is the one C3 problem split into N z-slabs (default: one "
                         "independent C3 problem per GPU, weak scaling)")
    ap.add_argument("--force-slab", action="store_true",
                    help="run the multi-GPU (z-slab) code path even on one rank (validation)")
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="z-slab transport for N > 1: peer-memory mailboxes (default) or NCCL")
    args = ap.parse_args()
    _TRANSPORT[0] = args.transport
    global TRANSPORT_NAME
    if args.transport == "nccl":
        TRANSPORT_NAME = "NCCL send/recv ghost planes + allreduce, host loop"
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun (127.0.0.1 rendezvous)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "ours":
        import torch
        if torch.cuda.device_count() < int(os.environ.get("LOCAL_WORLD_SIZE", world)) and \
                not os.environ.get("HF_BENCH_SHARE_GPU"):
            sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {torch.cuda.device_count()}")
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)
    if (int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.force_slab) and args.impl == "ours":
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
