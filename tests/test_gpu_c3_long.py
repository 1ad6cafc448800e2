"""north_star target at full length: C3 (100^3 nodes = 1M DoF, random inclusions, CN, dt 0.01,
rtol 1e-12), 300 time steps on the GPU against the fp64 oracle (OpenMP on the host cores).

Checked: every entry of u^150 (mid-run checkpoint, through hf_simulate_resume) and of u^300,
and the front face z = 0 after every one of the 300 steps, each at rel-L2 <= 1e-10
(BASELINE.json north_star; P:55-56 time loop, Alg. 1 P:93-113 per step).
"""
import time

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_07622_b200 as hf  # noqa: E402

DEV = torch.device("cuda:0")
BAR = 1e-10


def T(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def c3_oracle_run():
    p = synth.c3(nsteps=300)
    t0 = time.time()
    o, F = oracle.problem_oracle(p)
    half = p.nsteps // 2
    u150, up150, st1, it1, snap1 = o.simulate_resume(p.theta, p.dt, half, F, p.u0, None, 0, tol=p.rtol,
                                                     snap_plane=0)
    u300, _, st2, it2, snap2 = o.simulate_resume(p.theta, p.dt, p.nsteps - half, F, u150, up150, half,
                                                 tol=p.rtol, snap_plane=0)
    assert st1 == 0 and st2 == 0
    print(f"\n[c3 oracle] 300 steps in {time.time() - t0:.0f} s on {oracle.num_threads()} threads, "
          f"{int(it1.sum() + it2.sum())} PCG iterations")
    return p, F, u150, u300, np.concatenate([snap1, snap2]), np.concatenate([it1, it2])


def test_c3_300_steps_full_trajectory(c3_oracle_run):
    p, F, u150o, u300o, snapo, ito = c3_oracle_run
    ctx = hf.hf_create(p.grid, 0)
    hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
    Fd = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, Fd)
    # one run of 300 steps with the front face after every step
    u = T(p.u0)
    snap = torch.empty(p.nsteps * ctx.n_plane, dtype=torch.float64, device=DEV)
    st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, Fd, u, 0, snap, rtol=p.rtol)
    assert st["steps_done"] == p.nsteps and st["first_failed_step"] == -1
    sn = snap.cpu().numpy().reshape(p.nsteps, -1)
    worst = max(rel(sn[n], snapo[n]) for n in range(p.nsteps))
    assert worst <= BAR, worst
    r300 = rel(u.cpu().numpy(), u300o)
    assert r300 <= BAR, r300
    # the same trajectory as a checkpoint at step 150 and a resumed second half
    half = p.nsteps // 2
    u1 = T(p.u0)
    up = torch.empty_like(u1)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, half, Fd, u1, up, 0, rtol=p.rtol)
    r150 = rel(u1.cpu().numpy(), u150o)
    assert r150 <= BAR, r150
    hf.hf_simulate_resume(ctx, p.theta, p.dt, p.nsteps - half, Fd, u1, up, half, rtol=p.rtol)
    r300b = rel(u1.cpu().numpy(), u300o)
    assert r300b <= BAR, r300b
    # iteration counts are not a parity quantity (R16), but they must be close
    assert abs(st["total_iters"] - int(ito.sum())) <= 0.02 * ito.sum()
    print(f"[c3 300 steps] worst front-face rel-L2 {worst:.2e}, u150 {r150:.2e}, u300 {r300:.2e} / {r300b:.2e}, "
          f"iterations {st['total_iters']} (oracle {int(ito.sum())})")


@pytest.mark.parametrize("variant", ["ids", "mixed"])
def test_c3_300_steps_variants(c3_oracle_run, variant):
    """The same 300-step trajectory through material ids (1 B per element, EL_Q1P stencil) and
    through mixed precision (fp32 correction + fp64 finish, hf_set_mixed): u^300 and the front
    face after every step within 1e-10 of the fp64 oracle."""
    p, F, u150o, u300o, snapo, ito = c3_oracle_run
    ctx = hf.hf_create(p.grid, 0)
    if variant == "mixed":
        hf.hf_set_mixed(ctx, 1, 1e-5)
        hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
    else:
        hf.hf_set_material_ids(ctx, torch.tensor(p.extra["ids"], device=DEV),
                               [m[1] for m in p.extra["materials"]], [m[0] for m in p.extra["materials"]])
    Fd = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, Fd)
    u = T(p.u0)
    snap = torch.empty(p.nsteps * ctx.n_plane, dtype=torch.float64, device=DEV)
    st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, Fd, u, 0, snap, rtol=p.rtol)
    assert st["steps_done"] == p.nsteps and st["first_failed_step"] == -1
    sn = snap.cpu().numpy().reshape(p.nsteps, -1)
    worst = max(rel(sn[n], snapo[n]) for n in range(p.nsteps))
    r300 = rel(u.cpu().numpy(), u300o)
    assert worst <= BAR and r300 <= BAR, (worst, r300)
    print(f"\n[c3 300 steps, {variant}] worst front-face rel-L2 {worst:.2e}, u300 {r300:.2e}")
