"""On-chip PCG (hf_resident.cuh): each time step's whole Alg. 1 solve in one
cooperative launch with every PCG vector held in shared memory / registers.  Checked against the
fp64 oracle (rel-L2 <= 1e-10, north_star) and against the streaming kernels (same readings
R3-R6, so the two paths agree to rounding order), on grids that span several bricks in every
axis and ragged brick sizes, with Dirichlet faces, residual replacement, NOCONV and b = 0."""
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


def to_ids(k, c):
    """(k, c) pairs -> uint8 ids + material table (test side: np.unique of the pairs)."""
    kc, inv = np.unique(np.stack([k, c], 1), axis=0, return_inverse=True)
    assert len(kc) < 64
    return inv.astype(np.uint8).ravel(), kc[:, 0].copy(), kc[:, 1].copy()


def run(p, resident=1, nsteps=None, rtol=None, max_iter=10000, replace_every=-1, snap_plane=-1):
    ctx = hf.hf_create(p.grid, 0)
    ids, km, cm = to_ids(p.k, p.c)
    hf.hf_set_material_ids(ctx, ids, km, cm)
    hf.hf_set_resident(ctx, resident)
    if p.dirichlet_bits:
        hf.hf_set_dirichlet_faces(ctx, p.dirichlet_bits, p.dirichlet_values)
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    u = T(p.u0)
    n = p.nsteps if nsteps is None else nsteps
    snap = torch.empty(n * ctx.n_plane, dtype=torch.float64, device=DEV) if snap_plane >= 0 else None
    st = hf.hf_simulate(ctx, p.theta, p.dt, n, F, u, snap_plane, snap, rtol=p.rtol if rtol is None else rtol,
                        max_iter=max_iter, replace_every=replace_every, raise_on_noconv=False)
    torch.cuda.synchronize()
    plan = hf.hf_resident_plan(ctx)
    return u.cpu().numpy(), st, plan, (None if snap is None else snap.cpu().numpy()), ctx


def oracle_run(p, nsteps=None):
    o, F = oracle.problem_oracle(p)
    n = p.nsteps if nsteps is None else nsteps
    uo, st, it, _ = o.simulate(p.theta, p.dt, n, F, p.u0, tol=p.rtol)
    assert st == 0
    return uo, it


def test_plan_c3_and_c4():
    c3 = hf.hf_create(synth.c3(nsteps=1).grid, 0)
    g = synth.c3(nsteps=1).grid
    hf.hf_set_material_ids(c3, np.zeros(g.n_elems, np.uint8), [1.0], [1.0])
    assert hf.hf_resident_plan(c3)["eligible"] == 0          # opt-in (hf_set_resident)
    hf.hf_set_resident(c3, 1)
    pl = hf.hf_resident_plan(c3)
    assert pl["eligible"] == 1, pl.get("why")
    assert pl["px"] * pl["py"] * pl["pz"] <= 148
    assert pl["bx"] <= 31 and pl["by"] <= 25 and pl["bz"] <= pl["BZ"]
    # pairs (not ids), and 512^3, are not eligible
    c3p = hf.hf_create(g, 0)
    hf.hf_set_resident(c3p, 1)
    hf.hf_set_coefficients(c3p, T(np.ones(g.n_elems)), T(np.ones(g.n_elems)))
    assert hf.hf_resident_plan(c3p)["eligible"] == 0
    g4 = synth.c4_grid(512)
    c4 = hf.hf_create(g4, 0)
    hf.hf_set_resident(c4, 1)
    hf.hf_set_material_ids(c4, torch.zeros(g4.n_elems, dtype=torch.uint8, device=DEV), [1.0], [1.0])
    assert hf.hf_resident_plan(c4)["eligible"] == 0


def test_c1_matches_oracle_and_streaming():
    p = synth.c1()
    u, st, plan, _, _ = run(p)
    assert plan["last_used"] == 1, plan
    uo, it = oracle_run(p)
    assert st["steps_done"] == p.nsteps and st["first_failed_step"] == -1
    assert rel(u, uo) <= BAR, rel(u, uo)
    us, sts, plans, _, _ = run(p, resident=0)
    assert plans["last_used"] == 0
    assert rel(u, us) <= 1e-12
    assert abs(st["total_iters"] - sts["total_iters"]) <= 2 + 0.02 * sts["total_iters"]


GRIDS = {
    # several bricks per axis with ragged sizes; thin and flat grids; one-node-thick bricks
    "ragged": synth.Grid((70, 40, 13), (0.3, 0.2, 0.7), (-1.0, 2.0, 0.5)),
    "seams": synth.Grid((33, 65, 9), (0.2, 0.2, 0.2)),
    "flat": synth.Grid((40, 30, 1), (0.1, 0.1, 0.1)),
    "tall": synth.Grid((3, 4, 90), (0.2, 0.2, 0.1)),
}


@pytest.mark.parametrize("gname", list(GRIDS))
def test_grids_match_oracle(gname):
    g = GRIDS[gname]
    rng = np.random.default_rng(11)
    ids = (rng.random(g.n_elems) < 0.3).astype(np.int64)
    kmat, cmat = np.array([4.9e8, 4e6]) * 1e-8, np.array([3.724e6, 1.65e6]) * 1e-6
    p = synth.Problem(gname, g, kmat[ids], cmat[ids], np.zeros(g.n_nodes), theta=0.5, dt=0.01, nsteps=4,
                      rtol=1e-12, flux_face=synth.FACE_ZM, flux_const=1.0)
    u, st, plan, _, _ = run(p)
    assert plan["last_used"] == 1, plan
    uo, _ = oracle_run(p)
    assert rel(u, uo) <= BAR, (gname, rel(u, uo), plan)


def test_c2_dirichlet_closed_form():
    p = synth.c2()
    u, st, plan, _, _ = run(p)
    assert plan["last_used"] == 1
    uo, _ = oracle_run(p)
    assert rel(u, uo) <= BAR
    # the bar's exact discrete solution (sin mode, SURVEY 8(c) pin)
    h = 1.0 / 64
    lam = (6.0 / h ** 2) * (1 - np.cos(np.pi * h)) / (2 + np.cos(np.pi * h))
    G = (1 - 0.5 * p.dt * lam) / (1 + 0.5 * p.dt * lam)
    assert rel(u, p.u0 * G ** p.nsteps) <= BAR


def test_nonzero_dirichlet_and_beam():
    g = synth.Grid((20, 18, 16), (0.5, 0.5, 0.4), (-5.0, -4.5, 0.0))
    rng = np.random.default_rng(5)
    ids = (rng.random(g.n_elems) < 0.25).astype(np.int64)
    kmat, cmat = np.array([4.9, 0.04]), np.array([3.7, 1.65])
    p = synth.Problem("dirbeam", g, kmat[ids], cmat[ids], np.zeros(g.n_nodes), theta=0.5, dt=0.05, nsteps=5,
                      rtol=1e-12, flux_face=synth.FACE_ZM, flux_const=0.0,
                      beam=(10.0, 2.0, 0.0, 0.0), dirichlet_bits=(1 << synth.FACE_XP) | (1 << synth.FACE_YM),
                      dirichlet_values=(0.0, 3.0, -1.5, 0.0, 0.0, 0.0))
    u, st, plan, _, _ = run(p)
    assert plan["last_used"] == 1
    uo, _ = oracle_run(p)
    assert rel(u, uo) <= BAR, rel(u, uo)


@pytest.mark.parametrize("every", [3, 7])
def test_residual_replacement(every):
    p = synth.c3(n_nodes_axis=40, nsteps=3)
    u, st, plan, _, _ = run(p, replace_every=every)
    assert plan["last_used"] == 1
    uo, _ = oracle_run(p)
    assert rel(u, uo) <= BAR, rel(u, uo)


def test_noconv_and_zero_rhs():
    p = synth.c1()
    u, st, plan, _, _ = run(p, nsteps=3, max_iter=2)
    assert st["first_failed_step"] == 0 and st["rc"] == hf.HF_E_NOCONV
    # b = 0 (no load, u0 = 0): x = 0 with 0 iterations
    p0 = synth.Problem("zero", p.grid, p.k, p.c, np.zeros(p.grid.n_nodes), theta=1.0, dt=0.01, nsteps=2,
                       rtol=1e-12, flux_face=synth.FACE_ZM, flux_const=0.0)
    u0, st0, _, _, _ = run(p0)
    assert st0["total_iters"] == 0 and np.all(u0 == 0.0)


def test_deterministic_and_snapshots():
    p = synth.c3(n_nodes_axis=50, nsteps=3)
    u1, st1, _, s1, ctx = run(p, snap_plane=0)
    u2, st2, _, s2, _ = run(p, snap_plane=0)
    assert np.array_equal(u1, u2) and np.array_equal(s1, s2)
    assert st1["total_iters"] == st2["total_iters"]
    plane = ctx.n_plane
    np.testing.assert_array_equal(s1.reshape(3, -1)[-1], u1[:plane])


def test_c3_two_steps_full_size():
    p = synth.c3(nsteps=2)
    u, st, plan, _, _ = run(p)
    assert plan["last_used"] == 1 and plan["px"] * plan["py"] * plan["pz"] > 100, plan
    us, _, _, _, _ = run(p, resident=0)
    assert rel(u, us) <= 1e-12
    uo, it = oracle_run(p)
    assert rel(u, uo) <= BAR, rel(u, uo)
    print(f"\n[resident c3] plan {plan}, iterations {st['total_iters']} (oracle {int(it.sum())})")
