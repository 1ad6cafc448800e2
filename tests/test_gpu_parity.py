"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element.

Bars: operator apply / diagonal / load max-abs error <= 1e-12 of the
output scale (rounding-order differences only); PCG and time-step solutions rel-L2 <= 1e-10
(BASELINE.json north_star) at rtol 1e-12.
"""
import threading

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


def on_own_stream(fn, r):
    """Run a slab rank's thread on its own stream: ranks sharing the GPU wait for each other
    inside kernels, so they must never share (or implicitly synchronise with) a stream."""
    with torch.cuda.stream(torch.cuda.Stream(device=DEV)):
        fn(r)


def T(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def N(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def maxerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def make_ctx(grid, k, c, tile_r=None, **tuning):
    ctx = hf.hf_create(grid, 0)
    if tile_r is not None:
        hf.hf_set_tuning(ctx, "tile_r", tile_r)
    for key, v in tuning.items():
        hf.hf_set_tuning(ctx, key, v)
    hf.hf_set_coefficients(ctx, T(k), T(c))
    return ctx


GRIDS = {
    "1x1x1": synth.Grid((1, 1, 1), (1.0, 1.0, 1.0)),
    "c1": synth.Grid((8, 8, 8), (0.125, 0.125, 0.125)),
    "c2bar": synth.Grid((64, 4, 4), (1 / 64, 1 / 64, 1 / 64)),
    "ragged": synth.Grid((70, 40, 13), (0.3, 0.2, 0.7), (-1.0, 2.0, 0.5)),
    "seams": synth.Grid((33, 65, 9), (0.2, 0.2, 0.2)),
    "tall": synth.Grid((5, 3, 60), (0.1, 0.4, 0.05)),
}


# ---------------------------------------------------------------------------------------------
# operator apply (Eq. (1))

@pytest.mark.parametrize("tile_r", [0, 2, 4])
@pytest.mark.parametrize("gname", list(GRIDS))
def test_apply_matches_assembled(gname, tile_r):
    g = GRIDS[gname]
    k, c = synth.random_fields(g, seed=1)
    o = oracle.Oracle(g, k, c)
    ctx = make_ctx(g, k, c, tile_r)
    u = synth.random_vector(g.n_nodes, seed=2)
    ud = T(u)
    y = torch.empty_like(ud)
    for aK, aM in [(1.0, 0.0), (0.0, 1.0), (0.005, 1.0), (-0.005, 1.0)]:
        hf.hf_apply(ctx, aK, aM, ud, y)
        yo = o.spmv(aK, aM, u)
        assert maxerr(N(y), yo) <= 1e-12, (gname, aK, aM)
    # fused axpby (FGDbDMVM_C): y = c A u + b
    b = synth.random_vector(g.n_nodes, seed=3)
    hf.hf_apply_axpby(ctx, 0.01, 1.0, -1.0, ud, T(b), y)
    assert maxerr(N(y), b - o.spmv(0.01, 1.0, u)) <= 1e-12


def test_apply_host_buffers_and_determinism():
    g = GRIDS["ragged"]
    k, c = synth.random_fields(g, seed=4)
    ctx = hf.hf_create(g, 0)
    hf.hf_set_coefficients(ctx, k, c)            # host arrays, staged by the library
    u = synth.random_vector(g.n_nodes, seed=5)
    yh = np.empty_like(u)
    hf.hf_apply(ctx, 0.3, 1.0, u, yh)
    yd = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_apply(ctx, 0.3, 1.0, T(u), yd)
    yd2 = torch.empty_like(yd)
    hf.hf_apply(ctx, 0.3, 1.0, T(u), yd2)
    assert np.array_equal(yh, N(yd)) and np.array_equal(N(yd), N(yd2))
    o = oracle.Oracle(g, k, c)
    assert maxerr(yh, o.spmv(0.3, 1.0, u)) <= 1e-12


def test_apply_single_element_and_constant_field():
    g = GRIDS["1x1x1"]
    ctx = make_ctx(g, [2.0], [3.0])
    Ke, Me = oracle.element_matrices(g.h)
    for j in range(8):
        e = np.zeros(8)
        e[j] = 1.0
        y = torch.empty(8, dtype=torch.float64, device=DEV)
        hf.hf_apply(ctx, 0.25, 1.5, T(e), y)
        assert np.allclose(N(y), 0.5 * Ke[:, j] + 4.5 * Me[:, j], rtol=0, atol=1e-15)
    # K 1 = 0 on a heterogeneous grid
    g = GRIDS["ragged"]
    k, c = synth.random_fields(g, seed=6)
    ctx = make_ctx(g, k, c)
    y = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_apply(ctx, 1.0, 0.0, T(np.ones(g.n_nodes)), y)
    assert np.abs(N(y)).max() <= 1e-12 * k.max() * max(g.h)


# ---------------------------------------------------------------------------------------------
# Jacobi diagonal and flux load

@pytest.mark.parametrize("bits", [0, 0b000011, 0b110100])
def test_diag_matches(bits):
    g = GRIDS["ragged"]
    k, c = synth.random_fields(g, seed=7)
    o = oracle.Oracle(g, k, c)
    ctx = make_ctx(g, k, c)
    vals = (1.0, 2.0, 3.0, 4.0, 5.0, 6.0)
    o.set_dirichlet(bits, vals)
    hf.hf_set_dirichlet_faces(ctx, bits, vals)
    d = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_diag(ctx, 0.02, 1.0, d)
    assert maxerr(N(d), o.diag(0.02, 1.0)) <= 1e-13


@pytest.mark.parametrize("face", range(6))
def test_face_load_matches(face):
    g = GRIDS["ragged"]
    k, c = synth.random_fields(g, seed=8)
    o = oracle.Oracle(g, k, c, assemble=False)
    ctx = make_ctx(g, k, c)
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    for fc, beam in [(1.0, None), (0.0, (10.0, 2.0, 0.5, 3.0)), (0.3, (1.0, 0.7, -0.5, 4.0))]:
        hf.hf_face_load(ctx, face, fc, beam, F)
        Fo = o.face_load(face, fc, beam)
        assert maxerr(N(F), Fo) <= 1e-13, (face, fc, beam)


# ---------------------------------------------------------------------------------------------
# PCG (Alg. 1)

@pytest.mark.parametrize("driver", [0, 1])
def test_cg_matches_oracle(driver):
    p = synth.c1()
    o, F = oracle.problem_oracle(p)
    ctx = make_ctx(p.grid, p.k, p.c)
    hf.hf_set_driver(ctx, driver)
    b = synth.random_vector(p.grid.n_nodes, 9) * 1e5
    x = torch.zeros(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    info = hf.hf_cg(ctx, 0.01, 1.0, T(b), x, rtol=1e-12)
    xo, st, it, _ = o.pcg(0.01, 1.0, b, np.zeros_like(b), tol=1e-12)
    assert info["status"] == 0 and st == 0
    assert rel(N(x), xo) <= 1e-10
    assert abs(info["iters"] - it) <= 3
    assert info["relres"] <= 1e-12


def test_cg_dirichlet_zero_rhs_and_breakdown():
    g = GRIDS["ragged"]
    k, c = synth.random_fields(g, seed=10)
    o = oracle.Oracle(g, k, c)
    ctx = make_ctx(g, k, c)
    vals = (0.7, -0.3, 0.0, 0.0, 0.0, 0.0)
    o.set_dirichlet(3, vals)
    hf.hf_set_dirichlet_faces(ctx, 3, vals)
    F = o.face_load(synth.FACE_ZM, 1.0)
    b = o.rhs(0.5, 0.02, F, synth.random_vector(g.n_nodes, 11))
    x = T(np.zeros(g.n_nodes))
    info = hf.hf_cg(ctx, 0.01, 1.0, T(b), x)
    xo, st, it, _ = o.pcg(0.01, 1.0, b, np.zeros(g.n_nodes))
    assert info["status"] == 0 and rel(N(x), xo) <= 1e-10
    # b = 0 (with g = 0) -> x = 0 in 0 iterations
    hf.hf_set_dirichlet_faces(ctx, 0)
    x = T(np.ones(g.n_nodes))
    info = hf.hf_cg(ctx, 0.01, 1.0, T(np.zeros(g.n_nodes)), x)
    assert info["iters"] == 0 and np.all(N(x) == 0.0)
    # NaN input -> breakdown, reported not crashed
    bn = b.copy()
    bn[5] = np.nan
    info = hf.hf_cg(ctx, 0.01, 1.0, T(bn), T(np.zeros(g.n_nodes)), raise_on_noconv=False)
    assert info["rc"] in (hf.HF_E_BREAKDOWN, hf.HF_E_NOCONV)
    # max_iter too small -> NOCONV with the last iterate
    info = hf.hf_cg(ctx, 0.01, 1.0, T(b), T(np.zeros(g.n_nodes)), max_iter=3, raise_on_noconv=False)
    assert info["rc"] == hf.HF_E_NOCONV and info["iters"] == 3


# ---------------------------------------------------------------------------------------------
# time stepping

def _gpu_sim(p, driver=0, snap_plane=-1, tile_r=None, **tuning):
    ctx = make_ctx(p.grid, p.k, p.c, tile_r, **tuning)
    hf.hf_set_driver(ctx, driver)
    if p.dirichlet_bits:
        hf.hf_set_dirichlet_faces(ctx, p.dirichlet_bits, p.dirichlet_values)
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    u = T(p.u0)
    snap = None
    if snap_plane >= 0:
        snap = torch.empty(p.nsteps * ctx.n_plane, dtype=torch.float64, device=DEV)
    st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, snap_plane, snap, rtol=p.rtol)
    return N(u), st, (None if snap is None else N(snap)), ctx


@pytest.mark.parametrize("tile_r", [0, 2, 4])
def test_simulate_c1(tile_r):
    p = synth.c1()
    ug, st, _, _ = _gpu_sim(p, tile_r=tile_r)
    o, F = oracle.problem_oracle(p)
    uo, sto, it, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0, tol=p.rtol)
    assert st["steps_done"] == p.nsteps and st["first_failed_step"] == -1
    assert rel(ug, uo) <= 1e-10
    assert abs(st["total_iters"] - int(it.sum())) <= 3 * p.nsteps


def test_graph_and_host_drivers_bitwise_equal():
    p = synth.c1()
    ug, st0, s0, _ = _gpu_sim(p, driver=0, snap_plane=0)
    uh, st1, s1, _ = _gpu_sim(p, driver=1, snap_plane=0)
    assert np.array_equal(ug, uh) and np.array_equal(s0, s1)
    assert st0["total_iters"] == st1["total_iters"]


@pytest.mark.parametrize("driver,unroll", [(0, 1), (0, 3), (1, 1)])
def test_failed_step_stops_the_run(driver, unroll):
    """A step that does not converge (max_iter too small) stops the run: the later steps of the
    same call are skipped on the device (no host check between graph launches), the call returns
    NOCONV with the failing step, and the graph WHILE loops of the skipped steps terminate."""
    p = synth.c1()
    ctx = make_ctx(p.grid, p.k, p.c, unroll=unroll)
    hf.hf_set_driver(ctx, driver)
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = T(p.u0)
    st = hf.hf_simulate(ctx, p.theta, p.dt, 4, F, u, rtol=p.rtol, max_iter=2, raise_on_noconv=False)
    assert st["rc"] == hf.HF_E_NOCONV and st["first_failed_step"] == 0
    # the context stays usable: a converging run afterwards matches the oracle
    u2 = T(p.u0)
    st2 = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u2, rtol=p.rtol)
    o, Fo = oracle.problem_oracle(p)
    uo, _, _, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
    assert st2["first_failed_step"] == -1 and rel(N(u2), uo) <= 1e-10


def test_time_kernel_a_replay_then_simulate():
    """Instrumentation replay of kernel A leaves the context usable: the next run matches."""
    p = synth.c1()
    ug, st0, _, ctx = _gpu_sim(p)
    with pytest.raises(hf.HfError):
        hf.hf_time_kernel_a(make_ctx(p.grid, p.k, p.c), 5)      # no simulation yet: HF_E_STATE
    ms = hf.hf_time_kernel_a(ctx, 20)
    assert 0.0 < ms < 10.0
    msg = hf.hf_time_kernel_a_graph(ctx, 20)             # graph chain with programmatic edges
    assert 0.0 < msg < 10.0
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    u = T(p.u0)
    st1 = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol)
    assert np.array_equal(N(u), ug) and st1["total_iters"] == st0["total_iters"]


@pytest.mark.parametrize("unroll", [2, 4])
def test_unrolled_loop_body_bitwise_equal(unroll):
    p = synth.c1()
    ug, st0, _, _ = _gpu_sim(p, driver=0)
    uu, st1, _, _ = _gpu_sim(p, driver=0, unroll=unroll)
    assert np.array_equal(ug, uu) and st0["total_iters"] == st1["total_iters"]


def test_simulate_c2_closed_form():
    p = synth.c2()
    ug, st, _, _ = _gpu_sim(p)
    g = p.grid
    h = g.h[0]
    x, _, _ = g.node_coords()
    lam = (6 / h ** 2) * (1 - np.cos(np.pi * h)) / (2 + np.cos(np.pi * h))
    G = (1 - (1 - p.theta) * p.dt * lam) / (1 + p.theta * p.dt * lam)
    ex = G ** p.nsteps * np.sin(np.pi * x.ravel())
    ex[np.isclose(x.ravel(), 1.0)] = 0.0
    assert rel(ug, ex) <= 1e-10
    o, F = oracle.problem_oracle(p)
    uo, _, _, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0, tol=p.rtol)
    assert rel(ug, uo) <= 1e-10


def test_simulate_nonzero_dirichlet_and_beam():
    g = synth.Grid((20, 14, 9), (0.3, 0.3, 0.25), (-3.0, -2.0, 0.0))
    k, c = synth.random_fields(g, seed=12)
    p = synth.Problem("dir", g, k, c, synth.random_vector(g.n_nodes, 13), theta=0.5, dt=0.05, nsteps=8,
                      beam=(10.0, 1.0, 0.0, 0.0), flux_const=0.2, dirichlet_bits=0b100001,
                      dirichlet_values=(1.5, 0.0, 0.0, 0.0, 0.0, -0.5))
    ug, st, snap, _ = _gpu_sim(p, snap_plane=0)
    o, F = oracle.problem_oracle(p)
    uo, sto, it, so = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0, tol=p.rtol, snap_plane=0)
    assert sto == 0 and rel(ug, uo) <= 1e-10
    assert rel(snap, so.ravel()) <= 1e-10


def test_resume_equals_one_run():
    p = synth.c1()
    ctx = make_ctx(p.grid, p.k, p.c)
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u1 = T(p.u0)
    hf.hf_simulate(ctx, p.theta, p.dt, 10, F, u1)
    u2 = T(p.u0)
    up = torch.empty_like(u2)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, 4, F, u2, up, 0)
    hf.hf_simulate_resume(ctx, p.theta, p.dt, 6, F, u2, up, 4)
    assert np.array_equal(N(u1), N(u2))


@pytest.mark.parametrize("group", [None, 2, 1])
def test_batched_matches_individual(group):
    """Batched sims: systems stacked along z with per-system PCG (default group; groups of 2, the
    last group smaller; one system per group) against the oracle."""
    g = synth.Grid((12, 10, 9), (0.3, 0.3, 0.2))
    B = 3
    base_k, base_c = synth.random_fields(g, seed=14)
    ks = np.stack([base_k * synth.lognormal_perturbation(g.n_elems, seed=20 + j) for j in range(B)])
    cs = np.stack([base_c * (1.0 + 0.1 * j) for j in range(B)])
    u0 = np.zeros((B, g.n_nodes))
    for shared_c in (False, True):
        ctx = make_ctx(g, base_k, base_c, batch_group=group or 0)
        F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
        hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
        ub = T(u0.ravel())
        front = torch.empty(B * ctx.n_plane, dtype=torch.float64, device=DEV)
        stats = hf.hf_simulate_batched(ctx, B, T(ks.ravel()), None if shared_c else T(cs.ravel()), 0.5, 0.05, 6,
                                       F, ub, 0, front)
        ub = N(ub).reshape(B, -1)
        front = N(front).reshape(B, -1)
        for j in range(B):
            cj = base_c if shared_c else cs[j]
            o = oracle.Oracle(g, ks[j], cj)
            Fo = o.face_load(synth.FACE_ZM, 1.0)
            uo, st, it, _ = o.simulate(0.5, 0.05, 6, Fo, u0[j])
            assert rel(ub[j], uo) <= 1e-10, (shared_c, j)
            assert np.array_equal(front[j], ub[j][: ctx.n_plane])
            assert stats[j]["steps_done"] == 6


def test_batched_systems_have_their_own_pcg():
    """Per-system PCG in a stack (a13; Alg. 1 per solve): one system's load is 1e-3 x the others',
    another system is insulated with a zero load (b = 0: 0 iterations, x = 0); every system still
    meets rtol against its own ||b_j||, matches its oracle, and the iteration counts differ."""
    g = synth.Grid((12, 10, 9), (0.3, 0.3, 0.2))
    B = 5
    base_k, base_c = synth.random_fields(g, seed=51)
    ks = np.stack([base_k * synth.lognormal_perturbation(g.n_elems, seed=60 + j) for j in range(B)])
    ctx = make_ctx(g, base_k, base_c)
    # no flux; the systems differ by their initial fields, so b_j = L u0_j: system 1's right-hand
    # side is 1e-3 x the others', system 3's is zero
    scale = np.array([1.0, 1e-3, 1.0, 0.0, 1.0])
    rng = np.random.default_rng(7)
    u0 = np.stack([scale[j] * rng.standard_normal(g.n_nodes) for j in range(B)])
    Fz = np.zeros(g.n_nodes)
    ub = T(u0.ravel())
    stats = hf.hf_simulate_batched(ctx, B, T(ks.ravel()), None, 0.5, 0.05, 5, T(Fz), ub)
    ub = N(ub).reshape(B, -1)
    its = []
    for j in range(B):
        o = oracle.Oracle(g, ks[j], base_c)
        uo, st, it, _ = o.simulate(0.5, 0.05, 5, Fz, u0[j])
        if scale[j] == 0.0:
            assert np.all(ub[j] == 0.0) and stats[j]["total_iters"] == 0
        else:
            assert rel(ub[j], uo) <= 1e-10, j
            assert abs(stats[j]["total_iters"] - int(it.sum())) <= 2, (j, stats[j], it)
        its.append(stats[j]["total_iters"])
        assert stats[j]["steps_done"] == 5 and stats[j]["first_failed_step"] == -1
    assert len(set(its)) > 1, its


def test_batched_z_face_dirichlet():
    """Dirichlet values on the z faces apply to each stacked system's own z faces."""
    g = synth.Grid((8, 7, 6), (0.3, 0.3, 0.2))
    B = 3
    base_k, base_c = synth.random_fields(g, seed=71)
    ks = np.stack([base_k * synth.lognormal_perturbation(g.n_elems, seed=80 + j) for j in range(B)])
    vals = (0.0, 0.0, 0.0, 0.0, 1.5, -0.5)
    ctx = make_ctx(g, base_k, base_c)
    hf.hf_set_dirichlet_faces(ctx, 48, vals)
    ub = torch.zeros(B * g.n_nodes, dtype=torch.float64, device=DEV)
    stats = hf.hf_simulate_batched(ctx, B, T(ks.ravel()), None, 0.5, 0.05, 4, None, ub)
    ub = N(ub).reshape(B, -1)
    for j in range(B):
        o = oracle.Oracle(g, ks[j], base_c)
        o.set_dirichlet(48, vals)
        uo, st, it, _ = o.simulate(0.5, 0.05, 4, np.zeros(g.n_nodes), np.zeros(g.n_nodes))
        assert rel(ub[j], uo) <= 1e-10, j
        assert abs(stats[j]["total_iters"] - int(it.sum())) <= 2


def test_batched_follows_operator_setters():
    """Dirichlet faces / values and the element type changed between two batched calls on the
    same context reach every later call (the batched path must not keep stale operators)."""
    g = synth.Grid((10, 9, 8), (0.3, 0.3, 0.2))
    B = 4
    base_k, base_c = synth.random_fields(g, seed=31)
    ks = np.stack([base_k * synth.lognormal_perturbation(g.n_elems, seed=40 + j) for j in range(B)])
    ctx = make_ctx(g, base_k, base_c)
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    Fh = N(F)
    for bits, vals, elem in [(1, (0.0,) * 6, 0), (3, (0.5, -0.25, 0, 0, 0, 0), 0), (3, (0.5, -0.25, 0, 0, 0, 0), 1),
                             (0, (0.0,) * 6, 1)]:
        hf.hf_set_dirichlet_faces(ctx, bits, vals)
        hf.hf_set_element(ctx, elem)
        if elem == 1:
            hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
            Fh = N(F)
        ub = torch.zeros(B * g.n_nodes, dtype=torch.float64, device=DEV)
        hf.hf_simulate_batched(ctx, B, T(ks.ravel()), None, 0.5, 0.05, 4, F, ub)
        ub = N(ub).reshape(B, -1)
        for j in range(B):
            o = oracle.Oracle(g, ks[j], base_c, elem=elem)
            if bits:
                o.set_dirichlet(bits, vals)
            uo, st, it, _ = o.simulate(0.5, 0.05, 4, Fh, np.zeros(g.n_nodes))
            assert rel(ub[j], uo) <= 1e-10, (bits, vals, elem, j)


# ---------------------------------------------------------------------------------------------
# z-slabs through the in-process transport (same kernels and exchange protocol as NCCL)

@pytest.mark.parametrize("nranks", [2, 3])
def test_slab_local_transport(nranks):
    g = synth.Grid((14, 11, 17), (0.3, 0.3, 0.2))
    k, c = synth.random_fields(g, seed=15)
    theta, dt, nsteps = 0.5, 0.05, 5
    # single-context reference (GPU) and oracle
    ctx1 = make_ctx(g, k, c)
    F1 = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx1, synth.FACE_ZM, 1.0, None, F1)
    u0 = synth.random_vector(g.n_nodes, 16) * 0.01
    u1 = T(u0)
    hf.hf_simulate(ctx1, theta, dt, nsteps, F1, u1)
    ref = N(u1)
    o = oracle.Oracle(g, k, c)
    uo, _, _, _ = o.simulate(theta, dt, nsteps, o.face_load(synth.FACE_ZM, 1.0), u0)
    assert rel(ref, uo) <= 1e-10

    grp = hf.hf_local_group_create(nranks)
    plane = (g.ne[0] + 1) * (g.ne[1] + 1)
    out = [None] * nranks
    errs = []
    ctxs = [None] * nranks

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            ctx = hf.hf_create_slab(g, r, nranks, grp, transport=1, device=0)
            ctxs[r] = ctx
            lo, hi, lp, z0 = ctx.slab
            hf.hf_set_coefficients(ctx, T(k), T(c))
            F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=DEV)
            hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
            u = T(u0[z0 * plane:(z0 + lp) * plane])
            hf.hf_simulate(ctx, theta, dt, nsteps, F, u)
            out[r] = (lo, hi, z0, N(u))
            # apply on the slab: owned planes must equal the global apply
            y = torch.empty_like(u)
            hf.hf_apply(ctx, 0.2, 1.0, T(u0[z0 * plane:(z0 + lp) * plane]), y)
            out[r] = out[r] + (N(y),)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=on_own_stream, args=(rank_main, r)) for r in range(nranks)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs
    full = np.empty(g.n_nodes)
    yfull = np.empty(g.n_nodes)
    for lo, hi, z0, u, y in out:
        full[lo * plane:hi * plane] = u[(lo - z0) * plane:(hi - z0) * plane]
        yfull[lo * plane:hi * plane] = y[(lo - z0) * plane:(hi - z0) * plane]
    assert rel(full, ref) <= 1e-12
    assert rel(full, uo) <= 1e-10
    assert maxerr(yfull, o.spmv(0.2, 1.0, u0)) <= 1e-12
    del ctxs
    hf.hf_local_group_destroy(grp)


# ---------------------------------------------------------------------------------------------
# BASELINE sizes: C3 (1M DoF) in full, C4 (512^3) on sampled rows

@pytest.fixture(scope="module")
def c3():
    return synth.c3(nsteps=2)


def test_c3_apply_and_two_steps(c3):
    p = c3
    o, F = oracle.problem_oracle(p)
    ctx = make_ctx(p.grid, p.k, p.c)
    u = synth.random_vector(p.grid.n_nodes, 17)
    y = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    for aK, aM in [(p.theta * p.dt, 1.0), (-(1 - p.theta) * p.dt, 1.0)]:
        hf.hf_apply(ctx, aK, aM, T(u), y)
        assert maxerr(N(y), o.spmv(aK, aM, u)) <= 1e-12
    Fd = torch.empty_like(y)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, Fd)
    assert maxerr(N(Fd), F) <= 1e-13
    ud = T(p.u0)
    st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, Fd, ud, rtol=p.rtol)
    uo, sto, it, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0, tol=p.rtol)
    assert rel(N(ud), uo) <= 1e-10
    assert abs(st["total_iters"] - int(it.sum())) <= 10


@pytest.mark.slow
def test_c4_apply_sampled_rows():
    g = synth.c4_grid()
    k, c = synth.random_fields(g, seed=18)
    u = synth.random_vector(g.n_nodes, 19)
    ctx = make_ctx(g, k, c)
    y = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_apply(ctx, 0.005, 1.0, T(u), y)
    yg = N(y)
    del ctx
    torch.cuda.empty_cache()
    o = oracle.Oracle(g, k, c, assemble=False)
    rng = np.random.default_rng(20)
    nx, ny, nz = g.nn
    rows = rng.integers(0, g.n_nodes, 4096)
    # plus every boundary class: corners, faces, tile seams (x = 30/31/32, y = 30/31)
    extra = []
    for (i, j, kk) in [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (30, 30, 7), (31, 31, 8), (32, 62, 9), (61, 93, 500),
                       (nx - 1, 0, 3), (0, ny - 1, nz - 1)]:
        extra.append(i + nx * (j + ny * kk))
    rows = np.concatenate([rows, np.array(extra)])
    yo = o.apply_rows(0.005, 1.0, u, rows)
    assert maxerr(yg[rows], yo) <= 1e-12


def test_c5_corrosion_batched_small():
    """C5 recipe (corrosion plate, anisotropic voxels, Gaussian beam, perturbed k) at 20^3 nodes:
    each batched forward simulation matches the oracle; front-face output is the z = 0 plane."""
    B, nax, nsteps = 3, 20, 12
    probs = [synth.c5(j, n_nodes_axis=nax, nsteps=nsteps) for j in range(B)]
    g = probs[0].grid
    ctx = make_ctx(g, probs[0].k, probs[0].c)
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, probs[0].flux_face, probs[0].flux_const, probs[0].beam, F)
    ub = T(np.zeros(B * g.n_nodes))
    front = torch.empty(B * ctx.n_plane, dtype=torch.float64, device=DEV)
    kb = np.stack([p.k for p in probs]).ravel()
    cb = np.stack([p.c for p in probs]).ravel()
    hf.hf_simulate_batched(ctx, B, T(kb), T(cb), probs[0].theta, probs[0].dt, nsteps, F, ub, 0, front)
    ub = N(ub).reshape(B, -1)
    front = N(front).reshape(B, -1)
    for j, p in enumerate(probs):
        o, Fo = oracle.problem_oracle(p)
        uo, st, it, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
        assert st == 0 and rel(ub[j], uo) <= 1e-10, j
        assert np.array_equal(front[j], ub[j][:ctx.n_plane])
    # deeper corrosion (less conductive oxide near the rear) -> different front-face fields
    assert np.abs(front[0] - front[1]).max() > 1e-6 * np.abs(front[0]).max()


def test_c5_full_size_stacked_two_steps():
    """C5 at its BASELINE size (100^3 nodes per sim) in bench.py's launch configuration (a
    block-diagonal stack of 4 systems): 2 steps of two of the systems against the oracle."""
    B, nsteps = 4, 2
    probs = [synth.c5(j) for j in range(B)]            # the bench's dt = T_F / 300; 2 of its steps
    g = probs[0].grid
    ctx = make_ctx(g, probs[0].k, probs[0].c)
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, probs[0].flux_face, probs[0].flux_const, probs[0].beam, F)
    ub = T(np.zeros(B * g.n_nodes))
    front = torch.empty(B * ctx.n_plane, dtype=torch.float64, device=DEV)
    kb = np.stack([p.k for p in probs]).ravel()
    cb = np.stack([p.c for p in probs]).ravel()
    st = hf.hf_simulate_batched(ctx, B, T(kb), T(cb), probs[0].theta, probs[0].dt, nsteps, F, ub, 0, front)
    assert all(s["steps_done"] == nsteps for s in st)
    ub = N(ub).reshape(B, -1)
    for j in (0, 3):
        o, Fo = oracle.problem_oracle(probs[j])
        uo, sto, _, _ = o.simulate(probs[j].theta, probs[j].dt, nsteps, Fo, probs[j].u0, tol=probs[j].rtol)
        assert sto == 0 and rel(ub[j], uo) <= 1e-10, j


@pytest.mark.parametrize("transport", [0, 1, 2])
def test_slab_single_rank_nccl_and_local(transport):
    """A 1-rank slab context runs the slab driver -- through real NCCL for transport 0 (host loop,
    k_localsum, allreduce), through the peer-memory protocol for 1 (in-process group) and 2
    (export / connect handshake with itself; in-kernel publish and wait, step graph) -- and must
    reproduce the plain single-GPU run bit for bit (same kernels, same reduction order)."""
    p = synth.c1()
    ug, st, _, _ = _gpu_sim(p)
    if transport == 0:
        uid = hf.hf_nccl_unique_id()
        ctx = hf.hf_create_slab(p.grid, 0, 1, uid, transport=0, device=0)
    elif transport == 1:
        grp = hf.hf_local_group_create(1)
        ctx = hf.hf_create_slab(p.grid, 0, 1, grp, transport=1, device=0)
    else:
        ctx = hf.hf_create_slab(p.grid, 0, 1, None, transport=2, device=0)
        with pytest.raises(hf.HfError):          # not connected yet
            hf.hf_simulate(ctx, p.theta, p.dt, 1, None, T(p.u0))
        hf.hf_peer_setup(ctx, lambda b: [b])
    hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    u = T(p.u0)
    st2 = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol)
    assert np.array_equal(N(u), ug)
    assert st2["total_iters"] == st["total_iters"]
    del ctx


# ---------------------------------------------------------------------------------------------
# NEXT row f1: the paper's element (6 P1 tets per voxel)

@pytest.mark.parametrize("gname", ["1x1x1", "c1", "ragged", "seams"])
def test_tet_apply_diag_load(gname):
    g = GRIDS[gname]
    k, c = synth.random_fields(g, seed=41)
    o = oracle.Oracle(g, k, c, elem=1)
    ctx = make_ctx(g, k, c)
    hf.hf_set_element(ctx, 1)
    u = synth.random_vector(g.n_nodes, seed=42)
    y = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    for aK, aM in [(1.0, 0.0), (0.0, 1.0), (0.005, 1.0)]:
        hf.hf_apply(ctx, aK, aM, T(u), y)
        assert maxerr(N(y), o.spmv(aK, aM, u)) <= 1e-12, (gname, aK, aM)
    d = torch.empty_like(y)
    hf.hf_diag(ctx, 0.02, 1.0, d)
    assert maxerr(N(d), o.diag(0.02, 1.0)) <= 1e-13
    for face in (synth.FACE_ZM, synth.FACE_XP):
        for fc, beam in [(1.0, None), (0.0, (10.0, 0.7, 0.5, 0.3))]:
            hf.hf_face_load(ctx, face, fc, beam, y)
            assert maxerr(N(y), o.face_load(face, fc, beam)) <= 1e-13, (face, fc)


@pytest.mark.parametrize("driver", [0, 1])
def test_tet_simulate_matches_oracle(driver):
    g = synth.Grid((14, 11, 9), (0.3, 0.3, 0.25), (-2.0, -1.5, 0.0))
    ids = synth.inclusion_ids(g, seed=43)
    k, c = synth.ids_to_fields(ids)
    p = synth.Problem("tet", g, k, c, np.zeros(g.n_nodes), theta=0.5, dt=0.02, nsteps=6,
                      beam=(synth.BEAM_POWER, 1.5, 0.0, 0.0), dirichlet_bits=1 << synth.FACE_ZP,
                      dirichlet_values=(0, 0, 0, 0, 0, 0.25))
    ctx = make_ctx(g, k, c)
    hf.hf_set_element(ctx, 1)
    hf.hf_set_driver(ctx, driver)
    hf.hf_set_dirichlet_faces(ctx, p.dirichlet_bits, p.dirichlet_values)
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    u = T(p.u0)
    st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol)
    o, Fo = oracle.problem_oracle(p, elem=1)
    uo, sto, it, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
    assert sto == 0 and st["steps_done"] == p.nsteps
    assert rel(N(u), uo) <= 1e-10


def test_pdl_edges_do_not_change_results():
    """The programmatic-launch edges of the PCG loop body (tuning "pdl", default on) only let the
    next kernel start early: the solution is bit-identical to fully serialised edges."""
    p = synth.c1()
    outs = []
    for pdl in (0, 1):
        ctx = make_ctx(p.grid, p.k, p.c, pdl=pdl)
        F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
        hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
        u = T(p.u0)
        st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol)
        outs.append((N(u), st["total_iters"]))
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]


@pytest.mark.slow
@pytest.mark.parametrize("mixed", [None, 1e-7])
def test_c4_time_step_properties(mixed):
    """C4 (512^3 nodes, 134M DoF) in the configuration bench.py's c4_steps / c4_steps_mixed
    times: one backward-free CN step from u0 = 0 must leave a true residual ||dt F - A u1|| <=
    1e-10 ||dt F|| (the solve met rtol 1e-12 on the recurrence residual; Alg. 1 replaces it every
    50 iterations; mixed: the fp64 finish after the fp32 stage), and the stiffness part must
    carry no heat: sum(A u1) = sum(M u1) (K 1 = 0, K symmetric)."""
    g = synth.c4_grid()
    gen = torch.Generator(device=DEV).manual_seed(3)
    ox = torch.rand(g.n_elems, device=DEV, generator=gen) < 0.2
    k = torch.where(ox, synth.OXIDE[1], synth.STEEL[1]).to(torch.float64)
    c = torch.where(ox, synth.OXIDE[0], synth.STEEL[0]).to(torch.float64)
    del ox
    ctx = hf.hf_create(g, 0)
    if mixed:
        hf.hf_set_mixed(ctx, 1, mixed)
    hf.hf_set_coefficients(ctx, k, c)
    del k, c
    torch.cuda.empty_cache()
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = torch.zeros(g.n_nodes, dtype=torch.float64, device=DEV)
    theta, dt = 0.5, 0.01
    st = hf.hf_simulate(ctx, theta, dt, 1, F, u, rtol=1e-12)
    assert st["total_iters"] > 0
    y = torch.empty_like(u)
    hf.hf_apply_axpby(ctx, theta * dt, 1.0, -1.0, u, F * dt, y)         # r = dt F - A u1
    rel_res = float(torch.linalg.norm(y) / torch.linalg.norm(F * dt))
    assert rel_res <= 1e-10, rel_res
    hf.hf_apply(ctx, theta * dt, 1.0, u, y)
    sa = float(y.sum())
    hf.hf_apply(ctx, 0.0, 1.0, u, y)
    sm = float(y.sum())
    assert abs(sa - sm) <= 1e-9 * abs(sm), (sa, sm)
    assert abs(sm - dt * float(F.sum())) <= 1e-9 * abs(sm)


def test_empty_inputs():
    """Degenerate calls: 0 time steps leave u unchanged and report 0 steps; a batch of 0 systems
    is a no-op; a 0-iteration cap on a non-trivial step reports NOCONV at step 0."""
    p = synth.c1()
    ctx = make_ctx(p.grid, p.k, p.c)
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u0 = synth.random_vector(p.grid.n_nodes, 5)
    u = T(u0)
    st = hf.hf_simulate(ctx, p.theta, p.dt, 0, F, u, rtol=p.rtol)
    assert st["steps_done"] == 0 and st["total_iters"] == 0
    assert np.array_equal(N(u), u0)
    ub = torch.zeros(0, dtype=torch.float64, device=DEV)
    kb = torch.zeros(0, dtype=torch.float64, device=DEV)
    hf.hf_simulate_batched(ctx, 0, kb, None, p.theta, p.dt, 3, F, ub)
    u = T(u0)
    st = hf.hf_simulate(ctx, p.theta, p.dt, 2, F, u, rtol=p.rtol, max_iter=0, raise_on_noconv=False)
    assert st["rc"] == hf.HF_E_NOCONV and st["first_failed_step"] == 0


def test_slab_local_transport_tets_and_mixed_tets():
    """The paper's 6-tet element (row f1) on 2 in-process z-slabs against one context and the
    oracle's tet assembly; and the tet element through mixed precision (fp32 correction, fp64
    finish) against the oracle."""
    g = synth.Grid((10, 9, 12), (0.3, 0.3, 0.2))
    k, c = synth.random_fields(g, seed=25)
    theta, dt, nsteps, nranks = 0.5, 0.05, 4, 2
    o = oracle.Oracle(g, k, c, elem=1)
    Fo = o.face_load(synth.FACE_ZM, 1.0)
    u0 = synth.random_vector(g.n_nodes, 26) * 0.01
    uo, _, _, _ = o.simulate(theta, dt, nsteps, Fo, u0)
    # mixed precision, one context
    ctxm = hf.hf_create(g, 0)
    hf.hf_set_mixed(ctxm, 1, 1e-5)
    hf.hf_set_element(ctxm, 1)
    hf.hf_set_coefficients(ctxm, T(k), T(c))
    Fm = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctxm, synth.FACE_ZM, 1.0, None, Fm)
    um = T(u0)
    hf.hf_simulate(ctxm, theta, dt, nsteps, Fm, um)
    assert rel(N(um), uo) <= 1e-10
    # two slabs
    grp = hf.hf_local_group_create(nranks)
    plane = (g.ne[0] + 1) * (g.ne[1] + 1)
    out = [None] * nranks
    errs = []
    ctxs = [None] * nranks

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            ctx = hf.hf_create_slab(g, r, nranks, grp, transport=1, device=0)
            ctxs[r] = ctx
            lo, hi, lp, z0 = ctx.slab
            hf.hf_set_element(ctx, 1)
            hf.hf_set_coefficients(ctx, T(k), T(c))
            F = torch.empty(ctx.n_nodes, dtype=torch.float64, device=DEV)
            hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
            u = T(u0[z0 * plane:(z0 + lp) * plane])
            hf.hf_simulate(ctx, theta, dt, nsteps, F, u)
            out[r] = (lo, hi, z0, N(u))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=on_own_stream, args=(rank_main, r)) for r in range(nranks)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs
    full = np.empty(g.n_nodes)
    for lo, hi, z0, u in out:
        full[lo * plane:hi * plane] = u[(lo - z0) * plane:(hi - z0) * plane]
    assert rel(full, uo) <= 1e-10
    del ctxs
    hf.hf_local_group_destroy(grp)


def test_tuning_api_and_environment_defaults(monkeypatch):
    """hf_set_tuning / hf_get_tuning: values, range checks, unknown keys; HF_* environment
    variables only give the defaults of a context at its creation."""
    p = synth.c1()
    monkeypatch.setenv("HF_UNROLL", "3")
    monkeypatch.setenv("HF_ZCHUNK", "4")
    ctx = make_ctx(p.grid, p.k, p.c)
    monkeypatch.delenv("HF_UNROLL")
    monkeypatch.delenv("HF_ZCHUNK")
    assert hf.hf_get_tuning(ctx, "unroll") == 3 and hf.hf_get_tuning(ctx, "zchunk") == 4
    assert hf.hf_get_tuning(ctx, "tile_r") == 2                   # default below 16M nodes
    hf.hf_set_tuning(ctx, "tile_r", 4)
    assert hf.hf_get_tuning(ctx, "tile_r") == 4
    for key, bad in (("tile_r", 3), ("unroll", 51), ("pdl", 2), ("check_every", 0), ("nope", 1)):
        with pytest.raises(hf.HfError):
            hf.hf_set_tuning(ctx, key, bad)
    # the tuned context (R = 4 tiles, 4-plane chunks, 3 iterations per body) still matches
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    u = T(p.u0)
    hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol)
    o, Fo = oracle.problem_oracle(p)
    uo, _, _, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
    assert rel(N(u), uo) <= 1e-10
