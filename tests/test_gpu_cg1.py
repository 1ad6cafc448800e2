"""The single-reduction PCG (hf_set_cg_variant 1: the Chronopoulos-Gear arrangement of Alg. 1,
one stencil kernel per iteration) against the oracle at the fp64 bars
(rel-L2 <= 1e-10 at rtol 1e-12) and against Alg. 1's two-kernel path.  The same Krylov iterates
in exact arithmetic: iteration counts may differ by rounding near the stop test, not results."""
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


def T(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def N(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def sim(p, variant, driver=0, nsteps=None, ids=False, **kw):
    ctx = hf.hf_create(p.grid, 0)
    hf.hf_set_cg_variant(ctx, variant)
    if driver:
        hf.hf_set_driver(ctx, driver)
    if ids:
        hf.hf_set_material_ids(ctx, torch.tensor(p.extra["ids"], device=DEV), [m[1] for m in p.extra["materials"]],
                               [m[0] for m in p.extra["materials"]])
    else:
        hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, p.beam, F)
    u = T(p.u0)
    st = hf.hf_simulate(ctx, p.theta, p.dt, nsteps or p.nsteps, F, u, rtol=p.rtol, **kw)
    return N(u), st, hf.hf_cg_variant(ctx)["last_used"]


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_cg1_simulate_matches_oracle(name):
    p = synth.c1() if name == "c1" else synth.c3(nsteps=2)
    u, st, used = sim(p, 1)
    assert used == 1
    o, Fo = oracle.problem_oracle(p)
    uo, _, it, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
    assert rel(u, uo) <= 1e-10
    assert abs(st["total_iters"] - int(it.sum())) <= 2 * p.nsteps + 2


def test_cg1_equals_two_kernel_path_c3():
    """Same iterates in exact arithmetic: C3, 3 steps, the two variants within 1e-13 of each
    other and with the same iteration counts (+-1 per step)."""
    p = synth.c3(nsteps=3)
    u1, s1, _ = sim(p, 1)
    u0, s0, used0 = sim(p, 0)
    assert used0 == 0
    assert rel(u1, u0) <= 1e-13
    assert abs(s1["total_iters"] - s0["total_iters"]) <= p.nsteps


def test_cg1_material_ids_bitwise_pairs():
    """Materials by id stream uint8 ids into the same kernel (EL_Q1P): bitwise the pair result."""
    p = synth.c3(n_nodes_axis=40, nsteps=2)
    u_ids, _, used = sim(p, 1, ids=True)
    u_pairs, _, _ = sim(p, 1)
    assert used == 1
    assert np.array_equal(u_ids, u_pairs)


def test_cg1_dirichlet_ragged_and_replacement():
    """Non-zero Dirichlet faces, a ragged grid, more than 50 iterations per solve (residual
    replacement: r = b - A x, then w = A P^-1 r, through the IF node), against the oracle."""
    g = synth.Grid((70, 40, 13), (0.3, 0.2, 0.7), (-1.0, 2.0, 0.5))
    k, c = synth.random_fields(g, seed=95)
    ctx = hf.hf_create(g, 0)
    hf.hf_set_cg_variant(ctx, 1)
    hf.hf_set_coefficients(ctx, T(k), T(c))
    bits = (1 << synth.FACE_XM) | (1 << synth.FACE_ZP)
    vals = [1.0, 0, 0, 0, 0, -0.5]
    hf.hf_set_dirichlet_faces(ctx, bits, vals)
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = T(np.zeros(g.n_nodes))
    st = hf.hf_simulate(ctx, 0.5, 0.5, 4, F, u)
    assert hf.hf_cg_variant(ctx)["last_used"] == 1
    assert st["max_iters_step"] > 50
    o = oracle.Oracle(g, k, c)
    o.set_dirichlet(bits, tuple(vals))
    uo, _, it, _ = o.simulate(0.5, 0.5, 4, o.face_load(synth.FACE_ZM, 1.0), np.zeros(g.n_nodes))
    assert rel(N(u), uo) <= 1e-10
    assert abs(st["total_iters"] - int(it.sum())) <= 8


def test_cg1_host_driver_bitwise_graph():
    """The host-loop driver launches the same kernels in the same order: bitwise the graph run."""
    p = synth.c1()
    u_g, s_g, _ = sim(p, 1)
    u_h, s_h, used = sim(p, 1, driver=1)
    assert used == 1
    assert np.array_equal(u_g, u_h)
    assert s_g["total_iters"] == s_h["total_iters"]


def test_cg1_noconv_and_zero_rhs():
    p = synth.c1()
    _, st, _ = sim(p, 1, max_iter=3, raise_on_noconv=False)
    assert st["rc"] == hf.HF_E_NOCONV and st["first_failed_step"] == 0
    # b_F = 0 (zero flux, zero initial state): x_F = 0 without iterations
    q = synth.c1()
    q.flux_const = 0.0
    q.u0 = np.zeros_like(q.u0)
    u, st, _ = sim(q, 1)
    assert st["total_iters"] == 0 and not np.any(u)


def test_cg1_ineligible_contexts_run_alg1():
    """fp32 storage and the tet element are not eligible: the two-kernel path runs (variant 0)."""
    p = synth.c1()
    ctx = hf.hf_create(p.grid, 0)
    hf.hf_set_precision(ctx, 32)
    hf.hf_set_cg_variant(ctx, 1)
    hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = T(p.u0)
    hf.hf_simulate(ctx, p.theta, p.dt, 2, F, u, rtol=1e-6)
    assert hf.hf_cg_variant(ctx) == {"variant": 1, "last_used": 0}
    with pytest.raises(hf.HfError):
        hf.hf_set_cg_variant(ctx, 2)
