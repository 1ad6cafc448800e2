"""The fused PCG iteration (hf_set_tuning(ctx, "fuse_ab", 1): kernel A, a grid barrier and kernel B's work in one
launch inside the graph loop body) against the oracle: the same bars as the two-kernel path
(rel-L2 <= 1e-10 at rtol 1e-12).  The grouping of kernel B's partial sums differs, so iteration
counts may differ by rounding, not results."""

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


def fused_ctx(g, prec=64):
    ctx = hf.hf_create(g, 0)
    hf.hf_set_tuning(ctx, "fuse_ab", 1)
    if prec != 64:
        hf.hf_set_precision(ctx, prec)
    return ctx


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_fused_simulate_matches_oracle(name):
    p = synth.c1() if name == "c1" else synth.c3(nsteps=2)
    ctx = fused_ctx(p.grid)
    hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = T(p.u0)
    st = hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=p.rtol)
    o, Fo = oracle.problem_oracle(p)
    uo, _, it, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=p.rtol)
    assert rel(N(u), uo) <= 1e-10
    assert abs(st["total_iters"] - int(it.sum())) <= 2 * p.nsteps + 10


def test_fused_dirichlet_ragged_and_replacement():
    """Dirichlet faces, a ragged grid, more than 50 iterations per solve (residual replacement
    through the IF node after the fused launch)."""
    g = synth.Grid((70, 40, 13), (0.3, 0.2, 0.7), (-1.0, 2.0, 0.5))
    k, c = synth.random_fields(g, seed=95)
    ctx = fused_ctx(g)
    hf.hf_set_coefficients(ctx, T(k), T(c))
    bits = (1 << synth.FACE_XM) | (1 << synth.FACE_ZP)
    vals = [1.0, 0, 0, 0, 0, -0.5]
    hf.hf_set_dirichlet_faces(ctx, bits, vals)
    F = torch.empty(g.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, synth.FACE_ZM, 1.0, None, F)
    u = T(np.zeros(g.n_nodes))
    st = hf.hf_simulate(ctx, 0.5, 0.5, 4, F, u)
    assert st["max_iters_step"] > 50
    o = oracle.Oracle(g, k, c)
    o.set_dirichlet(bits, tuple(vals))
    uo, _, _, _ = o.simulate(0.5, 0.5, 4, o.face_load(synth.FACE_ZM, 1.0), np.zeros(g.n_nodes))
    assert rel(N(u), uo) <= 1e-10


def test_fused_fp32_and_cg():
    p = synth.c1()
    ctx = fused_ctx(p.grid, prec=32)
    hf.hf_set_coefficients(ctx, T(p.k), T(p.c))
    F = torch.empty(p.grid.n_nodes, dtype=torch.float64, device=DEV)
    hf.hf_face_load(ctx, p.flux_face, p.flux_const, None, F)
    u = T(p.u0)
    hf.hf_simulate(ctx, p.theta, p.dt, p.nsteps, F, u, rtol=1e-6)
    o, Fo = oracle.problem_oracle(p)
    uo, _, _, _ = o.simulate(p.theta, p.dt, p.nsteps, Fo, p.u0, tol=1e-12)
    assert rel(N(u), uo) <= 1e-4                  # the fp32 bar of C1 (DESIGN R18)
    # hf_cg on a fused context (graph driver)
    ctx2 = fused_ctx(p.grid)
    hf.hf_set_coefficients(ctx2, T(p.k), T(p.c))
    b = synth.random_vector(p.grid.n_nodes, 96)
    x = T(np.zeros(p.grid.n_nodes))
    hf.hf_cg(ctx2, 0.01, 1.0, T(b), x)
    xo, _, _, _ = o.pcg(0.01, 1.0, b, np.zeros_like(b))
    assert rel(N(x), xo) <= 1e-10
