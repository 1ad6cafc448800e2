"""The paper's CPU comparison method (NEXT f4; §5.3: sparse PCG with an incomplete
Cholesky preconditioner of drop tolerance 1e-3, single core), pinned against what the
mathematics fixes: droptol 0 is the exact Cholesky factor (numpy), a huge droptol leaves the
diagonal only (Jacobi-PCG, the oracle's Algorithm 1), and the preconditioned solves land on the
sparse direct solution and the oracle's transient."""
import numpy as np
import pytest

import comparator
import oracle
import synth

sp = pytest.importorskip("scipy.sparse")
spla = pytest.importorskip("scipy.sparse.linalg")


def _system(grid, seed, aK=0.01, aM=1.0, elem=0):
    k, c = synth.random_fields(grid, seed=seed)
    o = oracle.Oracle(grid, k, c, elem=elem)
    return o, o.csr(aK, aM)


@pytest.mark.parametrize("elem", [0, 1])
def test_droptol_zero_is_exact_cholesky(elem):
    g = synth.Grid((3, 3, 2), (0.3, 0.2, 0.7))
    o, A = _system(g, 71, aK=1.0, aM=0.5, elem=elem)
    f = comparator.ICFactor(A, droptol=0.0)
    Ld = f.dense()
    Ad = A.toarray()
    assert np.allclose(np.tril(Ld), Ld)
    assert np.abs(Ld @ Ld.T - Ad).max() <= 1e-13 * np.abs(Ad).max()
    assert np.abs(Ld - np.linalg.cholesky(Ad)).max() <= 1e-12 * np.abs(Ld).max()
    b = synth.random_vector(g.n_nodes, 72)
    x, it, rc = f.pcg(b, np.zeros_like(b), tol=1e-12)
    assert rc == comparator.IC_OK and it <= 1
    assert np.linalg.norm(Ad @ x - b) <= 1e-12 * np.linalg.norm(b)


def test_huge_droptol_is_jacobi_pcg():
    """Every off-diagonal dropped: L = diag(sqrt(a_ii)), so the method is Algorithm 1's Jacobi
    PCG (without residual replacement): the iterates match the oracle's."""
    g = synth.c1().grid
    o, A = _system(g, 73)
    f = comparator.ICFactor(A, droptol=1e30)
    assert f.nnz == g.n_nodes
    assert np.allclose(np.diag(f.dense()) ** 2, A.diagonal(), rtol=1e-15)
    b = synth.random_vector(g.n_nodes, 74)
    x, it, rc = f.pcg(b, np.zeros_like(b), tol=1e-10)
    xo, st, ito, _ = o.pcg(0.01, 1.0, b, np.zeros_like(b), tol=1e-10, replace_every=0)
    assert rc == 0 and st == 0 and abs(it - ito) <= 1
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)


def test_ic_pcg_matches_direct_solve_and_cuts_iterations():
    g = synth.Grid((12, 10, 9), (0.2, 0.2, 0.2))
    o, A = _system(g, 75, aK=0.05, aM=1.0)
    f = comparator.ICFactor(A, droptol=1e-3)
    assert g.n_nodes < f.nnz < sp.tril(A).nnz * 4
    b = synth.random_vector(g.n_nodes, 76)
    x, it, rc = f.pcg(b, np.zeros_like(b), tol=1e-13)
    xd = spla.spsolve(A.tocsc(), b)
    assert rc == 0
    assert np.linalg.norm(x - xd) <= 1e-10 * np.linalg.norm(xd)
    _, _, it_jac, _ = o.pcg(0.05, 1.0, b, np.zeros_like(b), tol=1e-13)
    assert it < it_jac / 2


def test_ic_transient_matches_oracle():
    p = synth.c1()
    o, F = oracle.problem_oracle(p)
    A = o.csr(p.theta * p.dt, 1.0)
    Lop = o.csr(-(1 - p.theta) * p.dt, 1.0)
    f = comparator.ICFactor(A, droptol=1e-3)
    u, iters, rc = f.simulate(Lop, F, p.dt, p.nsteps, p.u0, tol=p.rtol)
    uo, st, ito, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0, tol=p.rtol)
    assert rc == 0 and st == 0
    assert np.linalg.norm(u - uo) <= 1e-10 * np.linalg.norm(uo)
    assert iters.sum() < ito.sum()
