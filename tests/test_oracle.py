"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage or closed form it pins.  None of them re-types the oracle's
own formula: element matrices are checked against the tensor-product closed form and a
golden fixture, the solver against direct solves and exact discrete solutions, the
time stepper against the bar's closed form and the continuum series.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
import synth
from conftest import read_golden


# ---------------------------------------------------------------------------------------------
# element matrices

def _tensor_q1(h):
    """Independent closed form: K = kx⊗my⊗mz + mx⊗ky⊗mz + mx⊗my⊗kz, M = mx⊗my⊗mz, local
    node l = bx + 2by + 4bz (so the z factor is the outermost Kronecker factor)."""
    def k1(a):
        return np.array([[1.0, -1.0], [-1.0, 1.0]]) / a

    def m1(a):
        return np.array([[2.0, 1.0], [1.0, 2.0]]) * a / 6.0
    hx, hy, hz = h
    K = (np.kron(m1(hz), np.kron(m1(hy), k1(hx))) + np.kron(m1(hz), np.kron(k1(hy), m1(hx)))
         + np.kron(k1(hz), np.kron(m1(hy), m1(hx))))
    M = np.kron(m1(hz), np.kron(m1(hy), m1(hx)))
    return K, M


def test_element_matrices_unit_cube_golden(golden_dir):
    rows = {r[0]: [float(Fraction(v)) for v in r[1:]] for r in read_golden(f"{golden_dir}/q1_unit_cube.txt")}
    Ke, Me = oracle.element_matrices([1.0, 1.0, 1.0])
    np.testing.assert_allclose(Ke[0], rows["K_row0"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(Me[0], rows["M_row0"], rtol=1e-15, atol=0)


@pytest.mark.parametrize("h", [(1.0, 1.0, 1.0), (0.3, 0.2, 0.7), (0.303, 0.303, 0.128), (0.2, 0.2, 0.2)])
def test_element_matrices_tensor_product(h):
    Ke, Me = oracle.element_matrices(h)
    K, M = _tensor_q1(h)
    np.testing.assert_allclose(Ke, K, rtol=0, atol=1e-14 * np.abs(K).max())
    np.testing.assert_allclose(Me, M, rtol=0, atol=1e-14 * np.abs(M).max())
    # invariants: symmetric, K 1 = 0, sum(M) = volume
    assert np.allclose(Ke, Ke.T, atol=0) and np.allclose(Me, Me.T, atol=0)
    assert np.abs(Ke.sum(axis=1)).max() <= 1e-14 * np.abs(Ke).max()
    assert abs(Me.sum() - h[0] * h[1] * h[2]) <= 1e-15


# ---------------------------------------------------------------------------------------------
# assembly

def _small_grids():
    return [synth.Grid((1, 1, 1), (1.0, 1.0, 1.0)), synth.Grid((2, 2, 2), (0.5, 0.5, 0.5)),
            synth.Grid((3, 3, 2), (0.3, 0.2, 0.7)), synth.Grid((5, 4, 3), (0.2, 0.25, 0.1), (-1.0, 2.0, 0.5))]


@pytest.mark.parametrize("gi", range(4))
def test_assembly_invariants(gi):
    g = _small_grids()[gi]
    k, c = synth.random_fields(g, seed=10 + gi)
    o = oracle.Oracle(g, k, c)
    K = o.csr(1.0, 0.0).toarray()
    M = o.csr(0.0, 1.0).toarray()
    assert np.abs(K - K.T).max() <= 1e-13 * np.abs(K).max()
    assert np.abs(M - M.T).max() <= 1e-13 * np.abs(M).max()
    assert np.abs(K.sum(axis=1)).max() <= 1e-12 * np.abs(K).max()          # K 1 = 0
    vol = g.h[0] * g.h[1] * g.h[2]
    assert abs(M.sum() - (c * vol).sum()) <= 1e-12 * (c * vol).sum()      # sum M = sum c_e vol_e
    assert np.linalg.eigvalsh(M).min() > 0                                  # M SPD
    ev = np.linalg.eigvalsh(K)
    assert ev[0] > -1e-10 * ev[-1] and ev[1] > 1e-8 * ev[-1]               # K PSD, nullspace = span(1)
    # 27-point stencil: at most 27 nonzeros per row, exactly 27 at interior rows
    nnz_row = np.diff(o.csr().indptr)
    assert nnz_row.max() <= 27


@pytest.mark.parametrize("gi", range(4))
def test_ebe_equals_assembled(gi):
    """Eq. (1): the EbE sum, the per-DoF sum and the assembled SpMV agree."""
    g = _small_grids()[gi]
    k, c = synth.random_fields(g, seed=20 + gi)
    o = oracle.Oracle(g, k, c)
    u = synth.random_vector(g.n_nodes, seed=30 + gi)
    for aK, aM in [(1.0, 0.0), (0.0, 1.0), (0.005, 1.0), (-0.005, 1.0)]:
        y1 = o.spmv(aK, aM, u)
        y2 = o.apply_ebe(aK, aM, u)
        y3 = o.apply_rows(aK, aM, u, np.arange(g.n_nodes))
        scale = np.abs(y1).max()
        assert np.abs(y1 - y2).max() <= 1e-13 * scale
        assert np.abs(y1 - y3).max() <= 1e-13 * scale


def test_single_element_columns():
    """One element with k=2, c=3: A e_j is column j of 2 aK K + 3 aM M (closed form)."""
    h = (0.3, 0.2, 0.7)
    g = synth.Grid((1, 1, 1), h)
    o = oracle.Oracle(g, [2.0], [3.0])
    K, M = _tensor_q1(h)
    for j in range(8):
        e = np.zeros(8)
        e[j] = 1.0
        y = o.spmv(0.25, 1.5, e)
        np.testing.assert_allclose(y, 2 * 0.25 * K[:, j] + 3 * 1.5 * M[:, j], rtol=0, atol=1e-14)


def test_patch_test_linear_field():
    """Exact reproduction of linear fields (north_star): K u = 0 at interior nodes for u linear."""
    g = synth.Grid((6, 5, 4), (0.3, 0.2, 0.7), (1.0, -2.0, 0.0))
    kval = 7.5
    o = oracle.Oracle(g, np.full(g.n_elems, kval), np.ones(g.n_elems))
    x, y, z = g.node_coords()
    u = (0.3 + 1.7 * x - 2.2 * y + 0.9 * z).ravel()
    r = o.spmv(1.0, 0.0, u).reshape(g.nn[::-1])
    interior = r[1:-1, 1:-1, 1:-1]
    assert np.abs(interior).max() <= 1e-12 * kval * np.abs(u).max()
    # boundary rows carry the flux k du/dn: on the x = max face, sum of rows = k * 1.7 * area(face)
    face = r[:, :, -1].sum()
    area = (g.ne[1] * g.h[1]) * (g.ne[2] * g.h[2])
    assert abs(face - kval * 1.7 * area) <= 1e-10 * abs(kval * 1.7 * area)


# ---------------------------------------------------------------------------------------------
# flux load (reading R12)

def test_face_load_constant():
    g = synth.Grid((4, 3, 2), (0.5, 0.25, 1.0), (-1.0, 0.0, 0.0))
    o = oracle.Oracle(g, np.ones(g.n_elems), np.ones(g.n_elems), assemble=False)
    F = o.face_load(synth.FACE_ZM, 2.0).reshape(g.nn[::-1])
    q = 2.0 * 0.5 * 0.25
    plane = F[0]
    exp = np.full(plane.shape, q)
    exp[0, :] /= 2; exp[-1, :] /= 2; exp[:, 0] /= 2; exp[:, -1] /= 2
    np.testing.assert_allclose(plane, exp, rtol=1e-14)
    assert np.abs(F[1:]).max() == 0.0
    # laminate: sum F = f * 30 * 30 = 900; dt * sum F = 9 at dt = 0.01
    p = synth.laminate(1)
    o2 = oracle.Oracle(p.grid, p.k, p.c, assemble=False)
    F2 = o2.face_load(synth.FACE_ZM, 1.0)
    assert abs(F2.sum() - 900.0) <= 1e-10
    for face in range(6):  # every face: total = f * face area
        Ff = o.face_load(face, 1.0)
        d = face // 2
        dims = [g.ne[a] * g.h[a] for a in range(3) if a != d]
        assert abs(Ff.sum() - dims[0] * dims[1]) <= 1e-13


def test_face_load_beam_total():
    """Gaussian beam: sum F -> P * fraction of the beam on the face (erf closed form)."""
    g = synth.c5_grid(60)
    o = oracle.Oracle(g, np.ones(g.n_elems), np.ones(g.n_elems), assemble=False)
    P, s, cx, cy = 10.0, 2.0, 1.0, -0.5
    F = o.face_load(synth.FACE_ZM, 0.0, (P, s, cx, cy))

    def frac(a, b, c0):
        return 0.5 * (math.erf((b - c0) / (s * math.sqrt(2))) - math.erf((a - c0) / (s * math.sqrt(2))))
    exact = P * frac(-15, 15, cx) * frac(-15, 15, cy)
    assert abs(F.sum() - exact) <= 1e-4 * exact
    assert abs(F.sum() - exact) > 0  # quadrature, not the closed form


def test_face_load_beam_axes_on_a_rectangular_face():
    """The beam's in-plane axes (R12): on a rectangular face with the beam off centre and cut by
    one edge, the total is P times the product of the two truncated-normal masses and the load's
    centroid is the truncated-normal mean along each axis (closed forms); swapping the face axes
    changes both."""
    g = synth.Grid((40, 24, 4), (0.5, 0.5, 0.5), (-10.0, -6.0, 0.0))
    o = oracle.Oracle(g, np.ones(g.n_elems), np.ones(g.n_elems), assemble=False)
    P, s, cx, cy = 10.0, 1.5, 4.0, -2.5
    F = o.face_load(synth.FACE_ZM, 0.0, (P, s, cx, cy))
    r2 = math.sqrt(2.0)

    def mass(a, b, c0):
        return 0.5 * (math.erf((b - c0) / (s * r2)) - math.erf((a - c0) / (s * r2)))

    def mean(a, b, c0):
        phi = lambda t: math.exp(-0.5 * t * t) / math.sqrt(2 * math.pi)
        al, be = (a - c0) / s, (b - c0) / s
        return c0 + s * (phi(al) - phi(be)) / mass(a, b, c0)

    exact = P * mass(-10, 10, cx) * mass(-6, 6, cy)
    swapped = P * mass(-10, 10, cy) * mass(-6, 6, cx)
    assert abs(F.sum() - exact) <= 2e-4 * exact
    assert abs(swapped - exact) > 1e-2 * exact
    x, y, _ = g.node_coords()
    Fz = F.reshape(g.ne[2] + 1, g.ne[1] + 1, g.ne[0] + 1)[0]
    X, Y = x[0], y[0]
    # the nodal load's first moments equal the continuous ones for the bilinear face basis up to
    # quadrature error (sum_i phi_i(x) x_i = x on a Q1 face)
    mx = float((Fz * X).sum() / Fz.sum())
    my = float((Fz * Y).sum() / Fz.sum())
    assert abs(mx - mean(-10, 10, cx)) < 5e-3, (mx, mean(-10, 10, cx))
    assert abs(my - mean(-6, 6, cy)) < 5e-3, (my, mean(-6, 6, cy))
    assert np.count_nonzero(F.reshape(g.ne[2] + 1, -1)[1:]) == 0   # all load on the z = 0 face


# ---------------------------------------------------------------------------------------------
# PCG (Alg. 1)

def test_pcg_matches_direct_solve():
    p = synth.c1()
    o, F = oracle.problem_oracle(p)
    A = o.csr(p.dt * p.theta, 1.0).tocsc()
    b = synth.random_vector(p.grid.n_nodes, 3) * 1e6
    x, st, it, rel = o.pcg(p.dt * p.theta, 1.0, b, np.zeros_like(b), tol=1e-13)
    assert st == 0 and rel <= 1e-13
    xd = spla.spsolve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-10 * np.linalg.norm(xd)


def test_pcg_zero_rhs_and_finite_termination():
    g = synth.Grid((1, 1, 1), (1.0, 1.0, 1.0))
    o = oracle.Oracle(g, [2.0], [3.0])
    x, st, it, _ = o.pcg(0.5, 1.0, np.zeros(8), np.ones(8))
    assert st == 0 and it == 0 and np.all(x == 0)
    # Dirichlet on the -x face leaves 4 free DoFs -> exact in <= 4 iterations (Krylov)
    o.set_dirichlet(1 << synth.FACE_XM, (1.5, 0, 0, 0, 0, 0))
    b = np.arange(8, dtype=float)
    bl = o.rhs(1.0, 0.1, b * 0, b)  # any consistent lifted rhs
    x, st, it, rel = o.pcg(0.1, 1.0, bl, np.zeros(8), tol=1e-14)
    assert st == 0 and it <= 4


def test_pcg_dirichlet_matches_eliminated_direct():
    p = synth.c2()
    o, F = oracle.problem_oracle(p)
    o.set_dirichlet(p.dirichlet_bits, (0.7, -0.3, 0, 0, 0, 0))
    D = o.dirichlet_mask()
    b = o.rhs(p.theta, p.dt, F, np.cos(3 * np.arange(p.grid.n_nodes)))
    A = o.csr(p.theta * p.dt, 1.0).tocsr()
    free = ~D
    g = np.where(D, b, 0.0)
    # independent elimination: A_FF x_F = b_F (b already lifted by or_rhs) ; x_D = g_D
    xF = spla.spsolve(A[free][:, free].tocsc(), b[free])
    x, st, it, _ = o.pcg(p.theta * p.dt, 1.0, b, np.zeros_like(b))
    assert st == 0
    assert np.allclose(x[D], g[D], rtol=0, atol=0)
    assert np.linalg.norm(x[free] - xF) <= 1e-10 * np.linalg.norm(xF)
    # and the lift itself: b_F = (L u)_F - (A g~)_F
    un = np.cos(3 * np.arange(p.grid.n_nodes))
    L = o.csr(-(1 - p.theta) * p.dt, 1.0)
    bF = (L @ un + p.dt * F - A @ g)[free]
    assert np.abs(b[free] - bF).max() <= 1e-13 * np.abs(bF).max()


# ---------------------------------------------------------------------------------------------
# time stepper

def _bar_closed_form(p, modes):
    """Exact discrete solution on a uniform Q1 bar with insulated sides and Dirichlet-0 ends:
    sin(m pi x) is an eigenvector of K, M (K_y 1 = K_z 1 = 0), eigenvalue ratio
    lam_m = (6/h^2)(1 - cos(m pi h)) / (2 + cos(m pi h)); amplification per step
    G_m = (1 - (1-theta) dt lam_m) / (1 + theta dt lam_m)  (theta-scheme)."""
    g = p.grid
    h = g.h[0]
    x, _, _ = g.node_coords()
    x = x.ravel()
    u = np.zeros_like(x)
    for m, a in modes:
        lam = (6.0 / h ** 2) * (1.0 - np.cos(m * np.pi * h)) / (2.0 + np.cos(m * np.pi * h))
        G = (1.0 - (1.0 - p.theta) * p.dt * lam) / (1.0 + p.theta * p.dt * lam)
        u += a * G ** p.nsteps * np.sin(m * np.pi * x)
    u[np.isclose(x, 0.0) | np.isclose(x, 1.0)] = 0.0
    return u


def test_bar_discrete_closed_form_cn():
    p = synth.c2()
    o, F = oracle.problem_oracle(p)
    u, st, it, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0)
    assert st == 0
    ex = _bar_closed_form(p, [(1, 1.0)])
    assert np.linalg.norm(u - ex) <= 1e-10 * np.linalg.norm(ex)


def test_bar_closed_form_through_resume_segments():
    """Checkpoint / resume (R9 guess 2u^n - u^{n-1} across the seam): 200 CN steps as 70 + 130
    meet the same exact discrete solution, and the segments chain to the one-run trajectory."""
    p = synth.c2()
    o, F = oracle.problem_oracle(p)
    u1, up1, st1, it1, _ = o.simulate_resume(p.theta, p.dt, 70, F, p.u0, None, 0)
    u2, up2, st2, it2, _ = o.simulate_resume(p.theta, p.dt, 130, F, u1, up1, 70)
    assert st1 == 0 and st2 == 0
    ex = _bar_closed_form(p, [(1, 1.0)])
    assert np.linalg.norm(u2 - ex) <= 1e-10 * np.linalg.norm(ex)
    u, st, it, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0)
    assert np.array_equal(u, u2) and np.array_equal(it, np.concatenate([it1, it2]))
    # u_prev out is the iterate one step before the end
    u3, up3, _, _, _ = o.simulate_resume(p.theta, p.dt, 199, F, p.u0, None, 0)
    assert np.array_equal(up2, u3)


@pytest.mark.parametrize("theta", [1.0, 0.5, 0.0 + 0.6])
def test_bar_sine_series_any_theta(theta):
    """1D analytic series (north_star): u0 = sin(pi x) + 0.5 sin(3 pi x) decays mode by mode."""
    p = synth.c2()
    p.theta = theta
    p.nsteps = 40
    x, _, _ = p.grid.node_coords()
    p.u0 = (np.sin(np.pi * x) + 0.5 * np.sin(3 * np.pi * x)).ravel()
    o, F = oracle.problem_oracle(p)
    u, st, it, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0)
    ex = _bar_closed_form(p, [(1, 1.0), (3, 0.5)])
    assert st == 0
    assert np.linalg.norm(u - ex) <= 1e-10 * np.linalg.norm(ex)


def test_bar_continuum_and_second_order():
    """Against the PDE solution exp(-pi^2 t) sin(pi x): error ~ (pi h)^2/12-sized at h=1/64, and
    halving h and dt divides it by ~4 (CN second order in both)."""
    errs = []
    for n, dt in [(32, 1e-3), (64, 5e-4)]:
        h = 1.0 / n
        g = synth.Grid((n, 2, 2), (h, h, h))
        x, _, _ = g.node_coords()
        ones = np.ones(g.n_elems)
        p = synth.Problem("bar", g, ones, ones.copy(), np.sin(np.pi * x).ravel(), 0.5, dt, int(round(0.1 / dt)),
                          dirichlet_bits=3)
        o, F = oracle.problem_oracle(p)
        u, st, it, _ = o.simulate(p.theta, p.dt, p.nsteps, F, p.u0)
        ex = np.exp(-np.pi ** 2 * 0.1) * np.sin(np.pi * x.ravel())
        errs.append(np.linalg.norm(u - ex) / np.linalg.norm(ex))
    assert 1.0e-4 < errs[1] < 4.0e-4
    assert 3.6 < errs[0] / errs[1] < 4.4


def test_heat_content_balance():
    """1^T M (u^N - u^0) = N dt 1^T F under insulated sides (1^T K = 0)."""
    g = synth.Grid((10, 9, 8), (0.3, 0.3, 0.3))
    ids = synth.inclusion_ids(g, seed=4)
    k, c = synth.ids_to_fields(ids)
    o = oracle.Oracle(g, k, c)
    F = o.face_load(synth.FACE_ZM, 1.0)
    u0 = np.zeros(g.n_nodes)
    N, dt = 12, 0.01
    u, st, it, _ = o.simulate(0.5, dt, N, F, u0, tol=1e-13)
    M = o.csr(0.0, 1.0)
    lhs = (M @ u).sum() - (M @ u0).sum()
    rhs = N * dt * F.sum()
    assert st == 0 and abs(lhs - rhs) <= 1e-9 * abs(rhs)
    # insulated, no load: heat content constant and a constant field is a fixed point
    u2, st, _, _ = o.simulate(0.5, dt, 20, np.zeros_like(F), np.full(g.n_nodes, 3.25))
    assert np.abs(u2 - 3.25).max() <= 1e-10


def test_cn_time_self_convergence():
    """CN order >= 1.9 by self-convergence in dt."""
    g = synth.Grid((6, 6, 6), (0.3, 0.3, 0.3))
    k, c = synth.random_fields(g, seed=7)
    o = oracle.Oracle(g, k, c)
    F = o.face_load(synth.FACE_ZM, 1.0)
    T = 0.4
    sols = []
    for n in [8, 16, 128]:
        u, st, _, _ = o.simulate(0.5, T / n, n, F, np.zeros(g.n_nodes), tol=1e-14)
        sols.append(u)
    e1 = np.linalg.norm(sols[0] - sols[2])
    e2 = np.linalg.norm(sols[1] - sols[2])
    assert np.log2(e1 / e2) >= 1.9


def test_table2_grid_sizes(golden_dir):
    """Node counts of the laminate grids equal the DoF the paper prints, to the
    printed precision (3 significant digits; the 10.5e3 entry is 10,571 truncated)."""
    for s, printed in read_golden(f"{golden_dir}/table2_dofs.txt"):
        n = synth.laminate(int(s)).grid.n_nodes
        assert abs(n - float(printed)) <= 0.01 * float(printed), (s, n, printed)


def test_paper_materials(golden_dir):
    rows = {r[0]: (float(r[1]), float(r[2])) for r in read_golden(f"{golden_dir}/materials.txt")}
    assert synth.STEEL == rows["steel"] and synth.OXIDE == rows["oxide"]


# ---------------------------------------------------------------------------------------------
# the paper's element (NEXT row f1): 6 Kuhn P1 tetrahedra per voxel

def test_tet_voxel_unit_cube_closed_form():
    """Row 0 of the voxel matrix of the 6-tet split of the unit cube: node 0 lies in all 6 tets
    (diagonal 1), couples to its 3 edge neighbours with -1/3 and to nothing else in K."""
    K, M = oracle.tet_voxel_matrices([1.0, 1.0, 1.0])
    np.testing.assert_allclose(K[0], [1, -1 / 3, -1 / 3, 0, -1 / 3, 0, 0, 0], atol=1e-15)
    np.testing.assert_allclose(K[7], [0, 0, 0, -1 / 3, 0, -1 / 3, -1 / 3, 1], atol=1e-15)
    assert abs(M.sum() - 1.0) < 1e-15                          # six tets of volume 1/6
    assert np.allclose(K, K.T) and np.abs(K.sum(1)).max() < 1e-15


def test_tet_assembly_is_the_seven_point_laplacian():
    """Classical result: P1 elements on the Kuhn (Freudenthal) triangulation of a cubic grid give
    the 7-point finite-difference Laplacian times h (all diagonal-edge couplings cancel), while the
    mass matrix keeps the 15-point pattern with interior row sums h^3."""
    h = 0.5
    g = synth.Grid((5, 5, 5), (h, h, h))
    o = oracle.Oracle(g, np.ones(g.n_elems), np.ones(g.n_elems), elem=1)
    K = o.csr(1.0, 0.0).toarray()
    M = o.csr(0.0, 1.0).toarray()
    n = g.nn[0]
    i = 2 + n * (2 + n * 2)
    nz = np.flatnonzero(np.abs(K[i]) > 1e-14)
    expect = sorted([i, i - 1, i + 1, i - n, i + n, i - n * n, i + n * n])
    assert list(nz) == expect
    assert abs(K[i, i] - 6 * h) < 1e-14 and np.allclose(K[i, [i - 1, i + 1, i - n, i + n, i - n * n, i + n * n]], -h)
    assert np.count_nonzero(np.abs(M[i]) > 1e-16) == 15
    assert abs(M[i].sum() - h ** 3) < 1e-15


def test_tet_patch_test_and_invariants():
    g = synth.Grid((4, 5, 3), (0.3, 0.2, 0.7), (1.0, -2.0, 0.0))
    k, c = synth.random_fields(g, seed=31)
    o = oracle.Oracle(g, k, c, elem=1)
    K = o.csr(1.0, 0.0).toarray()
    M = o.csr(0.0, 1.0).toarray()
    assert np.abs(K - K.T).max() <= 1e-13 * np.abs(K).max()
    assert np.abs(K.sum(axis=1)).max() <= 1e-12 * np.abs(K).max()
    vol = g.h[0] * g.h[1] * g.h[2]
    assert abs(M.sum() - (c * vol).sum()) <= 1e-12 * (c * vol).sum()
    assert np.linalg.eigvalsh(M).min() > 0
    # linear fields are reproduced exactly by P1 (constant k): interior rows vanish
    o1 = oracle.Oracle(g, np.full(g.n_elems, 3.0), np.ones(g.n_elems), elem=1)
    x, y, z = g.node_coords()
    u = (0.4 - 1.3 * x + 2.1 * y + 0.7 * z).ravel()
    r = o1.spmv(1.0, 0.0, u).reshape(g.nn[::-1])
    assert np.abs(r[1:-1, 1:-1, 1:-1]).max() <= 1e-12 * 3.0 * np.abs(u).max()
    # EbE = assembled = per-row for the tet voxel matrices too
    uu = synth.random_vector(g.n_nodes, 32)
    y1 = o.spmv(0.01, 1.0, uu)
    assert np.abs(o.apply_ebe(0.01, 1.0, uu) - y1).max() <= 1e-13 * np.abs(y1).max()
    assert np.abs(o.apply_rows(0.01, 1.0, uu, np.arange(g.n_nodes)) - y1).max() <= 1e-13 * np.abs(y1).max()


def test_tet_face_load():
    g = synth.Grid((4, 3, 2), (0.5, 0.25, 1.0), (-1.0, 0.0, 0.0))
    o = oracle.Oracle(g, np.ones(g.n_elems), np.ones(g.n_elems), assemble=False, elem=1)
    F = o.face_load(synth.FACE_ZM, 2.0).reshape(g.nn[::-1])[0]
    A = 0.5 * 0.25
    # interior node: 6 triangles touch it (2 quads on the diagonal side x 2 + 2 singles): f A
    assert abs(F[1, 1] - 2.0 * A) < 1e-15
    # corner (0,0) lies on its quad's diagonal (2 triangles): f A / 3; corner (nx,0): 1 tri: f A/6
    assert abs(F[0, 0] - 2.0 * A / 3) < 1e-15 and abs(F[0, -1] - 2.0 * A / 6) < 1e-15
    for face in range(6):
        Ff = o.face_load(face, 1.0)
        d = face // 2
        dims = [g.ne[a] * g.h[a] for a in range(3) if a != d]
        assert abs(Ff.sum() - dims[0] * dims[1]) <= 1e-13
    gb = synth.c5_grid(60)
    ob = oracle.Oracle(gb, np.ones(gb.n_elems), np.ones(gb.n_elems), assemble=False, elem=1)
    P, s = 10.0, 2.0
    tot = ob.face_load(synth.FACE_ZM, 0.0, (P, s, 0.0, 0.0)).sum()
    ex = P * math.erf(15 / (s * math.sqrt(2))) ** 2
    assert abs(tot - ex) <= 1e-3 * ex


def test_tet_time_stepper_matches_direct():
    g = synth.Grid((6, 5, 4), (0.3, 0.3, 0.3))
    k, c = synth.random_fields(g, seed=33)
    o = oracle.Oracle(g, k, c, elem=1)
    F = o.face_load(synth.FACE_ZM, 1.0)
    u, st, it, _ = o.simulate(0.5, 0.05, 1, F, np.zeros(g.n_nodes), tol=1e-13)
    A = o.csr(0.025, 1.0).tocsc()
    xd = spla.spsolve(A, o.rhs(0.5, 0.05, F, np.zeros(g.n_nodes)))
    assert st == 0 and np.linalg.norm(u - xd) <= 1e-10 * np.linalg.norm(xd)


# ---------------------------------------------------------------------------------------------
# Vertex materials averaged over each element ("computed ... at each vertex and the values
# averaged over each element"): Q1 voxels average 8 corners, tets average their 4 vertices.

def _brute_tet_vertex_assembly(g, kn, cn):
    """Dense K, M of the Kuhn 6-tet mesh with per-tet coefficients = mean of the tet's 4 vertex
    values, built here from scratch (numpy: edge matrix inverse for the P1 gradients)."""
    import itertools
    nx, ny, nz = g.ne
    nx1, ny1 = nx + 1, ny + 1
    N = g.n_nodes
    K = np.zeros((N, N))
    M = np.zeros((N, N))
    h = np.asarray(g.h)
    for ez, ey, ex in itertools.product(range(nz), range(ny), range(nx)):
        for perm in itertools.permutations(range(3)):
            b = np.zeros(3, dtype=int)
            verts = [b.copy()]
            for ax in perm:
                b[ax] = 1
                verts.append(b.copy())
            idx = [(ex + v[0]) + nx1 * ((ey + v[1]) + ny1 * (ez + v[2])) for v in verts]
            P = np.array([v * h for v in verts], dtype=float)
            E = (P[1:] - P[0]).T                        # columns p_i - p_0
            Ginv = np.linalg.inv(E)                     # rows: grad lambda_1..3
            grads = np.vstack([-Ginv.sum(axis=0), Ginv])
            vol = abs(np.linalg.det(E)) / 6.0
            kt = np.mean(kn[idx])
            ct = np.mean(cn[idx])
            Kt = vol * grads @ grads.T
            Mt = vol * (np.ones((4, 4)) + np.eye(4)) / 20.0
            for a in range(4):
                for bb in range(4):
                    K[idx[a], idx[bb]] += kt * Kt[a, bb]
                    M[idx[a], idx[bb]] += ct * Mt[a, bb]
    return K, M


def test_vertex_materials_tets_match_brute_force():
    g = synth.Grid((3, 2, 2), (0.5, 0.4, 0.3), (1.0, -1.0, 0.0))
    rng = np.random.default_rng(5)
    kn = rng.uniform(1.0, 100.0, g.n_nodes)
    cn = rng.uniform(0.5, 2.0, g.n_nodes)
    o = oracle.Oracle(g, kn, cn, elem=1, vertex=True)
    K, M = _brute_tet_vertex_assembly(g, kn, cn)
    assert np.allclose(o.csr(1.0, 0.0).toarray(), K, rtol=0, atol=1e-12 * np.abs(K).max())
    assert np.allclose(o.csr(0.0, 1.0).toarray(), M, rtol=0, atol=1e-14 * np.abs(M).max())
    u = rng.standard_normal(g.n_nodes)
    assert np.allclose(o.apply_ebe(0.3, 1.2, u), (0.3 * K + 1.2 * M) @ u, atol=1e-11)
    rows = np.array([0, 5, 17, g.n_nodes - 1])
    assert np.allclose(o.apply_rows(0.3, 1.2, u, rows), ((0.3 * K + 1.2 * M) @ u)[rows], atol=1e-11)


def test_vertex_materials_constant_field_and_q1_corner_mean():
    g = synth.Grid((4, 3, 2), (0.3, 0.3, 0.2))
    ones = np.ones(g.n_nodes)
    # constant vertex fields: per-tet coefficients all equal -> the per-voxel tet operator
    o1 = oracle.Oracle(g, 7.0 * ones, 2.0 * ones, elem=1, vertex=True)
    o2 = oracle.Oracle(g, np.full(g.n_elems, 7.0), np.full(g.n_elems, 2.0), elem=1)
    assert np.allclose(o1.csr(1.0, 1.0).toarray(), o2.csr(1.0, 1.0).toarray(), rtol=1e-14, atol=0)
    # Q1: each voxel's coefficient is the mean of its 8 corners (computed here by slicing)
    rng = np.random.default_rng(6)
    kn = rng.uniform(1.0, 5.0, g.n_nodes)
    cn = rng.uniform(1.0, 5.0, g.n_nodes)
    nx, ny, nz = g.ne
    kv = kn.reshape(nz + 1, ny + 1, nx + 1)
    cv = cn.reshape(nz + 1, ny + 1, nx + 1)
    corner = lambda a: sum(a[dz:dz + nz, dy:dy + ny, dx:dx + nx] for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)) / 8
    oq = oracle.Oracle(g, kn, cn, elem=0, vertex=True)
    oe = oracle.Oracle(g, corner(kv).ravel(), corner(cv).ravel(), elem=0)
    assert np.allclose(oq.csr(0.4, 1.0).toarray(), oe.csr(0.4, 1.0).toarray(), rtol=1e-14, atol=0)
    # tets: the face load does not depend on the coefficients
    assert np.array_equal(o1.face_load(synth.FACE_ZM, 1.0), o2.face_load(synth.FACE_ZM, 1.0))
