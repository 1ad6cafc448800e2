"""ctypes wrapper of the plain C oracle (oracle/heat_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  The product
package ``paper_1905_07622_b200`` never imports it (tests/test_abi.py::test_product_never_uses_oracle
checks).

Every function follows the passage of PAPER.md cited in heat_oracle.c.  This file
only marshals numpy arrays; all arithmetic is in the C file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "heat_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_E_ARG, OR_E_NOCONV, OR_E_BREAKDOWN, OR_E_OOM = 0, -1, -3, -4, -8


def build(force: bool = False) -> str:
    """Compile heat_oracle.c into oracle/liboracle.so (plain -O2, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-D_GNU_SOURCE", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.or_create.restype = C.c_void_p
        L.or_create.argtypes = [_i64p, _dp, _dp, _dp, _dp, C.c_int, C.c_int]
        L.or_tet_voxel_matrices.argtypes = [_dp, _dp, _dp]
        L.or_create_vertex.restype = C.c_void_p
        L.or_create_vertex.argtypes = [_i64p, _dp, _dp, _dp, _dp, C.c_int, C.c_int]
        L.or_destroy.argtypes = [C.c_void_p]
        L.or_element_matrices.argtypes = [_dp, _dp, _dp]
        L.or_get_element_matrices.argtypes = [C.c_void_p, _dp, _dp]
        L.or_nnz.restype = C.c_int64
        L.or_nnz.argtypes = [C.c_void_p]
        L.or_csr_copy.argtypes = [C.c_void_p, _i64p, _i64p, _dp, _dp]
        L.or_spmv.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp, _dp]
        L.or_apply_ebe.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp, _dp]
        L.or_apply_rows.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp, _i64p, C.c_int64, _dp]
        L.or_face_load.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_void_p, _dp]
        L.or_set_dirichlet.argtypes = [C.c_void_p, C.c_uint, _dp]
        L.or_is_dirichlet.argtypes = [C.c_void_p, _u8p]
        L.or_diag.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp]
        L.or_pcg.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp, _dp, C.c_double, C.c_int,
                             C.c_int, _dp]
        L.or_rhs.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp, _dp, _dp]
        L.or_simulate_resume.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, _dp, _dp, C.c_void_p,
                                         C.c_int64, C.c_double, C.c_int, C.c_int, _i32p, C.c_int64, C.c_void_p]
        L.or_num_threads.restype = C.c_int
        L.or_num_threads.argtypes = []
        L.or_simulate.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, _dp, _dp, C.c_double,
                                  C.c_int, C.c_int, _i32p, C.c_int64, C.c_void_p]
        _lib = L
    return _lib


def num_threads() -> int:
    """OpenMP threads the oracle runs on (OMP_NUM_THREADS, default all host cores)."""
    return int(lib().or_num_threads())


def element_matrices(h: Sequence[float]):
    """(K_e, M_e) 8x8 for an hx x hy x hz voxel by 2x2x2 Gauss quadrature."""
    Ke = np.zeros(64)
    Me = np.zeros(64)
    lib().or_element_matrices(np.asarray(h, dtype=np.float64), Ke, Me)
    return Ke.reshape(8, 8), Me.reshape(8, 8)


def tet_voxel_matrices(h: Sequence[float]):
    """(K, M) 8x8 of a voxel split into 6 Kuhn P1 tetrahedra (NEXT row f1)."""
    Ke = np.zeros(64)
    Me = np.zeros(64)
    lib().or_tet_voxel_matrices(np.asarray(h, dtype=np.float64), Ke, Me)
    return Ke.reshape(8, 8), Me.reshape(8, 8)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """Assembled-matrix reference for one grid and one (k, c) field."""

    def __init__(self, grid, k, c, assemble: bool = True, elem: int = 0, vertex: bool = False):
        """k, c per element; vertex=True: k, c per node, averaged over each element's vertices
        (Q1: the voxel's 8 corners; elem=1: each tet's 4 vertices)."""
        self.grid = grid
        self.nn = grid.n_nodes
        self._k = _f64(k)
        self._c = _f64(c)
        n = grid.n_nodes if vertex else grid.n_elems
        assert self._k.size == n and self._c.size == n
        create = lib().or_create_vertex if vertex else lib().or_create
        self._p = create(np.asarray(grid.ne, dtype=np.int64), _f64(grid.h), _f64(grid.origin),
                         self._k, self._c, 1 if assemble else 0, elem)
        self.elem = elem
        if not self._p:
            raise MemoryError("or_create failed")

    def __del__(self):
        if getattr(self, "_p", None):
            lib().or_destroy(self._p)
            self._p = None

    # -- operators -----------------------------------------------------------------------------
    def spmv(self, aK, aM, u):
        y = np.empty(self.nn)
        assert lib().or_spmv(self._p, aK, aM, _f64(u), y) == OR_OK
        return y

    def apply_ebe(self, aK, aM, u):
        y = np.empty(self.nn)
        lib().or_apply_ebe(self._p, aK, aM, _f64(u), y)
        return y

    def apply_rows(self, aK, aM, u, rows):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty(rows.size)
        lib().or_apply_rows(self._p, aK, aM, _f64(u), rows, rows.size, out)
        return out

    def csr(self, aK=1.0, aM=0.0):
        """scipy CSR of aK K + aM M."""
        import scipy.sparse as sp
        nnz = lib().or_nnz(self._p)
        rp = np.empty(self.nn + 1, dtype=np.int64)
        col = np.empty(nnz, dtype=np.int64)
        Kv = np.empty(nnz)
        Mv = np.empty(nnz)
        assert lib().or_csr_copy(self._p, rp, col, Kv, Mv) == OR_OK
        return sp.csr_matrix((aK * Kv + aM * Mv, col, rp), shape=(self.nn, self.nn))

    def face_load(self, face: int, f_const: float = 0.0, beam=None):
        F = np.empty(self.nn)
        bp = None
        if beam is not None:
            barr = _f64(beam)
            bp = barr.ctypes.data_as(C.c_void_p)
        assert lib().or_face_load(self._p, face, f_const, bp, F) == OR_OK
        return F

    def set_dirichlet(self, bits: int, values=(0.0,) * 6):
        lib().or_set_dirichlet(self._p, bits, _f64(values))

    def dirichlet_mask(self):
        m = np.empty(self.nn, dtype=np.uint8)
        lib().or_is_dirichlet(self._p, m)
        return m.astype(bool)

    def diag(self, aK, aM):
        d = np.empty(self.nn)
        assert lib().or_diag(self._p, aK, aM, d) == OR_OK
        return d

    def pcg(self, aK, aM, b, x0, tol=1e-12, max_iter=10000, replace_every=50):
        x = _f64(x0).copy()
        info = np.zeros(3)
        st = lib().or_pcg(self._p, aK, aM, _f64(b), x, tol, max_iter, replace_every, info)
        return x, st, int(info[0]), float(info[1])

    def rhs(self, theta, dt, F, un):
        b = np.empty(self.nn)
        lib().or_rhs(self._p, theta, dt, _f64(F), _f64(un), b)
        return b

    def simulate(self, theta, dt, nsteps, F, u0, tol=1e-12, max_iter=10000, replace_every=50,
                 snap_plane: Optional[int] = None):
        u = _f64(u0).copy()
        iters = np.zeros(max(nsteps, 1), dtype=np.int32)
        snap = None
        sp_arg = None
        if snap_plane is not None:
            plane = (self.grid.ne[0] + 1) * (self.grid.ne[1] + 1)
            snap = np.zeros((max(nsteps, 1), plane))
            sp_arg = snap.ctypes.data_as(C.c_void_p)
        st = lib().or_simulate(self._p, theta, dt, nsteps, _f64(F), u, tol, max_iter, replace_every,
                               iters, -1 if snap_plane is None else snap_plane, sp_arg)
        return u, st, iters[:nsteps], snap


    def simulate_resume(self, theta, dt, nsteps, F, u, u_prev, step0, tol=1e-12, max_iter=10000,
                        replace_every=50, snap_plane: Optional[int] = None):
        """Checkpoint / resume of the time loop: the guess of the first step is 2 u - u_prev when
        step0 > 0 (R9).  Returns (u^{n+nsteps}, u^{n+nsteps-1}, status, iters, snap)."""
        u = _f64(u).copy()
        up = _f64(u_prev if u_prev is not None else u).copy()
        iters = np.zeros(max(nsteps, 1), dtype=np.int32)
        snap = None
        sp_arg = None
        if snap_plane is not None:
            plane = (self.grid.ne[0] + 1) * (self.grid.ne[1] + 1)
            snap = np.zeros((max(nsteps, 1), plane))
            sp_arg = snap.ctypes.data_as(C.c_void_p)
        st = lib().or_simulate_resume(self._p, theta, dt, nsteps, _f64(F), u, up.ctypes.data_as(C.c_void_p),
                                      step0 if u_prev is not None else 0, tol, max_iter, replace_every, iters,
                                      -1 if snap_plane is None else snap_plane, sp_arg)
        return u, up, st, iters[:nsteps], snap


def problem_oracle(p, assemble=True, elem=0):
    """Oracle for a synth.Problem with its Dirichlet faces and flux load applied."""
    o = Oracle(p.grid, p.k, p.c, assemble=assemble, elem=elem)
    if p.dirichlet_bits:
        o.set_dirichlet(p.dirichlet_bits, p.dirichlet_values)
    F = o.face_load(p.flux_face, p.flux_const, p.beam)
    return o, F
