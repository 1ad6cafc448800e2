"""ctypes wrapper of comparator/ic_pcg.c: the paper's CPU comparison method (sparse PCG with an
incomplete Cholesky preconditioner, drop tolerance 1e-3; §5.3, Table 3), one core.

A comparison program run by tools/ic_comparator.py and tests/ only; the product package never
imports it.  All arithmetic is in the C file; this module marshals arrays."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ic_pcg.c")
_LIB = os.path.join(_HERE, "libic_pcg.so")
IC_OK, IC_E_ARG, IC_E_NOCONV, IC_E_BREAKDOWN, IC_E_OOM = 0, -1, -3, -4, -8


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"],
                       check=True)
    return _LIB


_lib = None
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.ic_factor.argtypes = [C.c_int64, _i64p, _i64p, _dp, C.c_double, C.POINTER(C.c_void_p)]
        L.ic_free.argtypes = [C.c_void_p]
        L.ic_nnz.restype = C.c_int64
        L.ic_nnz.argtypes = [C.c_void_p]
        L.ic_to_dense.argtypes = [C.c_void_p, _dp]
        L.ic_pcg.argtypes = [C.c_int64, _i64p, _i64p, _dp, C.c_void_p, _dp, _dp, C.c_double, C.c_int,
                             C.POINTER(C.c_int)]
        L.ic_simulate.argtypes = [C.c_int64, _i64p, _i64p, _dp, _dp, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                  _dp, C.c_double, C.c_int, _i32p]
        _lib = L
    return _lib


def _csr_arrays(A):
    A = A.tocsr()
    A.sort_indices()
    return (np.ascontiguousarray(A.indptr, dtype=np.int64), np.ascontiguousarray(A.indices, dtype=np.int64),
            np.ascontiguousarray(A.data, dtype=np.float64))


class ICFactor:
    """A ~ L L^T by threshold incomplete Cholesky (droptol 0: the exact Cholesky factor)."""

    def __init__(self, A, droptol: float = 1e-3):
        self.n = A.shape[0]
        self.rp, self.col, self.val = _csr_arrays(A)
        p = C.c_void_p()
        rc = lib().ic_factor(self.n, self.rp, self.col, self.val, droptol, C.byref(p))
        if rc != IC_OK:
            raise RuntimeError(f"ic_factor failed: {rc}")
        self._p = p

    def __del__(self):
        if getattr(self, "_p", None) and self._p.value and _lib is not None:
            _lib.ic_free(self._p)

    @property
    def nnz(self) -> int:
        return int(lib().ic_nnz(self._p))

    def dense(self) -> np.ndarray:
        D = np.empty((self.n, self.n))
        lib().ic_to_dense(self._p, D)
        return D

    def pcg(self, b, x0, tol=1e-12, max_iter=10000):
        x = np.array(x0, dtype=np.float64, copy=True)
        it = C.c_int(0)
        rc = lib().ic_pcg(self.n, self.rp, self.col, self.val, self._p, np.ascontiguousarray(b, dtype=np.float64), x,
                          tol, max_iter, C.byref(it))
        return x, it.value, rc

    def simulate(self, Lop, F, dt, nsteps, u0, tol=1e-6, max_iter=10000):
        """theta loop with A = this factor's matrix, b = Lop u^n + dt F (Lop on A's pattern)."""
        lrp, lcol, lval = _csr_arrays(Lop)
        assert np.array_equal(lrp, self.rp) and np.array_equal(lcol, self.col), "Lop must share A's pattern"
        u = np.array(u0, dtype=np.float64, copy=True)
        iters = np.zeros(nsteps, dtype=np.int32)
        Fp = np.ascontiguousarray(F, dtype=np.float64) if F is not None else None
        rc = lib().ic_simulate(self.n, self.rp, self.col, self.val, lval, self._p,
                               Fp.ctypes.data_as(C.c_void_p) if Fp is not None else None, dt, nsteps, u, tol,
                               max_iter, iters)
        return u, iters, rc
