"""TEST INFRASTRUCTURE ONLY: ctypes view of the plain-C oracle restatement
(oracle/restate.c -> oracle/_build/liborestate.so).

Used by tests/ (as the checker), __graft_entry__.smoke() and bench.py's
cpu_baseline leg.  Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liborestate.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "restate"], check=True)


class _Msc(C.Structure):
    _fields_ = [("n", C.c_int), ("p", C.c_int), ("nd", C.c_int), ("ns", C.c_int),
                ("d_ranges", C.c_void_p), ("s_ranges", C.c_void_p),
                ("dfac", C.c_void_p), ("sfac", C.c_void_p),
                ("e_nrows", C.c_int), ("e_rp", C.c_void_p), ("e_ci", C.c_void_p),
                ("e_v", C.c_void_p),
                ("f_nrows", C.c_int), ("f_rp", C.c_void_p), ("f_ci", C.c_void_p),
                ("f_v", C.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.rs_matvec.argtypes = [C.c_int, _i32p, _i32p, _f64p, _f64p, _f64p]
        L.rs_ilut.argtypes = [C.c_int, _i32p, _i32p, _f64p, C.c_double, C.POINTER(vp)]
        L.rs_exact.argtypes = [C.c_int, _i32p, _i32p, _f64p, C.POINTER(vp)]
        L.rs_factors_free.argtypes = [vp]
        L.rs_factors_dims.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]
        L.rs_factors_get.argtypes = [vp, _i32p, _i32p, _f64p, _i32p, _i32p, _f64p, _i32p]
        L.rs_solve.argtypes = [vp, _f64p, _f64p]
        L.rs_msc_apply.argtypes = [C.POINTER(_Msc), _f64p, _f64p]
        L.rs_gmres.argtypes = [C.c_int, _i32p, _i32p, _f64p, C.POINTER(_Msc), C.c_int,
                               _f64p, C.c_int, C.c_int, C.c_double, _f64p,
                               C.POINTER(C.c_int), C.POINTER(C.c_int), _f64p,
                               C.POINTER(C.c_int)]
        _lib = L
    return _lib


class SingularMatrixError(RuntimeError):
    def __init__(self, msg, pivot):
        super().__init__(msg)
        self.pivot_index = pivot


def matvec(rp, ci, v, x):
    y = np.empty(len(rp) - 1)
    lib().rs_matvec(len(rp) - 1, rp, ci, v, np.ascontiguousarray(x, np.float64), y)
    return y


class Factors:
    def __init__(self, h):
        self.h = h
        n, nl, nu = C.c_int(), C.c_int64(), C.c_int64()
        lib().rs_factors_dims(h, C.byref(n), C.byref(nl), C.byref(nu))
        self.dim = n.value
        d = self.dim
        self.lrp = np.empty(d + 1, np.int32); self.lci = np.empty(nl.value, np.int32)
        self.lv = np.empty(nl.value)
        self.urp = np.empty(d + 1, np.int32); self.uci = np.empty(nu.value, np.int32)
        self.uv = np.empty(nu.value)
        self.perm = np.empty(d, np.int32)
        lib().rs_factors_get(h, self.lrp, self.lci, self.lv, self.urp, self.uci,
                             self.uv, self.perm)

    @property
    def nnz(self):
        return int(self.lrp[-1] + self.urp[-1])

    def solve(self, b):
        x = np.empty(self.dim)
        lib().rs_solve(self.h, np.ascontiguousarray(b, np.float64), x)
        return x

    def __del__(self):
        if getattr(self, "h", None):
            lib().rs_factors_free(self.h)
            self.h = None


def factor_ilut(n, rp, ci, v, tol):
    h = C.c_void_p()
    rc = lib().rs_ilut(n, rp, ci, v, tol, C.byref(h))
    if rc != 0:
        piv = -1 - rc
        raise SingularMatrixError(f"factor_ilut: zero pivot at index {piv}", piv)
    return Factors(h)


def factor_exact(n, rp, ci, v):
    h = C.c_void_p()
    rc = lib().rs_exact(n, rp, ci, v, C.byref(h))
    if rc != 0:
        piv = -1 - rc
        raise SingularMatrixError(f"dense_lu: zero pivot at index {piv}", piv)
    return Factors(h)


def _sub_csr(rp, ci, v, b, e):
    """extract_block(A, b, e, b, e) for a block-diagonal range (rows sorted)."""
    s, t = rp[b], rp[e]
    cols = ci[s:t]
    keep = (cols >= b) & (cols < e)
    rows = np.repeat(np.arange(e - b), np.diff(rp[b:e + 1]))
    rows, cols, vals = rows[keep], cols[keep] - b, v[s:t][keep]
    nrp = np.zeros(e - b + 1, np.int32)
    np.add.at(nrp, rows + 1, 1)
    return np.cumsum(nrp).astype(np.int32), cols.astype(np.int32), vals.copy()


class Msc:
    """MSC preconditioner assembled from D/E/F/S^ CSR + ranges (the oracle
    restatement of build_preconditioner, preconditioner.cpp:26-83, for the
    block-diagonal Schur case)."""

    def __init__(self, n, p, D, E, F, S, d_ranges, s_ranges, tolA=1e-4, sA=0):
        self.n, self.p = n, p
        self.dfac, self.sfac = [], []
        for bi, (b, e) in enumerate(d_ranges):
            blk = _sub_csr(*D, b, e)
            try:
                f = (factor_exact(e - b, *blk) if (e - b) <= sA
                     else factor_ilut(e - b, *blk, tolA))
            except SingularMatrixError as err:
                raise SingularMatrixError(
                    f"build_preconditioner: (1,1) block {bi}: {err}", err.pivot_index)
            self.dfac.append(f)
        for si, (b, e) in enumerate(s_ranges):
            blk = _sub_csr(*S, b, e)
            try:
                self.sfac.append(factor_exact(e - b, *blk))
            except SingularMatrixError as err:
                raise SingularMatrixError(
                    f"build_preconditioner: Schur block {si}: {err}", err.pivot_index)
        self.E, self.F = E, F
        self._dr = np.ascontiguousarray(np.asarray(d_ranges, np.int32).reshape(-1))
        self._sr = np.ascontiguousarray(np.asarray(s_ranges, np.int32).reshape(-1))
        self._dptr = (C.c_void_p * len(self.dfac))(*[f.h for f in self.dfac])
        self._sptr = (C.c_void_p * max(1, len(self.sfac)))(*[f.h for f in self.sfac])
        self.s = _Msc(n, p, len(self.dfac), len(self.sfac),
                      self._dr.ctypes.data, self._sr.ctypes.data,
                      C.cast(self._dptr, C.c_void_p), C.cast(self._sptr, C.c_void_p),
                      len(E[0]) - 1, E[0].ctypes.data, E[1].ctypes.data, E[2].ctypes.data,
                      len(F[0]) - 1, F[0].ctypes.data, F[1].ctypes.data, F[2].ctypes.data)

    def apply(self, y):
        x = np.empty(self.n)
        lib().rs_msc_apply(C.byref(self.s), np.ascontiguousarray(y, np.float64), x)
        return x

    @property
    def stored_nnz(self):
        return (sum(f.nnz for f in self.dfac) + sum(f.nnz for f in self.sfac)
                + len(self.E[1]) + len(self.F[1]))


def gmres(A, b, restart, max_iters=3000, rel_tol=1e-8, msc: Msc | None = None,
          side="right"):
    rp, ci, v = A
    n = len(rp) - 1
    x = np.empty(n)
    its, conv, nh = C.c_int(), C.c_int(), C.c_int(max_iters + 64)
    hist = np.empty(max_iters + 64)
    sd = 0 if msc is None else (1 if side == "right" else 2)
    rc = lib().rs_gmres(n, rp, ci, v, C.byref(msc.s) if msc else None, sd,
                        np.ascontiguousarray(b, np.float64), restart, max_iters,
                        rel_tol, x, C.byref(its), C.byref(conv), hist, C.byref(nh))
    if rc != 0:
        raise ValueError("gmres: bad solver configuration")
    return dict(x=x, iterations=its.value, converged=bool(conv.value),
                history=hist[: nh.value].copy())
