"""TEST INFRASTRUCTURE ONLY: ctypes view of oracle/_ref/libmscref.so.

libmscref.so is the unmodified reference library (/root/reference/proj/src,
compiled in place by oracle/Makefile) plus the marshalling driver
oracle/refdrv.cpp.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; the product
package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libmscref.so")
REF_SRC = "/root/reference/proj"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH) or os.path.isdir(REF_SRC)


def build() -> None:
    """Compile the reference in place (only where /root/reference exists)."""
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref", "-j8"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error.argtypes = [C.POINTER(C.c_int)]
        L.ref_random_vector.argtypes = [C.c_int, C.c_uint, _f64p]
        L.ref_problem_free.argtypes = [vp]
        L.ref_problem_oseen.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double,
                                        C.c_int, C.c_int, C.POINTER(vp)]
        L.ref_problem_from_csr.argtypes = [C.c_int, _i32p, _i32p, _f64p, C.c_int,
                                           C.c_int, _i32p, C.POINTER(vp)]
        L.ref_problem_random_saddle.argtypes = [C.c_int, C.c_int, C.c_uint,
                                                C.c_double, C.POINTER(vp)]
        L.ref_problem_dims.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int64)]
        L.ref_csr_shape.restype = C.c_int64
        L.ref_csr_shape.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_csr_get.argtypes = [vp, C.c_int, _i32p, _i32p, _f64p]
        L.ref_get_perm.argtypes = [vp, _i32p]
        L.ref_get_scaled_rhs.argtypes = [vp, _f64p]
        L.ref_get_d_ranges.argtypes = [vp, _i32p]
        L.ref_nested_dissection.argtypes = [C.c_int, _i32p, _i32p, C.c_int, _i32p, _i32p, C.c_int]
        L.ref_nested_dissection.restype = C.c_int
        L.ref_set_overlap.argtypes = [vp, C.c_int]
        L.ref_set_overlap.restype = None
        L.ref_build_schur.argtypes = [vp, C.c_char_p, C.c_int, C.c_int, C.c_int,
                                      _i32p, C.c_int]
        L.ref_exact_schur.argtypes = [vp]
        L.ref_num_aggregates.argtypes = [vp]
        L.ref_get_schur_ranges.argtypes = [vp, _i32p]
        L.ref_build_precond.argtypes = [vp, C.c_double, C.c_int]
        L.ref_build_precond_parallel.argtypes = [vp, C.c_double, C.c_int, C.c_int]
        L.ref_problem_from_arrays.argtypes = [C.c_int, _i32p, _i32p, _f64p, C.c_int,
                                              C.c_int, _i32p, C.POINTER(vp)]
        L.ref_problem_set_schur.argtypes = [vp, C.c_char_p, _i32p, _i32p, _f64p, C.c_int,
                                            _i32p]
        L.ref_precond_begin.argtypes = [vp]
        L.ref_precond_set_dfactor.argtypes = [vp, C.c_int, C.c_int, _i32p, _i32p, _f64p,
                                              _i32p, _i32p, _f64p]
        L.ref_apply_threads.argtypes = [vp, _f64p, _f64p, C.c_int]
        L.ref_time_apply.restype = C.c_double
        L.ref_time_apply.argtypes = [vp, _f64p, _f64p, C.c_int]
        L.ref_time_apply_threads.restype = C.c_double
        L.ref_time_apply_threads.argtypes = [vp, _f64p, _f64p, C.c_int, C.c_int]
        L.ref_num_dfactors.argtypes = [vp]
        L.ref_stored_nnz.restype = C.c_int64
        L.ref_stored_nnz.argtypes = [vp]
        L.ref_factor_dims.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_factor_get.argtypes = [vp, C.c_int, C.c_int, _i32p, _i32p, _f64p,
                                     _i32p, _i32p, _f64p, _i32p]
        L.ref_apply.argtypes = [vp, _f64p, _f64p]
        L.ref_matvec.argtypes = [vp, C.c_int, _f64p, _f64p]
        L.ref_gmres.argtypes = [vp, C.c_int, _f64p, C.c_int, C.c_int, C.c_double,
                                C.c_int, _f64p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                _f64p, C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.ref_factor_ilut.argtypes = [C.c_int, _i32p, _i32p, _f64p, C.c_double,
                                      C.POINTER(vp)]
        L.ref_factor_exact.argtypes = [C.c_int, _i32p, _i32p, _f64p, C.POINTER(vp)]
        L.ref_factors_free.argtypes = [vp]
        L.ref_factors_dims.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64)]
        L.ref_factors_get.argtypes = [vp, _i32p, _i32p, _f64p, _i32p, _i32p, _f64p,
                                      _i32p]
        L.ref_factors_from_arrays.restype = vp
        L.ref_factors_from_arrays.argtypes = [C.c_int, _i32p, _i32p, _f64p, _i32p,
                                              _i32p, _f64p, C.c_void_p]
        L.ref_factors_from_csr.restype = vp
        L.ref_factors_from_csr.argtypes = [C.c_int, _i32p, _i32p, _f64p, _i32p, _i32p, _f64p]
        L.ref_solve.argtypes = [vp, _f64p, _f64p]
        L.ref_time_block_solves.restype = C.c_double
        L.ref_time_block_solves.argtypes = [C.c_int, C.POINTER(vp), _f64p, _f64p,
                                            C.c_int, C.c_int]
        L.ref_hardware_threads.restype = C.c_int
        L.ref_mm_read.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ref_random_dd_sparse.restype = vp
        L.ref_random_dd_sparse.argtypes = [C.c_int, C.c_double, C.c_uint]
        L.ref_oseen_raw_d.argtypes = [C.c_int, C.c_double, C.POINTER(vp)]
        L.ref_mat_dims.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int64)]
        L.ref_mat_get.argtypes = [vp, vp, vp, vp]
        L.ref_mat_free.argtypes = [vp]
        L.ref_mm_write.argtypes = [C.c_char_p, C.c_int, C.c_int, vp, vp, vp]
        L.ref_mm_read_vector.argtypes = [C.c_char_p, C.POINTER(C.c_int), vp]
        L.ref_mm_write_vector.argtypes = [C.c_char_p, C.c_int, vp]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, msg, pivot):
        super().__init__(msg)
        self.pivot_index = pivot


def _check(rc):
    if rc != 0:
        piv = C.c_int(-1)
        msg = lib().ref_last_error(C.byref(piv)).decode()
        raise RefError(msg, piv.value)


def random_vector(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().ref_random_vector(n, seed, out)
    return out


class Csr:
    def __init__(self, nrows, ncols, rp, ci, v):
        self.nrows, self.ncols = nrows, ncols
        self.rp, self.ci, self.v = rp, ci, v

    @property
    def nnz(self):
        return int(self.rp[-1])

    def to_dense(self):
        a = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            s, e = self.rp[i], self.rp[i + 1]
            a[i, self.ci[s:e]] = self.v[s:e]
        return a


class Factors:
    """Reference TriangularFactors (factorization.hpp:18-27) as arrays."""

    def __init__(self, handle, owned=True):
        self.h = handle
        self.owned = owned
        d, nl, nu = C.c_int(), C.c_int64(), C.c_int64()
        lib().ref_factors_dims(handle, C.byref(d), C.byref(nl), C.byref(nu))
        self.dim = d.value
        n = self.dim
        self.L = Csr(n, n, np.empty(n + 1, np.int32), np.empty(nl.value, np.int32),
                     np.empty(nl.value))
        self.U = Csr(n, n, np.empty(n + 1, np.int32), np.empty(nu.value, np.int32),
                     np.empty(nu.value))
        self.perm = np.empty(n, np.int32)
        lib().ref_factors_get(handle, self.L.rp, self.L.ci, self.L.v, self.U.rp,
                              self.U.ci, self.U.v, self.perm)

    def solve(self, b):
        x = np.empty(self.dim)
        _check(lib().ref_solve(self.h, np.ascontiguousarray(b, np.float64), x))
        return x

    def __del__(self):
        if self.owned and self.h:
            lib().ref_factors_free(self.h)
            self.h = None


def factor_ilut(a: Csr, tol: float) -> Factors:
    h = C.c_void_p()
    _check(lib().ref_factor_ilut(a.nrows, a.rp, a.ci, a.v, tol, C.byref(h)))
    return Factors(h)


def factor_exact(a: Csr) -> Factors:
    h = C.c_void_p()
    _check(lib().ref_factor_exact(a.nrows, a.rp, a.ci, a.v, C.byref(h)))
    return Factors(h)


def factors_from_arrays(n, L: Csr, U: Csr, perm=None):
    pp = None if perm is None else np.ascontiguousarray(perm, np.int32)
    h = lib().ref_factors_from_arrays(n, L.rp, L.ci, L.v, U.rp, U.ci, U.v,
                                      None if pp is None else pp.ctypes.data)
    f = Factors(h)
    f._keep = pp
    return f


def factors_from_csr(n, L: Csr, U: Csr):
    """ILUT factors from reference-invariant CSR (sorted rows, no explicit
    zeros, identity row permutation), without the triplet sort."""
    c = lambda a, t: np.ascontiguousarray(a, t)  # noqa: E731
    h = lib().ref_factors_from_csr(n, c(L.rp, np.int32), c(L.ci, np.int32), c(L.v, np.float64),
                                   c(U.rp, np.int32), c(U.ci, np.int32), c(U.v, np.float64))
    return Factors(h)


def cpu_info():
    """CPU model and logical CPU count of this host."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


class Problem:
    """A reference PartitionedMatrix + MSC preconditioner pipeline."""

    C, D, E, F, G, SHAT = range(6)

    def __init__(self, handle):
        self.h = handle
        n, p, nb, nnz = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        lib().ref_problem_dims(handle, C.byref(n), C.byref(p), C.byref(nb), C.byref(nnz))
        self.n, self.p, self.nblocks = n.value, p.value, nb.value

    @classmethod
    def oseen(cls, grid_n, nu, nA, stretched=False, stretch=1.056, anchored=False):
        h = C.c_void_p()
        _check(lib().ref_problem_oseen(grid_n, nu, int(stretched), stretch, nA,
                                       int(anchored), C.byref(h)))
        return cls(h)

    @classmethod
    def from_csr(cls, a: Csr, p, ranges=()):
        h = C.c_void_p()
        rr = np.asarray(ranges, np.int32).reshape(-1)
        if rr.size == 0:
            rr = np.zeros(2, np.int32)
        _check(lib().ref_problem_from_csr(a.nrows, a.rp, a.ci, a.v, p,
                                          len(ranges), rr, C.byref(h)))
        return cls(h)

    @classmethod
    def from_arrays(cls, a: Csr, p, ranges):
        """C given as reference-invariant CSR (sorted rows, no zeros), e.g.
        the product's bit-identical setup; no triplet sort."""
        h = C.c_void_p()
        rr = np.ascontiguousarray(np.asarray(ranges, np.int32).reshape(-1))
        _check(lib().ref_problem_from_arrays(a.nrows, np.ascontiguousarray(a.rp, np.int32),
                                             np.ascontiguousarray(a.ci, np.int32),
                                             np.ascontiguousarray(a.v, np.float64), p,
                                             len(rr) // 2, rr, C.byref(h)))
        return cls(h)

    @classmethod
    def random_saddle(cls, p, ng, seed, density=0.2):
        h = C.c_void_p()
        _check(lib().ref_problem_random_saddle(p, ng, seed, density, C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_problem_free(self.h)
            self.h = None

    @property
    def n_g(self):
        return self.n - self.p

    def csr(self, which) -> Csr:
        nr, nc = C.c_int(), C.c_int()
        nnz = lib().ref_csr_shape(self.h, which, C.byref(nr), C.byref(nc))
        if nnz < 0:
            raise ValueError("matrix not available")
        a = Csr(nr.value, nc.value, np.empty(nr.value + 1, np.int32),
                np.empty(nnz, np.int32), np.empty(nnz))
        lib().ref_csr_get(self.h, which, a.rp, a.ci, a.v)
        return a

    def perm(self):
        out = np.empty(self.n, np.int32)
        lib().ref_get_perm(self.h, out)
        return out

    def scaled_rhs(self):
        out = np.empty(self.n)
        _check(lib().ref_get_scaled_rhs(self.h, out))
        return out

    def d_ranges(self):
        out = np.empty(2 * self.nblocks, np.int32)
        lib().ref_get_d_ranges(self.h, out)
        return out.reshape(-1, 2)

    def build_schur(self, variant="lum", sz=0, mode=0, sizes=None, workers=1, overlap=-1):
        """aggregates (numbering, or overlapped with `overlap` as
        make_aggregates does, benchmark.cpp:74-88) + build_msc."""
        lib().ref_set_overlap(self.h, int(overlap))
        s = np.asarray(sizes if sizes is not None else [0], np.int32)
        _check(lib().ref_build_schur(self.h, variant.encode(), mode, sz, len(s), s,
                                     workers))

    def exact_schur(self):
        _check(lib().ref_exact_schur(self.h))

    def schur_ranges(self):
        k = lib().ref_num_aggregates(self.h)
        out = np.empty(2 * k, np.int32)
        lib().ref_get_schur_ranges(self.h, out)
        return out.reshape(-1, 2)

    def build_precond(self, tolA=1e-4, sA=0):
        _check(lib().ref_build_precond(self.h, tolA, sA))

    def build_precond_parallel(self, tolA=1e-4, sA=0, workers=0):
        """build_preconditioner with the per-block factorisations on
        `workers` threads (0 = all): the same MscPreconditioner."""
        _check(lib().ref_build_precond_parallel(self.h, tolA, sA, workers))

    def set_schur(self, variant, s_hat: Csr, ranges):
        rr = np.ascontiguousarray(np.asarray(ranges, np.int32).reshape(-1))
        _check(lib().ref_problem_set_schur(self.h, variant.encode(),
                                           np.ascontiguousarray(s_hat.rp, np.int32),
                                           np.ascontiguousarray(s_hat.ci, np.int32),
                                           np.ascontiguousarray(s_hat.v, np.float64),
                                           len(rr) // 2, rr))

    def precond_from_factors(self, get_block):
        """MscPreconditioner with the reference's own Schur factors and the
        interior factors get_block(b) -> (n, L: Csr, U: Csr) (e.g. downloaded
        from the GPU)."""
        _check(lib().ref_precond_begin(self.h))
        for b in range(self.nblocks):
            n, L, U = get_block(b)
            _check(lib().ref_precond_set_dfactor(
                self.h, b, n, np.ascontiguousarray(L.rp, np.int32),
                np.ascontiguousarray(L.ci, np.int32), np.ascontiguousarray(L.v, np.float64),
                np.ascontiguousarray(U.rp, np.int32), np.ascontiguousarray(U.ci, np.int32),
                np.ascontiguousarray(U.v, np.float64)))

    def apply_threads(self, y, workers=0):
        x = np.empty(self.n)
        _check(lib().ref_apply_threads(self.h, np.ascontiguousarray(y, np.float64), x,
                                       workers))
        return x

    def time_apply(self, y, reps=1, workers=None):
        """Wall seconds of `reps` applies: the stock single-threaded
        MscPreconditioner::apply (workers None) or the threaded block sweep."""
        x = np.empty(self.n)
        y = np.ascontiguousarray(y, np.float64)
        if workers is None:
            s = lib().ref_time_apply(self.h, y, x, reps)
        else:
            s = lib().ref_time_apply_threads(self.h, y, x, reps, workers)
            if s < 0:
                _check(-1)
        return s, x

    def stored_nnz(self):
        return int(lib().ref_stored_nnz(self.h))

    def factors(self, kind, idx):
        d, nl, nu = C.c_int(), C.c_int64(), C.c_int64()
        if lib().ref_factor_dims(self.h, kind, idx, C.byref(d), C.byref(nl), C.byref(nu)):
            raise IndexError(idx)
        n = d.value
        L = Csr(n, n, np.empty(n + 1, np.int32), np.empty(nl.value, np.int32),
                np.empty(nl.value))
        U = Csr(n, n, np.empty(n + 1, np.int32), np.empty(nu.value, np.int32),
                np.empty(nu.value))
        perm = np.empty(n, np.int32)
        lib().ref_factor_get(self.h, kind, idx, L.rp, L.ci, L.v, U.rp, U.ci, U.v, perm)
        return L, U, perm

    def apply(self, y):
        x = np.empty(self.n)
        _check(lib().ref_apply(self.h, np.ascontiguousarray(y, np.float64), x))
        return x

    def matvec(self, x, which=0):
        a_rows = self.csr(which).nrows if which else self.n
        y = np.empty(a_rows)
        _check(lib().ref_matvec(self.h, which, np.ascontiguousarray(x, np.float64), y))
        return y

    def gmres(self, b, restart, max_iters=3000, rel_tol=1e-8, left=False,
              use_prec=True):
        x = np.empty(self.n)
        its, conv, nh, secs = C.c_int(), C.c_int(), C.c_int(max_iters + 64), C.c_double()
        hist = np.empty(max_iters + 64)
        _check(lib().ref_gmres(self.h, int(use_prec), np.ascontiguousarray(b, np.float64),
                               restart, max_iters, rel_tol, int(left), x,
                               C.byref(its), C.byref(conv), hist, C.byref(nh),
                               C.byref(secs)))
        return dict(x=x, iterations=its.value, converged=bool(conv.value),
                    history=hist[: nh.value].copy(), seconds=secs.value)


def nested_dissection(rp, ci, target):
    """The reference's nested_dissection(build_graph(A), target) of a CSR
    pattern: (forward permutation, block ranges)."""
    n = len(rp) - 1
    perm = np.empty(n, np.int32)
    cap = max(1, 2 * target + 2)
    ranges = np.empty(2 * cap, np.int32)
    nb = lib().ref_nested_dissection(n, np.ascontiguousarray(rp, np.int32),
                                     np.ascontiguousarray(ci, np.int32), target, perm, ranges, cap)
    _check(0 if nb >= 0 else -1)
    return perm, ranges[: 2 * nb].reshape(-1, 2)


def time_block_solves(factors, rhs, reps, workers):
    arr = (C.c_void_p * len(factors))(*[f.h for f in factors])
    out = np.empty_like(rhs)
    secs = lib().ref_time_block_solves(len(factors), arr,
                                       np.ascontiguousarray(rhs), out, reps, workers)
    return secs, out


def hardware_threads():
    return lib().ref_hardware_threads()


# ---- Matrix Market (reference load/write_(matrix|vector)_market) ----------

def _vp(a):
    return a.ctypes.data_as(C.c_void_p)


def _mat_to_csr(h) -> Csr:
    try:
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_int64()
        lib().ref_mat_dims(h, C.byref(nr), C.byref(nc), C.byref(nnz))
        rp = np.empty(nr.value + 1, np.int32)
        ci = np.empty(max(1, nnz.value), np.int32)
        v = np.empty(max(1, nnz.value))
        lib().ref_mat_get(h, _vp(rp), _vp(ci), _vp(v))
        return Csr(nr.value, nc.value, rp, ci[:nnz.value].copy(), v[:nnz.value].copy())
    finally:
        lib().ref_mat_free(h)


def mm_read(path) -> Csr:
    h = C.c_void_p()
    _check(lib().ref_mm_read(os.fsencode(path), C.byref(h)))
    return _mat_to_csr(h)


def random_dd_sparse(n, density, seed) -> Csr:
    """oracle::random_dd_sparse with std::mt19937(seed) (tests/oracles.hpp:100-120)."""
    return _mat_to_csr(C.c_void_p(lib().ref_random_dd_sparse(n, density, seed)))


def oseen_raw_d(grid_n, nu) -> Csr:
    """generate_oseen(grid_n, nu).matrices.D (unscaled, original numbering)."""
    h = C.c_void_p()
    _check(lib().ref_oseen_raw_d(grid_n, nu, C.byref(h)))
    return _mat_to_csr(h)


def mm_write(path, a: Csr) -> None:
    rp = np.ascontiguousarray(a.rp, np.int32)
    ci = np.ascontiguousarray(a.ci, np.int32)
    v = np.ascontiguousarray(a.v, np.float64)
    _check(lib().ref_mm_write(os.fsencode(path), a.nrows, a.ncols, _vp(rp), _vp(ci), _vp(v)))


def mm_read_vector(path) -> np.ndarray:
    n = C.c_int()
    _check(lib().ref_mm_read_vector(os.fsencode(path), C.byref(n), None))
    out = np.empty(n.value)
    _check(lib().ref_mm_read_vector(os.fsencode(path), C.byref(n), _vp(out)))
    return out


def mm_write_vector(path, v) -> None:
    v = np.ascontiguousarray(v, np.float64)
    _check(lib().ref_mm_write_vector(os.fsencode(path), len(v), _vp(v)))
