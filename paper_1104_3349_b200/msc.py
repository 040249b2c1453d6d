"""Python mirror of the reference's solve-phase API (proj/include/msc/) over
the C ABI (include/mscg.h).  Names, argument meaning and error behaviour
follow the reference:

    SparseMatrix / matvec                 sparse_matrix.hpp:34-87
    TriangularFactors                     factorization.hpp:18-27
    SingularMatrixError(pivot_index)      sparse_matrix.hpp:23-28
    build_preconditioner(...)             preconditioner.hpp:66-68
    MscPreconditioner.apply / stored_nnz / d_factors / schur_factors
                                          preconditioner.hpp:34-64
    SolverConfig / SolveReport / gmres    gmres.hpp:17-47
    true_residual                         gmres.hpp:36
    fill_factor                           preconditioner.hpp:125

Host problem setup (generate_oseen -> scale_rows -> partition_saddle ->
aggregates -> build_msc) is exposed as `oseen_problem` / `Problem`.
Every numerical call runs on the GPU; without a device the calls raise
CudaError (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _capi as api



def _destroy(name, h):
    """Handle release for __del__: at interpreter shutdown the module globals
    may already be gone, and a destructor must not raise."""
    try:
        getattr(api.lib(), name)(h)
    except Exception:  # noqa: BLE001
        pass


class MscError(RuntimeError):
    pass


class SingularMatrixError(MscError):
    def __init__(self, what, pivot_index=-1, block=-1):
        super().__init__(what)
        self.pivot_index = pivot_index
        self.block = block


class CudaError(MscError):
    pass


class IoError(MscError):
    """msc::IoError (proj/include/msc/matrix_market.hpp:16-24)."""


def _check(rc, st: api.Status):
    if rc == api.MSCG_OK:
        return
    msg = st.message.decode(errors="replace")
    if rc == api.MSCG_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == api.MSCG_ERR_SINGULAR:
        raise SingularMatrixError(msg, st.pivot_index, st.block)
    if rc == api.MSCG_ERR_CUDA:
        raise CudaError(msg)
    if rc == api.MSCG_ERR_OUT_OF_MEMORY:
        raise MemoryError(msg)
    if rc == api.MSCG_ERR_IO:
        raise IoError(msg)
    raise MscError(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class SparseMatrix:
    """Host CSR (int32 row offsets / columns, fp64 values)."""
    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    @classmethod
    def from_dense(cls, a: np.ndarray) -> "SparseMatrix":
        a = np.asarray(a, np.float64)
        rows, cols = np.nonzero(a)
        rp = np.zeros(a.shape[0] + 1, np.int32)
        np.add.at(rp, rows + 1, 1)
        return cls(a.shape[0], a.shape[1], np.cumsum(rp).astype(np.int32),
                   cols.astype(np.int32), a[rows, cols].astype(np.float64))

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_offsets))
        d[rows, self.col_indices] = self.values
        return d

    def arrays(self):
        return (np.ascontiguousarray(self.row_offsets, np.int32),
                np.ascontiguousarray(self.col_indices, np.int32),
                np.ascontiguousarray(self.values, np.float64))


class Context:
    """One CUDA device + stream (mscg_ctx)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        st = api.Status()
        _check(api.lib().mscg_ctx_create(device, C.byref(self.h), C.byref(st)), st)
        self.device = device

    @property
    def stream_handle(self) -> int:
        return api.lib().mscg_ctx_stream(self.h) or 0

    def synchronize(self):
        st = api.Status()
        _check(api.lib().mscg_ctx_synchronize(self.h, C.byref(st)), st)

    @property
    def launches(self) -> int:
        return int(api.lib().mscg_ctx_launches(self.h))

    def set_stream(self, stream_handle: int | None):
        """Order later calls on an external cudaStream_t (e.g.
        torch.cuda.current_stream().cuda_stream, so that work and NCCL
        collectives interleave in stream order); None restores the context's
        own stream."""
        st = api.Status()
        _check(api.lib().mscg_ctx_set_stream(self.h, C.c_void_p(stream_handle or None),
                                             int(stream_handle is None), C.byref(st)), st)

    def set_correction(self, mode):
        """Interior correction of preconditioners built later on this context:
        "off" (the reference's E SpMV + second interior solve), "on" (W = D^-1 E
        precomputed, x1 = z1 - W z2), "auto" (on when W saves bytes), None
        (default: MSCG_CORRECTION or auto)."""
        m = {"off": 0, "on": 1, "auto": 2, None: -1}[mode]
        st = api.Status()
        _check(api.lib().mscg_ctx_set_correction(self.h, m, C.byref(st)), st)

    def torch_stream(self):
        import torch
        return torch.cuda.ExternalStream(self.stream_handle, device=f"cuda:{self.device}")

    def __del__(self):
        if getattr(self, "h", None):
            _destroy("mscg_ctx_destroy", self.h)
            self.h = None


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _vec_args(x, n):
    """(pointer, mem, keepalive, is_torch) for a host ndarray or CUDA tensor."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.device.type != "cuda" or x.dtype != torch.float64 or not x.is_contiguous():
                raise ValueError("device vectors must be contiguous float64 CUDA tensors")
            if x.numel() != n:
                raise ValueError(f"length mismatch: {x.numel()} vs {n}")
            return C.c_void_p(x.data_ptr()), api.MEM_DEVICE, x, True
    except ImportError:
        pass
    a = np.ascontiguousarray(x, np.float64)
    if a.size != n:
        raise ValueError(f"length mismatch: {a.size} vs {n}")
    return _ptr(a), api.MEM_HOST, a, False


class DeviceMatrix:
    """HBM-resident CSR (SELL-32) for matvec / GMRES operators."""

    def __init__(self, ctx: Context, a: SparseMatrix | None = None, _borrow=None):
        self.ctx = ctx
        self._owned = a is not None
        if _borrow is not None:
            self.h = C.c_void_p(_borrow)
            self.nrows = self.ncols = None
            return
        rp, ci, v = a.arrays()
        self._keep = (rp, ci, v)
        self.h = C.c_void_p()
        st = api.Status()
        _check(api.lib().mscg_csr_upload(ctx.h, a.nrows, a.ncols, _ptr(rp), _ptr(ci), _ptr(v),
                                         C.byref(self.h), C.byref(st)), st)
        self.nrows, self.ncols = a.nrows, a.ncols

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "h", None):
            _destroy("mscg_csr_destroy", self.h)
            self.h = None


def matvec(a: DeviceMatrix, x):
    """y = A x (reference order, bit-identical)."""
    px, mem, keep, is_t = _vec_args(x, a.ncols)
    if is_t:
        import torch
        y = torch.empty(a.nrows, dtype=torch.float64, device=x.device)
        py = C.c_void_p(y.data_ptr())
        torch.cuda.current_stream().synchronize()
    else:
        y = np.empty(a.nrows)
        py = _ptr(y)
    st = api.Status()
    _check(api.lib().mscg_spmv(a.h, px, py, mem, C.byref(st)), st)
    if is_t:
        a.ctx.synchronize()
    return y


@dataclass
class TriangularFactors:
    lower: SparseMatrix
    upper: SparseMatrix
    row_perm: np.ndarray
    kind: str

    def dim(self):
        return self.upper.nrows

    def nnz(self):
        return self.lower.nnz + self.upper.nnz


class DeviceFactors(TriangularFactors):
    """factor_ilut / factor_exact of one block, resident on the device
    (factorization.hpp:18-43): the reference CSR fields are downloaded once,
    `solve` runs the device triangular solve."""

    def __init__(self, ctx: Context, handle, kind: str):
        self.ctx, self.h = ctx, handle
        st = api.Status()
        d, nl, nu = C.c_int(), C.c_int64(), C.c_int64()
        L = api.lib()
        _check(L.mscg_factors_get(handle, C.byref(d), C.byref(nl), C.byref(nu), None, None,
                                  None, None, None, None, None, C.byref(st)), st)
        n = d.value
        lrp, urp = np.empty(n + 1, np.int32), np.empty(n + 1, np.int32)
        lci, lv = np.empty(max(1, nl.value), np.int32), np.empty(max(1, nl.value))
        uci, uv = np.empty(max(1, nu.value), np.int32), np.empty(max(1, nu.value))
        perm = np.empty(n, np.int32)
        _check(L.mscg_factors_get(handle, C.byref(d), C.byref(nl), C.byref(nu), _ptr(lrp),
                                  _ptr(lci), _ptr(lv), _ptr(urp), _ptr(uci), _ptr(uv),
                                  _ptr(perm), C.byref(st)), st)
        super().__init__(SparseMatrix(n, n, lrp, lci[: nl.value], lv[: nl.value]),
                         SparseMatrix(n, n, urp, uci[: nu.value], uv[: nu.value]), perm, kind)

    def solve(self, b):
        """x = U^-1 L^-1 P b (factorization.cpp:129-158) on the device."""
        b = np.ascontiguousarray(b, np.float64)
        if b.shape != (self.dim(),):
            raise ValueError("solve: rhs length mismatch")
        x = np.empty(self.dim())
        st = api.Status()
        _check(api.lib().mscg_factors_solve(self.h, _ptr(b), _ptr(x), api.MEM_HOST,
                                            C.byref(st)), st)
        return x

    def __del__(self):
        if getattr(self, "h", None):
            _destroy("mscg_factors_destroy", self.h)
            self.h = None


def _factor(a: SparseMatrix, kind: int, tol: float, ctx: Context | None):
    if a.nrows != a.ncols:
        raise ValueError("factor_exact: matrix not square" if kind else
                         "factor_ilut: matrix not square")
    ctx = ctx or default_context()
    rp, ci, v = a.arrays()
    h = C.c_void_p()
    st = api.Status()
    _check(api.lib().mscg_factor(ctx.h, a.nrows, _ptr(rp), _ptr(ci), _ptr(v), kind, tol,
                                 C.byref(h), C.byref(st)), st)
    return DeviceFactors(ctx, h, "exact" if kind else "incomplete")


def factor_ilut(a: SparseMatrix, drop_tol: float, ctx: Context | None = None) -> DeviceFactors:
    """Row-wise ILUT (factorization.hpp:38) on the device (ilut_kernel)."""
    return _factor(a, 0, drop_tol, ctx)


def factor_exact(a: SparseMatrix, ctx: Context | None = None) -> DeviceFactors:
    """LU with partial pivoting (factorization.hpp:32) on the device."""
    return _factor(a, 1, 0.0, ctx)


class MscPreconditioner:
    """Device-resident MSC preconditioner B = [D 0; F S^][D^-1 0; 0 S^-1][D E; 0 S^]."""

    def __init__(self, ctx: Context, handle, kind: str, sA: int, d_sizes=None):
        self.ctx = ctx
        self.h = handle
        self._kind = kind
        self._sA = sA
        n, p, nb, ns = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        api.lib().mscg_precond_dims(self.h, C.byref(n), C.byref(p), C.byref(nb), C.byref(ns))
        self.n, self.p, self.nblocks, self.nschur = n.value, p.value, nb.value, ns.value
        self.matrix = DeviceMatrix(ctx, _borrow=api.lib().mscg_precond_matrix(self.h))
        self.matrix.nrows = self.matrix.ncols = self.n

    def kind(self):
        return self._kind

    def dim(self):
        return self.n

    def stored_nnz(self) -> int:
        return int(api.lib().mscg_precond_stored_nnz(self.h))

    def build_times(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        api.lib().mscg_precond_build_times(self.h, C.byref(a), C.byref(b), C.byref(c))
        return dict(ilut_s=a.value, schur_lu_s=b.value, pack_s=c.value)

    def correction(self):
        """Explicit interior correction in use: dict(on, entries, kmax, build_s)."""
        on, k = C.c_int(), C.c_int()
        e, t = C.c_int64(), C.c_double()
        api.lib().mscg_precond_correction(self.h, C.byref(on), C.byref(e), C.byref(k), C.byref(t))
        return dict(on=bool(on.value), entries=e.value, kmax=k.value, build_s=t.value)

    def apply(self, y):
        """x = B^-1 y.  Host ndarray in -> ndarray out; CUDA tensor in -> tensor out."""
        py, mem, keep, is_t = _vec_args(y, self.n)
        if is_t:
            import torch
            x = torch.empty(self.n, dtype=torch.float64, device=y.device)
            px = C.c_void_p(x.data_ptr())
            torch.cuda.current_stream().synchronize()
        else:
            x = np.empty(self.n)
            px = _ptr(x)
        st = api.Status()
        _check(api.lib().mscg_precond_apply(self.h, py, px, mem, C.byref(st)), st)
        if is_t:
            self.ctx.synchronize()
        return x

    def apply_on_stream(self, y, x, stream_handle: int):
        """Enqueue x = B^-1 y (contiguous float64 CUDA tensors) on the given
        cudaStream_t; safe to call from several threads at once."""
        st = api.Status()
        _check(api.lib().mscg_precond_apply_stream(self.h, C.c_void_p(y.data_ptr()),
                                                   C.c_void_p(x.data_ptr()),
                                                   C.c_void_p(stream_handle), C.byref(st)), st)

    def use_correction(self, on: bool):
        """Apply with the explicit correction panels (when built) or the
        reference's E SpMV + second interior solve."""
        api.lib().mscg_precond_use_correction(self.h, int(bool(on)))

    def apply_async(self, y_ptr: int, x_ptr: int):
        """Enqueue x = B^-1 y on the context stream (raw device pointers)."""
        st = api.Status()
        _check(api.lib().mscg_precond_apply(self.h, C.c_void_p(y_ptr), C.c_void_p(x_ptr),
                                            api.MEM_DEVICE, C.byref(st)), st)

    def _factors(self, kind: int, idx: int) -> TriangularFactors:
        st = api.Status()
        d, nl, nu = C.c_int(), C.c_int64(), C.c_int64()
        L = api.lib()
        _check(L.mscg_precond_factor(self.h, kind, idx, C.byref(d), C.byref(nl), C.byref(nu),
                                     None, None, None, None, None, None, None, C.byref(st)), st)
        n = d.value
        lrp, urp = np.empty(n + 1, np.int32), np.empty(n + 1, np.int32)
        lci, lv = np.empty(max(1, nl.value), np.int32), np.empty(max(1, nl.value))
        uci, uv = np.empty(max(1, nu.value), np.int32), np.empty(max(1, nu.value))
        perm = np.empty(n, np.int32)
        _check(L.mscg_precond_factor(self.h, kind, idx, C.byref(d), C.byref(nl), C.byref(nu),
                                     _ptr(lrp), _ptr(lci), _ptr(lv), _ptr(urp), _ptr(uci),
                                     _ptr(uv), _ptr(perm), C.byref(st)), st)
        lower = SparseMatrix(n, n, lrp, lci[: nl.value], lv[: nl.value])
        upper = SparseMatrix(n, n, urp, uci[: nu.value], uv[: nu.value])
        exact = kind == 1 or n <= self._sA
        return TriangularFactors(lower, upper, perm, "exact" if exact else "incomplete")

    def d_factors(self, idx: int) -> TriangularFactors:
        return self._factors(0, idx)

    def schur_factors(self, idx: int) -> TriangularFactors:
        return self._factors(1, idx)

    def __del__(self):
        if getattr(self, "h", None):
            _destroy("mscg_precond_destroy", self.h)
            self.h = None


class Problem:
    """Host setup layer: partitioned saddle system in the final numbering."""

    def __init__(self, handle):
        self.h = handle
        n, p, nb, sep = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        nnz = C.c_int64()
        api.lib().mscg_problem_dims(self.h, C.byref(n), C.byref(p), C.byref(nb), C.byref(nnz),
                                    C.byref(sep))
        self.n, self.p, self.nblocks = n.value, p.value, nb.value
        self.separator_size = sep.value
        self.variant = None

    @property
    def n_g(self):
        return self.n - self.p

    def _csr(self, which) -> SparseMatrix:
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_int64()
        rp, ci, v = C.POINTER(C.c_int)(), C.POINTER(C.c_int)(), C.POINTER(C.c_double)()
        rc = api.lib().mscg_problem_csr(self.h, which, C.byref(nr), C.byref(nc), C.byref(nnz),
                                        C.byref(rp), C.byref(ci), C.byref(v))
        if rc:
            raise ValueError("matrix not available (build_msc first?)")
        n, m = nr.value, nnz.value
        return SparseMatrix(n, nc.value, np.ctypeslib.as_array(rp, (n + 1,)).copy(),
                            np.ctypeslib.as_array(ci, (max(m, 1),))[:m].copy(),
                            np.ctypeslib.as_array(v, (max(m, 1),))[:m].copy())

    @property
    def C(self) -> SparseMatrix:
        return self._csr(0)

    @property
    def s_hat(self) -> SparseMatrix:
        return self._csr(5)

    def perm(self) -> np.ndarray:
        return np.ctypeslib.as_array(api.lib().mscg_problem_perm(self.h), (self.n,)).copy()

    def d_ranges(self) -> np.ndarray:
        return np.ctypeslib.as_array(api.lib().mscg_problem_d_ranges(self.h),
                                     (2 * self.nblocks,)).reshape(-1, 2).copy()

    def scaled_rhs(self):
        p = api.lib().mscg_problem_scaled_rhs(self.h)
        return None if not p else np.ctypeslib.as_array(p, (self.n,)).copy()

    def build_msc(self, variant="lum", sz=0, mode="equal", sizes=None, threads=0,
                  ctx: "Context | None" = None, overlap=-1, widths=None):
        """build_msc (schur_approx.cpp:88-161) over numbering aggregates; on the
        host (threads) or, with ctx, on the device — S^ bit-identical either way.
        Overlapped variants ("omscn", "omscnr", "olum"): aggregate_overlapped
        (aggregates.cpp:50-85) with `widths`, or `overlap` per aggregate
        (< 0: sz; last 0; clipped as benchmark.cpp:74-88 does); the
        preconditioner then factors the banded S^ whole."""
        m = {"equal": 0, "anchored": 1, "explicit": 2}[mode]
        s = np.ascontiguousarray(sizes if sizes is not None else [0], np.int32)
        st = api.Status()
        if variant.startswith("o") or widths is not None:
            w = None if widths is None else np.ascontiguousarray(widths, np.int32)
            _check(api.lib().mscg_problem_build_schur_overlapped(
                ctx.h if ctx is not None else None, self.h, variant.encode(), m, sz, len(s),
                _ptr(s), int(overlap), 0 if w is None else len(w),
                _ptr(w) if w is not None else None, threads,
                C.byref(st)), st)
        elif ctx is not None:
            _check(api.lib().mscg_problem_build_schur_device(
                ctx.h, self.h, variant.encode(), m, sz, len(s), _ptr(s), C.byref(st)), st)
        else:
            _check(api.lib().mscg_problem_build_schur(self.h, variant.encode(), m, sz, len(s),
                                                      _ptr(s), threads, C.byref(st)), st)
        self.variant = variant
        return self

    def schur_ranges(self) -> np.ndarray:
        k = api.lib().mscg_problem_num_aggregates(self.h)
        if k < 0:
            raise ValueError("build_msc first")
        return np.ctypeslib.as_array(api.lib().mscg_problem_schur_ranges(self.h),
                                     (2 * k,)).reshape(-1, 2).copy()

    def __del__(self):
        if getattr(self, "h", None):
            _destroy("mscg_problem_destroy", self.h)
            self.h = None


def oseen_problem(grid_n, nu, n_a, stretched=False, stretch=1.056, anchored=False,
                  threads=0, ctx: "Context | None" = None) -> Problem:
    """generate_oseen -> scale_rows -> partition_saddle(Interleaved) [-> anchoring].
    With ctx the assembly and row scaling run on the device (bit-identical)."""
    h = C.c_void_p()
    st = api.Status()
    if ctx is not None:
        _check(api.lib().mscg_problem_oseen_device(ctx.h, grid_n, nu, int(stretched), stretch,
                                                   n_a, int(anchored), threads, C.byref(h),
                                                   C.byref(st)), st)
    else:
        _check(api.lib().mscg_problem_oseen(grid_n, nu, int(stretched), stretch, n_a,
                                            int(anchored), threads, C.byref(h), C.byref(st)), st)
    return Problem(h)


def nested_dissection(a: SparseMatrix, target_blocks: int, ctx: "Context | None" = None,
                      threads: int = 0):
    """nested_dissection(build_graph(a), target_blocks) (graph.cpp:178-230):
    (forward permutation, block ranges) — on the device with a context, else
    on the host; identical to the reference either way."""
    rp, ci, _ = a.arrays()
    n = a.nrows
    perm = np.empty(max(n, 1), np.int32)
    cap = 2 * max(1, target_blocks) + 2
    ranges = np.empty(2 * cap, np.int32)
    nb = C.c_int()
    st = api.Status()
    _check(api.lib().mscg_nested_dissection(ctx.h if ctx is not None else None, n, _ptr(rp),
                                            _ptr(ci), target_blocks, threads, _ptr(perm),
                                            C.byref(nb), _ptr(ranges), cap, C.byref(st)), st)
    return perm[:n], ranges[: 2 * min(nb.value, cap)].reshape(-1, 2)


def partitioned_problem(c: SparseMatrix, p: int, d_ranges=()) -> Problem:
    """PartitionedMatrix::from_split(C, p, d_ranges)."""
    rp, ci, v = c.arrays()
    rr = np.ascontiguousarray(np.asarray(d_ranges, np.int32).reshape(-1))
    if rr.size == 0:
        rr = np.zeros(2, np.int32)
    h = C.c_void_p()
    st = api.Status()
    _check(api.lib().mscg_problem_from_csr(c.nrows, _ptr(rp), _ptr(ci), _ptr(v), p,
                                           len(d_ranges), _ptr(rr), C.byref(h), C.byref(st)), st)
    return Problem(h)


def build_preconditioner(problem: Problem, tolA: float = 1e-4, sA: int = 400,
                         ctx: Context | None = None) -> MscPreconditioner:
    """Factor every interior block (ILUT(tolA) above sA, exact LU at or below)
    and every Schur block on the GPU."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    st = api.Status()
    _check(api.lib().mscg_precond_build_problem(ctx.h, problem.h, tolA, sA, C.byref(h),
                                                C.byref(st)), st)
    return MscPreconditioner(ctx, h, problem.variant or "msc", sA)


class PreconditionerShard:
    """The interior blocks [block_begin, block_end) of an MSC preconditioner
    split across ranks: its D blocks, E rows and F columns, with
    the Schur factors replicated.  Vectors are CUDA float64 tensors of global
    length n; a rank touches its interior rows `rows` and the interface rows.
    One apply = apply_begin -> all-reduce(t) over ranks -> apply_end."""

    def __init__(self, ctx: Context, handle, block_begin: int, block_end: int):
        self.ctx = ctx
        self.h = handle
        self.block_begin, self.block_end = block_begin, block_end
        n, p, nb, ns = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        api.lib().mscg_precond_dims(self.h, C.byref(n), C.byref(p), C.byref(nb), C.byref(ns))
        self.n, self.p = n.value, p.value
        lo, hi = C.c_int(), C.c_int()
        api.lib().mscg_precond_shard_rows(self.h, C.byref(lo), C.byref(hi))
        self.rows = (lo.value, hi.value)

    @property
    def n_g(self):
        return self.n - self.p

    def stored_nnz(self) -> int:
        return int(api.lib().mscg_precond_stored_nnz(self.h))

    def apply_begin(self, y, t):
        """z1 = D_r^-1 y1 (own rows); t = F_r z1 (this rank's share of F z1)."""
        st = api.Status()
        _check(api.lib().mscg_precond_apply_shard(self.h, 0, C.c_void_p(y.data_ptr()),
                                                  C.c_void_p(t.data_ptr()), None,
                                                  C.byref(st)), st)

    def apply_end(self, y, t, x):
        """With t = F z1 summed over ranks: x2 = S^-1 (y2 - t), x1 = z1 - D_r^-1 E_r x2."""
        st = api.Status()
        _check(api.lib().mscg_precond_apply_shard(self.h, 1, C.c_void_p(y.data_ptr()),
                                                  C.c_void_p(t.data_ptr()),
                                                  C.c_void_p(x.data_ptr()), C.byref(st)), st)

    def spmv(self, x, y, y2part, with_interface_block: bool):
        """y[rows] = C[rows, :] x and y2part = F_r x[rows] (+ C22 x2 on one
        rank); the interface rows of C x are y2part summed over ranks."""
        st = api.Status()
        _check(api.lib().mscg_precond_spmv_shard(self.h, C.c_void_p(x.data_ptr()),
                                                 C.c_void_p(y.data_ptr()),
                                                 C.c_void_p(y2part.data_ptr()),
                                                 int(with_interface_block), C.byref(st)), st)

    def gmres(self, b, cfg: "SolverConfig", rank: int, world: int, group=None):
        """Distributed right-preconditioned GMRES (DCGS2) across the ranks'
        shards; every rank calls it with the same global-length b (numpy or a
        CUDA float64 tensor).  Returns (x, SolveReport): x global-length with
        this rank's interior rows and the interface filled (others zero).
        The exchanges run through torch.distributed.all_reduce on `group`,
        ordered on the context stream (bound to torch's current stream)."""
        import torch
        import torch.distributed as dist
        if cfg.side != "right" or cfg.orth != "dcgs2":
            raise ValueError("gmres_shard: right preconditioning with DCGS2 only")
        dev = torch.device("cuda", torch.cuda.current_device())
        cap = max(2 * cfg.restart + 4, self.n_g, 8)
        buf = torch.zeros(cap, dtype=torch.float64, device=dev)
        prev = self.ctx.stream_handle
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)

        def _reduce(count, _user):
            dist.all_reduce(buf[:count], group=group)

        cb = api.ALLREDUCE_FN(_reduce)
        pb, mem, keep, is_t = _vec_args(b, self.n)
        if is_t:
            x = torch.zeros(self.n, dtype=torch.float64, device=b.device)
            px = C.c_void_p(x.data_ptr())
        else:
            x = np.zeros(self.n)
            px = _ptr(x)
        c = api.GmresConfig(cfg.restart, cfg.max_iters, cfg.rel_tol, 0, _ORTH[cfg.orth])
        rep = api.GmresReport()
        hcap = cfg.max_iters + 64
        hist = np.empty(hcap)
        st = api.Status()
        try:
            _check(api.lib().mscg_gmres_shard(self.ctx.h, self.h, rank, world, pb, px, mem,
                                              C.byref(c), C.c_void_p(buf.data_ptr()), cap, cb,
                                              None, C.byref(rep), _ptr(hist), hcap,
                                              C.byref(st)), st)
        finally:
            self.ctx.set_stream(prev if prev else None)
        return x, SolveReport(iterations=rep.iterations, converged=bool(rep.converged),
                              residual_history=hist[: rep.history_len].tolist(),
                              solve_seconds=rep.solve_seconds)

    def __del__(self):
        if getattr(self, "h", None):
            _destroy("mscg_precond_destroy", self.h)
            self.h = None


def build_preconditioner_shard(problem: Problem, block_begin: int, block_end: int,
                               tolA: float = 1e-4, sA: int = 400,
                               ctx: Context | None = None) -> PreconditionerShard:
    """Factor only the interior blocks [block_begin, block_end) (plus the
    replicated Schur blocks) on this rank's GPU."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    st = api.Status()
    _check(api.lib().mscg_precond_build_problem_shard(ctx.h, problem.h, tolA, sA, block_begin,
                                                      block_end, C.byref(h), C.byref(st)), st)
    return PreconditionerShard(ctx, h, block_begin, block_end)


def build_preconditioner_arrays(ctx: Context, c: SparseMatrix, p: int, d_ranges,
                                s_hat: SparseMatrix, s_ranges, tolA=1e-4, sA=400,
                                kind="msc") -> MscPreconditioner:
    """s_ranges None: S^ is an overlapped band, factored whole (one exact LU,
    the reference's schur_single_)."""
    rp, ci, v = c.arrays()
    srp, sci, sv = s_hat.arrays()
    dr = np.ascontiguousarray(np.asarray(d_ranges, np.int32).reshape(-1))
    single = s_ranges is None
    sr = np.ascontiguousarray(np.asarray([0, 0] if single else s_ranges, np.int32).reshape(-1))
    h = C.c_void_p()
    st = api.Status()
    _check(api.lib().mscg_precond_build(ctx.h, c.nrows, p, _ptr(rp), _ptr(ci), _ptr(v),
                                        len(dr) // 2, _ptr(dr), _ptr(srp), _ptr(sci), _ptr(sv),
                                        -1 if single else len(sr) // 2, _ptr(sr), tolA, sA,
                                        C.byref(h), C.byref(st)), st)
    return MscPreconditioner(ctx, h, kind, sA)


_ORTH = {"mgs": 0, "cgs2": 1, "dcgs2": 2}


@dataclass
class SolverConfig:
    restart: int = 300
    max_iters: int = 3000
    rel_tol: float = 1e-9
    side: str = "right"
    orth: str = "dcgs2"  # "dcgs2" (two basis sweeps), "cgs2" (three) or "mgs" (reference order)


@dataclass
class SolveReport:
    iterations: int = 0
    converged: bool = False
    residual_history: list = field(default_factory=list)
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    fill_factor: float = 0.0


def gmres(a: DeviceMatrix, b_precond: MscPreconditioner | None, rhs, cfg: SolverConfig,
          ctx: Context | None = None):
    """Restarted GMRES; returns (x, SolveReport)."""
    ctx = ctx or (b_precond.ctx if b_precond else a.ctx)
    n = a.nrows if a.nrows is not None else b_precond.n
    pb, mem, keep, is_t = _vec_args(rhs, n)
    if is_t:
        import torch
        x = torch.empty(n, dtype=torch.float64, device=rhs.device)
        px = C.c_void_p(x.data_ptr())
        torch.cuda.current_stream().synchronize()
    else:
        x = np.empty(n)
        px = _ptr(x)
    c = api.GmresConfig(cfg.restart, cfg.max_iters, cfg.rel_tol,
                        1 if cfg.side == "left" else 0, _ORTH[cfg.orth])
    rep = api.GmresReport()
    cap = cfg.max_iters + 64
    hist = np.empty(cap)
    st = api.Status()
    _check(api.lib().mscg_gmres(ctx.h, a.h, b_precond.h if b_precond else None, pb, px, mem,
                                C.byref(c), C.byref(rep), _ptr(hist), cap, C.byref(st)), st)
    r = SolveReport(iterations=rep.iterations, converged=bool(rep.converged),
                    residual_history=hist[: rep.history_len].tolist(),
                    solve_seconds=rep.solve_seconds)
    return x, r


def true_residual(a: DeviceMatrix, x, b, ctx: Context | None = None) -> float:
    ctx = ctx or a.ctx
    n = a.nrows
    px, mem, kx, _ = _vec_args(x, n)
    pb, mem2, kb, _ = _vec_args(b, n)
    if mem != mem2:
        raise ValueError("x and b must both be host arrays or both device tensors")
    out = C.c_double()
    st = api.Status()
    _check(api.lib().mscg_true_residual(ctx.h, a.h, px, pb, mem, C.byref(out), C.byref(st)), st)
    return out.value


def fill_factor(b: MscPreconditioner, c: SparseMatrix) -> float:
    return b.stored_nnz() / c.nnz


# ---- Matrix Market coordinate I/O (proj/include/msc/matrix_market.hpp:26-36)


def load_matrix_market(path) -> SparseMatrix:
    """Coordinate real/integer, general/symmetric/skew-symmetric; 1-based
    indices, duplicates summed, zeros dropped (reference
    load_matrix_market, matrix_market.cpp:20-90)."""
    p = os.fsencode(path)
    st = api.Status()
    nr, nc, nnz = C.c_int(), C.c_int(), C.c_int64()
    _check(api.lib().mscg_mm_read(p, C.byref(nr), C.byref(nc), C.byref(nnz), None, None,
                                  None, C.byref(st)), st)
    rp = np.empty(nr.value + 1, np.int32)
    ci = np.empty(max(1, nnz.value), np.int32)
    v = np.empty(max(1, nnz.value))
    _check(api.lib().mscg_mm_read(p, C.byref(nr), C.byref(nc), C.byref(nnz), _ptr(rp),
                                  _ptr(ci), _ptr(v), C.byref(st)), st)
    return SparseMatrix(nr.value, nc.value, rp, ci[:nnz.value].copy(), v[:nnz.value].copy())


def write_matrix_market(path, a: SparseMatrix) -> None:
    """General coordinate file, 17 significant digits (matrix_market.cpp:92-110)."""
    rp, ci, v = a.arrays()
    st = api.Status()
    _check(api.lib().mscg_mm_write(os.fsencode(path), a.nrows, a.ncols, _ptr(rp), _ptr(ci),
                                   _ptr(v), C.byref(st)), st)


def load_vector_market(path) -> np.ndarray:
    p = os.fsencode(path)
    st = api.Status()
    n = C.c_int()
    _check(api.lib().mscg_mm_read_vector(p, C.byref(n), None, C.byref(st)), st)
    out = np.empty(n.value)
    _check(api.lib().mscg_mm_read_vector(p, C.byref(n), _ptr(out), C.byref(st)), st)
    return out


def write_vector_market(path, v) -> None:
    v = np.ascontiguousarray(v, np.float64)
    st = api.Status()
    _check(api.lib().mscg_mm_write_vector(os.fsencode(path), len(v), _ptr(v), C.byref(st)), st)
