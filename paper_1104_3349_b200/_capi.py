"""ctypes binding of include/mscg.h (libmscg.so, built in-tree for sm_100a)."""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
# MSCG_LIB: an alternate in-tree build of the same library (A/B measurements)
LIB_PATH = os.environ.get("MSCG_LIB") or os.path.join(PKG, "libmscg.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "mscg.h")

MSCG_OK = 0
MSCG_ERR_INVALID_ARGUMENT = 1
MSCG_ERR_SINGULAR = 2
MSCG_ERR_CUDA = 3
MSCG_ERR_OUT_OF_MEMORY = 4
MSCG_ERR_RUNTIME = 5
MSCG_ERR_IO = 6
MEM_HOST = 0
MEM_DEVICE = 1

vp = C.c_void_p
ip = C.POINTER(C.c_int)
i64p = C.POINTER(C.c_int64)
dp = C.POINTER(C.c_double)


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("block", C.c_int), ("pivot_index", C.c_int),
                ("message", C.c_char * 512)]


class GmresConfig(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iters", C.c_int), ("rel_tol", C.c_double),
                ("side", C.c_int), ("orth", C.c_int)]


ALLREDUCE_FN = C.CFUNCTYPE(None, C.c_int, C.c_void_p)


class GmresReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("history_len", C.c_int),
                ("history_total", C.c_int), ("solve_seconds", C.c_double),
                ("final_true_residual", C.c_double)]


_SIGS = {
    "mscg_abi_version": (C.c_int, []),
    "mscg_mm_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_int64), vp, vp, vp, C.POINTER(Status)]),
    "mscg_mm_write": (C.c_int, [C.c_char_p, C.c_int, C.c_int, vp, vp, vp, C.POINTER(Status)]),
    "mscg_mm_read_vector": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), vp, C.POINTER(Status)]),
    "mscg_mm_write_vector": (C.c_int, [C.c_char_p, C.c_int, vp, C.POINTER(Status)]),
    "mscg_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp), C.POINTER(Status)]),
    "mscg_ctx_destroy": (None, [vp]),
    "mscg_ctx_stream": (vp, [vp]),
    "mscg_ctx_synchronize": (C.c_int, [vp, C.POINTER(Status)]),
    "mscg_ctx_set_stream": (C.c_int, [vp, vp, C.c_int, C.POINTER(Status)]),
    "mscg_ctx_launches": (C.c_int64, [vp]),
    "mscg_ctx_set_correction": (C.c_int, [vp, C.c_int, C.POINTER(Status)]),
    "mscg_problem_oseen": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_double, C.c_int,
                                     C.c_int, C.c_int, C.POINTER(vp), C.POINTER(Status)]),
    "mscg_problem_oseen_device": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, C.c_double,
                                            C.c_int, C.c_int, C.c_int, C.POINTER(vp),
                                            C.POINTER(Status)]),
    "mscg_problem_from_csr": (C.c_int, [C.c_int, vp, vp, vp, C.c_int, C.c_int, vp,
                                        C.POINTER(vp), C.POINTER(Status)]),
    "mscg_problem_destroy": (None, [vp]),
    "mscg_problem_dims": (None, [vp, ip, ip, ip, i64p, ip]),
    "mscg_problem_csr": (C.c_int, [vp, C.c_int, ip, ip, i64p, C.POINTER(ip), C.POINTER(ip),
                                   C.POINTER(dp)]),
    "mscg_problem_perm": (ip, [vp]),
    "mscg_problem_d_ranges": (ip, [vp]),
    "mscg_problem_scaled_rhs": (dp, [vp]),
    "mscg_problem_build_schur_device": (C.c_int, [vp, vp, C.c_char_p, C.c_int, C.c_int,
                                                  C.c_int, vp, C.POINTER(Status)]),
    "mscg_problem_build_schur": (C.c_int, [vp, C.c_char_p, C.c_int, C.c_int, C.c_int, vp,
                                           C.c_int, C.POINTER(Status)]),
    "mscg_problem_build_schur_overlapped": (C.c_int, [vp, vp, C.c_char_p, C.c_int, C.c_int,
                                                      C.c_int, vp, C.c_int, C.c_int, vp,
                                                      C.c_int, C.POINTER(Status)]),
    "mscg_problem_num_aggregates": (C.c_int, [vp]),
    "mscg_problem_schur_ranges": (ip, [vp]),
    "mscg_csr_upload": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, C.POINTER(vp),
                                  C.POINTER(Status)]),
    "mscg_csr_destroy": (None, [vp]),
    "mscg_spmv": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(Status)]),
    "mscg_precond_build": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, C.c_int, vp, vp, vp, vp,
                                     C.c_int, vp, C.c_double, C.c_int, C.POINTER(vp),
                                     C.POINTER(Status)]),
    "mscg_precond_build_problem": (C.c_int, [vp, vp, C.c_double, C.c_int, C.POINTER(vp),
                                             C.POINTER(Status)]),
    "mscg_precond_build_shard": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, C.c_int, vp, vp,
                                           vp, vp, C.c_int, vp, C.c_double, C.c_int, C.c_int,
                                           C.c_int, C.POINTER(vp), C.POINTER(Status)]),
    "mscg_precond_build_problem_shard": (C.c_int, [vp, vp, C.c_double, C.c_int, C.c_int,
                                                   C.c_int, C.POINTER(vp), C.POINTER(Status)]),
    "mscg_precond_shard_rows": (C.c_int, [vp, ip, ip]),
    "mscg_precond_apply_shard": (C.c_int, [vp, C.c_int, vp, vp, vp, C.POINTER(Status)]),
    "mscg_precond_spmv_shard": (C.c_int, [vp, vp, vp, vp, C.c_int, C.POINTER(Status)]),
    "mscg_precond_destroy": (None, [vp]),
    "mscg_precond_apply": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(Status)]),
    "mscg_precond_apply_stream": (C.c_int, [vp, vp, vp, vp, C.POINTER(Status)]),
    "mscg_precond_stored_nnz": (C.c_int64, [vp]),
    "mscg_precond_dims": (C.c_int, [vp, ip, ip, ip, ip]),
    "mscg_precond_factor": (C.c_int, [vp, C.c_int, C.c_int, ip, i64p, i64p, vp, vp, vp, vp, vp,
                                      vp, vp, C.POINTER(Status)]),
    "mscg_precond_build_times": (C.c_int, [vp, dp, dp, dp]),
    "mscg_factor": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_int, C.c_double, C.POINTER(vp),
                              C.POINTER(Status)]),
    "mscg_factors_get": (C.c_int, [vp, ip, i64p, i64p, vp, vp, vp, vp, vp, vp, vp,
                                   C.POINTER(Status)]),
    "mscg_factors_solve": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(Status)]),
    "mscg_factors_destroy": (None, [vp]),
    "mscg_precond_correction": (C.c_int, [vp, ip, i64p, ip, dp]),
    "mscg_precond_matrix": (vp, [vp]),
    "mscg_gmres": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, C.POINTER(GmresConfig),
                             C.POINTER(GmresReport), vp, C.c_int, C.POINTER(Status)]),
    "mscg_gmres_shard": (C.c_int, [vp, vp, C.c_int, C.c_int, vp, vp, C.c_int,
                                   C.POINTER(GmresConfig), vp, C.c_int, vp, vp,
                                   C.POINTER(GmresReport), vp, C.c_int, C.POINTER(Status)]),
    "mscg_nested_dissection": (C.c_int, [vp, C.c_int, vp, vp, C.c_int, C.c_int, vp,
                                         C.POINTER(C.c_int), vp, C.c_int, C.POINTER(Status)]),
    "mscg_precond_nnz": (C.c_int, [vp, C.POINTER(C.c_int64)]),
    "mscg_precond_use_correction": (C.c_int, [vp, C.c_int]),
    "mscg_precond_layout_bytes": (C.c_int, [vp, C.POINTER(C.c_int64)]),
    "mscg_random_vector": (None, [C.c_int, C.c_uint, vp]),
    "mscg_bench_apply": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, dp, dp, i64p,
                                   C.POINTER(Status)]),
    "mscg_debug_trace_dsolve": (C.c_int, [vp, vp, vp, vp, C.c_int, C.POINTER(Status)]),
    "mscg_true_residual": (C.c_int, [vp, vp, vp, vp, C.c_int, dp, C.POINTER(Status)]),
}

_lib = None


def declared_symbols() -> list[str]:
    """Function names declared in include/mscg.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mscg_[a-z0-9_]+)\s*\(", src)))


def lib():
    """Load libmscg.so; raise loudly if it was not built (there is no
    fallback implementation)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1104_3349_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
