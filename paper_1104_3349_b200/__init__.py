"""B200-native solve phase of the mini-Schur-complement DD preconditioner
(arXiv:1104.3349): C-ABI library libmscg.so (hand-written sm_100a kernels)
plus a Python mirror of the reference's C++ API."""
from .msc import (  # noqa: F401
    Context,
    CudaError,
    DeviceMatrix,
    MscError,
    MscPreconditioner,
    PreconditionerShard,
    Problem,
    SingularMatrixError,
    SolveReport,
    SolverConfig,
    SparseMatrix,
    TriangularFactors,
    build_preconditioner,
    build_preconditioner_arrays,
    build_preconditioner_shard,
    default_context,
    fill_factor,
    gmres,
    matvec,
    oseen_problem,
    partitioned_problem,
    true_residual,
)

__all__ = [n for n in dir() if not n.startswith("_")]
