"""B200-native solve phase of the mini-Schur-complement DD preconditioner
(arXiv:1104.3349): C-ABI library libmscg.so (hand-written sm_100a kernels)
plus a Python mirror of the reference's C++ API."""
from .msc import (  # noqa: F401
    Context,
    CudaError,
    DeviceFactors,
    DeviceMatrix,
    IoError,
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
    factor_exact,
    factor_ilut,
    fill_factor,
    gmres,
    load_matrix_market,
    load_vector_market,
    matvec,
    nested_dissection,
    oseen_problem,
    partitioned_problem,
    true_residual,
    write_matrix_market,
    write_vector_market,
)

__all__ = [n for n in dir() if not n.startswith("_")]
