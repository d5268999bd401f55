"""B200-native MLMC random-walk estimator for e^{tA}v (hot path of arXiv 1904.12754).

The compute path is the in-tree CUDA library ``_lib/libexpmc_b200.so`` (sm_100a) behind the
C-ABI ``include/expmc_b200.h``; this package is its Python host mirror of the reference's
C++ API (``api``) plus the synthetic config inputs (``configs``).  Importing it fails loudly
when the library has not been built: there is no CPU fallback.
"""
from .api import (  # noqa: F401
    Context,
    CudaError,
    DomainError,
    ExpmcError,
    InvalidArgument,
    IoError,
    LANE_ENTRY,
    LANE_FEM,
    LANE_FORWARD,
    LevelStats,
    MlmcOptions,
    MlmcProblem,
    MlmcResult,
    NotImplementedMode,
    OutOfRange,
    SampleMode,
    SparseMatrix,
    bench_gather,
    nccl_unique_id,
    bias_estimate,
    device_count,
    initial_level,
    McResult,
    mc_auto,
    mc_batch,
    mc_forward_scalar,
    mc_single_entry,
    load_fem_system,
    read_matrix_market,
    read_vector,
    mlmc_driver,
    FemSystem,
    fem_context,
    mlmc_driver_fem,
    mlmc_driver_forward,
    solve_convdiff_point,
    node_communicability,
    spectral_scale,
    total_communicability,
    mlmc_driver_rows,
    optimal_allocation,
    run_level,
    version,
)

__version__ = "0.1.0"
