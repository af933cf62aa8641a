"""B200-native hot path of the sketched long-step IPM (arXiv 2209.08722).

Drop-in for the reference package `skipm`'s solver API on the data-parallel
path: sketch (hash + ADW) -> CholeskyQR2 preconditioner -> PCG on
A D^2 A' dy = p -> correction v and fused step kernels, all on the GPU
(hand-written sm_100a CUDA in csrc/, C ABI in include/skb.h). There is no
CPU fallback: without the built libskb.so or a CUDA device, calls raise.
"""

from .errors import (  # noqa: F401
    Breakdown,
    DegenerateRow,
    DimensionMismatch,
    EmptyDataset,
    Infeasible,
    InvalidDensity,
    InvalidDims,
    InvalidZeta,
    InvariantViolated,
    MaxIterations,
    NeighborhoodViolated,
    NonpositivePoint,
    NonpositiveScaling,
    NotPositiveDefinite,
    ParseError,
    RankDeficient,
    Singular,
    SkipmError,
    StaleFactor,
    TooLarge,
    TooLargeForDiagnostic,
    Unbounded,
    ZeroRow,
)
from .lp_model import (  # noqa: F401
    DeviceLP,
    LinearProgram,
    make_lp,
    random_feasible_lp,
    random_lp,
    validate,
)

__version__ = "0.1.0"

_LAZY = {
    "IpmIterate": "ipm_core", "IpmParams": "ipm_core", "SolveReport": "ipm_core",
    "StepRecord": "ipm_core", "default_start": "ipm_core", "duality_measure": "ipm_core",
    "feasible_start": "ipm_core", "in_neighborhood": "ipm_core", "make_iterate": "ipm_core",
    "phase1_point": "ipm_core", "solve": "ipm_core", "ipm_step": "ipm_core",
    "NormalOperator": "krylov_solvers", "pcg": "krylov_solvers", "SolverTrace": "krylov_solvers",
    "chebyshev": "krylov_solvers", "direct_solve": "krylov_solvers",
    "unpreconditioned_cg": "krylov_solvers", "phase1_lp": "start",
    "build_preconditioner": "preconditioning", "apply_inv": "preconditioning",
    "apply_pinv_adw": "preconditioning", "PreconditionerFactor": "preconditioning",
    "SketchOperator": "sketching", "auto_sketch_dims": "sketching",
    "build_sparse_embedding": "sketching", "build_identity_sketch": "sketching",
    "build_gaussian_sketch": "sketching", "apply_sketch": "sketching",
    "compute_v": "correction", "check_v_norm": "correction",
    "check_v_small_enough": "correction", "CorrectionVector": "correction",
    "SvmDataset": "ingest", "SvmLpMapping": "ingest", "svm_to_lp": "ingest",
    "extract_svm_solution": "ingest", "load_libsvm": "ingest", "save_matrix_market": "ingest",
    "load_matrix_market": "ingest", "to_device": "ingest",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f"{__name__}.{mod}"), name)
