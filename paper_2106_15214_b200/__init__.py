"""B200-native beta-NMF (joint-MM and block MU) -- drop-in for the solver
entry points of the reference ``betanmf`` package (arXiv 2106.15214).

    import paper_2106_15214_b200 as betanmf
    res = betanmf.fit(V, betanmf.SolverConfig(beta=1, rank=49, algorithm="jmm"))

The per-iteration work runs in libbnmf.so (CUDA, sm_100a); there is no CPU
fallback.  See DESIGN.md and INTEGRATION.md.
"""

from .core import (
    DEFAULT_FLOOR,
    BetaParam,
    DataMatrix,
    DivergenceDomainError,
    FactorPair,
    beta_divergence,
    default_kappa,
    gamma_exponent,
)
from .solver import (
    FitResult,
    SolverConfig,
    Termination,
    TraceRow,
    fit,
    get_context,
    init_factors,
    normalize,
    run_bmm,
    run_jmm,
    should_stop,
    synthetic_low_rank,
)
from .updates import Algorithm, OpCounter, UpdateKind
from .kernels import (
    KktResiduals,
    MajorizerAnchor,
    bmm_update_h,
    bmm_update_w,
    jmm_update_h,
    jmm_update_w,
    kkt_residuals,
    objective,
)
from .harness import BenchReport, format_report, match_columns, run_bench, summarize
from .matrixio import load_matrix, load_sparse, save_factors, save_trace
from . import parallel  # noqa: F401  (N-column sharding helpers)
from . import harness, matrixio  # noqa: F401  (multi-seed harness, matrix IO; cli.py uses both)

__version__ = "0.1.0"

__all__ = [
    "Algorithm",
    "BenchReport",
    "BetaParam",
    "DEFAULT_FLOOR",
    "DataMatrix",
    "DivergenceDomainError",
    "FactorPair",
    "FitResult",
    "KktResiduals",
    "MajorizerAnchor",
    "OpCounter",
    "SolverConfig",
    "Termination",
    "TraceRow",
    "UpdateKind",
    "beta_divergence",
    "bmm_update_h",
    "bmm_update_w",
    "default_kappa",
    "fit",
    "format_report",
    "gamma_exponent",
    "get_context",
    "init_factors",
    "jmm_update_h",
    "jmm_update_w",
    "kkt_residuals",
    "load_matrix",
    "load_sparse",
    "match_columns",
    "normalize",
    "objective",
    "run_bench",
    "run_bmm",
    "run_jmm",
    "save_factors",
    "save_trace",
    "should_stop",
    "summarize",
    "synthetic_low_rank",
]
