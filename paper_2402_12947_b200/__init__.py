"""B200-native combined-smoother hot path for arXiv 2402.12947 (`simplexmg`).

Drop-in for the reference's smoother/solver API (pkg/src/simplexmg):

    from paper_2402_12947_b200 import (combined_smooth, chebyshev_smooth,
        apply_local_correction, vcycle, solve_stationary, as_preconditioner, cg)

The arithmetic runs in the in-tree sm_100a library
``paper_2402_12947_b200/lib/libsimplexmg_b200.so`` (C-ABI:
include/simplexmg_b200.h) -- there is no CPU fallback.  Reference objects
(``simplexmg.mg.Hierarchy``, ``CsrMatrix``, ``LocalCorrection``,
``SmootherConfig``) are accepted as they are.
"""

from .sparse import (CsrMatrix, DenseFactor, EigenEstimateError, IndefiniteOperatorError,
                     NotPositiveDefiniteError, cg, dense_factor, dot, estimate_lambda_max,
                     spmv, transpose, triple_product)
from .smoothers import (LocalCorrection, SmootherConfig, ZeroDiagonalError,
                        adjusted_lambda_max, apply_local_correction, build_local_correction,
                        chebyshev_smooth, combined_smooth, dofs_for_regions, jacobi_lambda_max,
                        sgs_sweep)
from .mg import (DeviceHierarchy, Hierarchy, Level, ProblemSpec, Prolongation,
                 as_preconditioner, build_hierarchy, solve_stationary, vcycle)
from .transfer import PointLocationError, locate_point, prolong_add, restrict_residual

__all__ = [
    "CsrMatrix", "DenseFactor", "EigenEstimateError", "IndefiniteOperatorError",
    "NotPositiveDefiniteError", "cg", "dense_factor", "dot", "estimate_lambda_max", "spmv",
    "transpose", "triple_product", "LocalCorrection", "SmootherConfig", "ZeroDiagonalError",
    "adjusted_lambda_max", "apply_local_correction", "build_local_correction",
    "chebyshev_smooth", "combined_smooth", "dofs_for_regions", "jacobi_lambda_max", "sgs_sweep",
    "DeviceHierarchy", "Hierarchy", "Level", "Prolongation", "as_preconditioner",
    "build_hierarchy", "solve_stationary", "vcycle", "ProblemSpec", "PointLocationError",
    "locate_point", "prolong_add", "restrict_residual",
]
