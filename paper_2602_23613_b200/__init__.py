"""B200-native AMG-PCG hot path for lowest-order Nedelec H(curl) systems
(arXiv 2602.23613): a drop-in for ``hcurl_amg.multilevel`` whose setup and
solve run as sm_100a CUDA kernels behind the C-ABI in ``include/hcamg.h``."""

from .multilevel import (Hierarchy, Level, SolveReport, amg_solve, build_hierarchy, operator_complexity, pcg,
                         vcycle)
from .sparse import NotPositiveDefiniteError, cholesky, csr, solve
from . import smoothers
from ._lib import NativeUnavailable

__all__ = ["Hierarchy", "Level", "SolveReport", "amg_solve", "build_hierarchy", "operator_complexity", "pcg",
           "vcycle", "NotPositiveDefiniteError", "cholesky", "csr", "solve", "NativeUnavailable"]
