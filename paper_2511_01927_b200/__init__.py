"""B200-native CIRR contour-integral stage (drop-in for cieig.solvers).

The hot path of DeepContour's CI solve (arxiv 2511.01927): pencil assembly,
batched complex-FP64 LU on the DMMA tensor pipe, multi-RHS solves with the
quadrature moments, rank-revealing orthonormalisation, projected pencil and
small eigensolver -- hand-written sm_100a kernels in libcirr.so behind the
reference's Python API.  See DESIGN.md and include/cirr.h.
"""

from .contours import Contour, QuadratureRule, contours_from_json, contours_to_json, quadrature_for  # noqa: F401
from .errors import (  # noqa: F401
    CieigError,
    ConvergenceError,
    CutUndefinedError,
    DeviceError,
    DimensionError,
    EmptyPredictionError,
    FormatError,
    IndefiniteBError,
    NoEigenvaluesFound,
    ParameterError,
    ParameterWarning,
    RankZeroError,
    SingularShiftError,
)
from .solvers import (  # noqa: F401
    DevicePencil,
    EigenResult,
    MultiResult,
    ProjectorContext,
    SolverConfig,
    SolveStats,
    apply_projector,
    cirr_solve,
    feast_solve,
    read_eigenvectors,
    solve_multi,
    solve_multi_batch,
    write_eigenvectors,
)

from .kde import kde_eval  # noqa: F401
from .scouting import SCOUT_METHODS, RitzEstimate, calibrate_margin, scout, scout_contour  # noqa: F401

__version__ = "0.1.0"
