"""B200-native HiKF hot path (arXiv:1404.3816): bbFMM Q H^T + the per-step
cross-covariance Kalman update, as hand-written sm_100a FP64 kernels behind
the reference ``hikf`` package's own Python API.

Drop-in surface (reference hikf/__init__.py:10-26 and hikf.filters):
    KernelSpec, Grid2D, PointSet, FmmConfig, FmmTree, build_tree,
    DecompositionError, spd_solve, filters.{hikf_precompute_fmm, hikf_init,
    hikf_predict, hikf_update, HikfState, HikfPrecompute,
    NumericalConsistencyError}
"""

from ._lib import DecompositionError, NumericalConsistencyError
from .fmm import FmmConfig, FmmTree, build_tree
from .grids import Grid2D, PointSet
from .kernels import KernelSpec, value_at_zero
from .linalg import spd_solve
from . import experiment, filters, space3d, tomography


__all__ = [
    "KernelSpec", "value_at_zero", "Grid2D", "PointSet", "FmmConfig", "FmmTree", "build_tree",
    "DecompositionError", "NumericalConsistencyError", "spd_solve", "filters", "tomography", "experiment", "space3d",
]

__version__ = "0.1.0"
