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


def warmup() -> None:
    """Load the library's device code and prime its memory pool with one tiny
    tree + Q H^T + two updates (~0.1 s).  Optional: without it the first real call
    pays CUDA's lazy kernel loading (cfg4 tree + Q H^T: ~0.1 s after warm-up,
    0.16-0.23 s cold)."""
    import numpy as np

    grid = Grid2D(32, 32, 1.0 / 32, 1.0 / 32)
    H = tomography.build_ray_operator(grid, tomography.default_acquisition(grid, 4, 4, 0.0, 1.0))

    class _Model:
        pass

    model = _Model()
    model.H, model.m, model.alpha, model.initial_mean = H, grid.m, 0.0, np.zeros(grid.m)
    tree = build_tree(grid.cell_centers(), KernelSpec("exponential", variance=1.0, length_scale=0.3),
                      FmmConfig(n_cheb=6, max_leaf_points=16))
    pre = filters.hikf_precompute_fmm(model, tree)
    st = filters.hikf_init(model)
    for _ in range(2):
        st = filters.hikf_update(filters.hikf_predict(st, pre), H, 1e-3, np.zeros(H.shape[0]))
    st.mean  # noqa: B018  (resolves the deferred statuses)


__all__ = [
    "KernelSpec", "value_at_zero", "Grid2D", "PointSet", "FmmConfig", "FmmTree", "build_tree",
    "DecompositionError", "NumericalConsistencyError", "spd_solve", "filters", "tomography", "experiment", "space3d",
    "warmup",
]

__version__ = "0.1.0"
