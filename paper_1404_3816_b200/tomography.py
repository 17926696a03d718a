"""Crosswell straight-ray operator (input producer of the hot path).

Mirror of the reference tomography.py:20-133 (Acquisition,
default_acquisition, build_ray_operator): the ray/cell intersection tracing
runs in native C++ inside libhikf_b200.so (hikf_ray_operator), reproducing
the reference's breakpoint, midpoint and grazing-ray rules so the CSR pattern
is bit-identical (tests/test_gpu_parity.py, test_boundary.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse

from . import _lib


@dataclass(frozen=True)
class Acquisition:
    sources: np.ndarray = field(repr=False)
    receivers: np.ndarray = field(repr=False)

    def __post_init__(self):
        for name in ("sources", "receivers"):
            arr = np.asarray(getattr(self, name), dtype=float)
            if arr.ndim != 2 or arr.shape[1] != 2 or arr.shape[0] < 1:
                raise ValueError(f"{name} must have shape (k, 2) with k >= 1")
            object.__setattr__(self, name, arr)

    @property
    def n(self) -> int:
        return len(self.sources) * len(self.receivers)

    def ray_endpoints(self):
        """(n, 2) sources and receivers, source-major (tomography.py:38-43)."""
        nr = len(self.receivers)
        return np.repeat(self.sources, nr, axis=0), np.tile(self.receivers, (len(self.sources), 1))


def default_acquisition(grid, n_sources=6, n_receivers=48, source_x=None, receiver_x=None) -> Acquisition:
    """Vertical wells with uniformly spaced stations (tomography.py:46-73)."""
    xmin, xmax, ymin, ymax = grid.extent
    if source_x is None:
        source_x = xmin + 0.5 * grid.dx
    if receiver_x is None:
        receiver_x = xmax - 0.5 * grid.dx
    for x in (source_x, receiver_x):
        if not (xmin <= x <= xmax):
            raise ValueError("well x position lies outside the grid")

    def stations(k):
        return ymin + (np.arange(k) + 0.5) * (ymax - ymin) / k

    src = np.column_stack([np.full(n_sources, source_x), stations(n_sources)])
    rcv = np.column_stack([np.full(n_receivers, receiver_x), stations(n_receivers)])
    return Acquisition(src, rcv)


def build_ray_operator(grid, acq) -> scipy.sparse.csr_matrix:
    """Sparse (n, m) matrix of exact ray-cell intersection lengths."""
    src, rcv = acq.ray_endpoints()
    src = np.ascontiguousarray(src, dtype=float)
    rcv = np.ascontiguousarray(rcv, dtype=float)
    n = src.shape[0]
    x0, y0 = grid.origin
    lib = _lib.load()
    nnz = ctypes.c_int64(0)
    args = (grid.nx, grid.ny, float(grid.dx), float(grid.dy), float(x0), float(y0), n, src.ctypes.data, rcv.ctypes.data)
    _lib.check(lib.hikf_ray_operator(*args, None, None, None, ctypes.byref(nnz)))
    indptr = np.zeros(n + 1, dtype=np.int32)
    indices = np.zeros(nnz.value, dtype=np.int32)
    data = np.zeros(nnz.value, dtype=np.float64)
    _lib.check(lib.hikf_ray_operator(*args, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data,
                                     ctypes.byref(nnz)))
    return scipy.sparse.csr_matrix((data, indices, indptr), shape=(n, grid.m))
