"""Crosswell straight-ray operator (input producer of the hot path).

Mirror of the reference tomography.py:20-133 (Acquisition,
default_acquisition, build_ray_operator): the ray/cell intersection tracing
runs in native C++ inside libhikf_b200.so (hikf_ray_operator), or on the GPU
(hikf_ray_operator_device: one CTA per ray, the result stays in HBM),
reproducing the reference's breakpoint, midpoint and grazing-ray rules so the
CSR pattern and lengths are bit-identical (tests/test_gpu_parity.py,
test_boundary.py).
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


def build_ray_operator_device(grid, acq):
    """build_ray_operator traced on the GPU; returns a filters.DeviceCSR in HBM
    that hikf_precompute_fmm / hikf_update accept wherever they take H."""
    import torch

    from .filters import DeviceCSR, _dev
    src, rcv = acq.ray_endpoints()
    src = np.ascontiguousarray(src, dtype=float)
    rcv = np.ascontiguousarray(rcv, dtype=float)
    n = src.shape[0]
    x0, y0 = grid.origin
    lib = _lib.load()
    dev = _dev()
    indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    cap = n * (grid.nx + grid.ny)  # a ray crosses at most nx + ny - 1 cells
    indices = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    data = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
    nnz = ctypes.c_int64(0)
    _lib.check(lib.hikf_ray_operator_device(grid.nx, grid.ny, float(grid.dx), float(grid.dy), float(x0), float(y0), n,
                                            src.ctypes.data, rcv.ctypes.data, indptr.data_ptr(), indices.data_ptr(),
                                            data.data_ptr(), cap, ctypes.byref(nnz), _lib.stream_ptr()))
    k = nnz.value
    return DeviceCSR.from_device(indptr, indices[:k].clone(), data[:k].clone(), (n, grid.m))
