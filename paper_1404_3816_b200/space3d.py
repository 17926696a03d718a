"""3D scenario pieces for BASELINE cfg3 / cfg5.

PARITY UNPINNED: the reference ``hikf`` package is 2D and isotropic only, so
there is no reference output here.  Every rule is the direct 3D extension of
the reference's 2D one and is restated, and checked against exact algebra, in
oracle/hikf_oracle3d.py; the CUDA path is tested against that oracle
(tests/test_gpu_3d.py).

* ``Grid3D``: cells x fastest, then y, then z.
* ``crosswell_3d``: seeded jittered stations on the x = xmin / xmax faces,
  rays source-major.
* ``build_ray_operator_3d`` (host) / ``build_ray_operator_3d_device`` (GPU):
  exact ray / voxel intersection lengths, bit-identical to each other and to
  the oracle.
* ``KernelSpec3``: variance exp(-|(dx/lx, dy/ly, dz/lz)|^p), p = 2 (gaussian)
  or 1 (exponential).
* ``build_tree3d`` / ``FmmTree3D``: the octree bbFMM (csrc/fmm3d.cu);
  ``filters.hikf_precompute_fmm`` accepts it in place of a 2D tree.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse

from . import _lib


@dataclass(frozen=True)
class Grid3D:
    nx: int
    ny: int
    nz: int
    dx: float = 1.0
    dy: float = 1.0
    dz: float = 1.0
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise ValueError("nx, ny and nz must be positive")
        if not (self.dx > 0 and self.dy > 0 and self.dz > 0):
            raise ValueError("dx, dy and dz must be positive")

    @property
    def m(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def extent(self):
        x0, y0, z0 = self.origin
        return (x0, x0 + self.nx * self.dx, y0, y0 + self.ny * self.dy, z0, z0 + self.nz * self.dz)

    def cell_centers(self) -> "PointSet3":
        x0, y0, z0 = self.origin
        xs = x0 + (np.arange(self.nx) + 0.5) * self.dx
        ys = y0 + (np.arange(self.ny) + 0.5) * self.dy
        zs = z0 + (np.arange(self.nz) + 0.5) * self.dz
        nx, ny, nz = self.nx, self.ny, self.nz
        return PointSet3(np.column_stack([np.tile(xs, ny * nz), np.tile(np.repeat(ys, nx), nz),
                                          np.repeat(zs, nx * ny)]))


@dataclass(frozen=True)
class PointSet3:
    coords: np.ndarray = field(repr=False)

    def __post_init__(self):
        c = np.asarray(self.coords, dtype=float)
        if c.ndim != 2 or c.shape[1] != 3 or c.shape[0] < 1:
            raise ValueError("coords must have shape (m, 3) with m >= 1")
        if not np.all(np.isfinite(c)):
            raise ValueError("coordinates must be finite")
        object.__setattr__(self, "coords", c)

    def __len__(self) -> int:
        return self.coords.shape[0]


@dataclass(frozen=True)
class Acquisition3D:
    sources: np.ndarray = field(repr=False)
    receivers: np.ndarray = field(repr=False)

    def __post_init__(self):
        for name in ("sources", "receivers"):
            a = np.asarray(getattr(self, name), dtype=float)
            if a.ndim != 2 or a.shape[1] != 3 or a.shape[0] < 1:
                raise ValueError(f"{name} must have shape (k, 3) with k >= 1")
            object.__setattr__(self, name, a)

    @property
    def n(self) -> int:
        return len(self.sources) * len(self.receivers)

    def ray_endpoints(self):
        nr = len(self.receivers)
        return np.repeat(self.sources, nr, axis=0), np.tile(self.receivers, (len(self.sources), 1))


def face_stations(k: int, x: float, ylo: float, yhi: float, zlo: float, zhi: float, seed) -> np.ndarray:
    """k stations on x = const, one per cell of the first k cells (y fastest) of
    an a x b lattice (a = ceil(sqrt k), b = ceil(k / a)), jittered uniformly
    inside the cell with PCG64(seed)."""
    a = int(math.ceil(math.sqrt(k)))
    b = int(math.ceil(k / a))
    u = np.random.default_rng(seed).random((a * b, 2))
    idx = np.arange(a * b)
    y = ylo + (idx % a + u[:, 0]) * ((yhi - ylo) / a)
    z = zlo + (idx // a + u[:, 1]) * ((zhi - zlo) / b)
    return np.column_stack([np.full(a * b, float(x)), y, z])[:k]


def crosswell_3d(grid: Grid3D, n_sources: int, n_receivers: int, seed: int) -> Acquisition3D:
    x0, x1, y0, y1, z0, z1 = grid.extent
    return Acquisition3D(face_stations(n_sources, x0, y0, y1, z0, z1, [seed, 1]),
                         face_stations(n_receivers, x1, y0, y1, z0, z1, [seed, 2]))


def _grid_args(grid: Grid3D):
    n3 = (ctypes.c_int64 * 3)(grid.nx, grid.ny, grid.nz)
    d3 = (ctypes.c_double * 3)(grid.dx, grid.dy, grid.dz)
    o3 = (ctypes.c_double * 3)(*[float(v) for v in grid.origin])
    return n3, d3, o3


def build_ray_operator_3d(grid: Grid3D, acq: Acquisition3D) -> scipy.sparse.csr_matrix:
    src, rcv = (np.ascontiguousarray(a, dtype=float) for a in acq.ray_endpoints())
    n = src.shape[0]
    n3, d3, o3 = _grid_args(grid)
    lib = _lib.load()
    nnz = ctypes.c_int64(0)
    _lib.check(lib.hikf_ray_operator_3d(n3, d3, o3, n, src.ctypes.data, rcv.ctypes.data, None, None, None,
                                        ctypes.byref(nnz)))
    indptr = np.zeros(n + 1, dtype=np.int32)
    indices = np.zeros(nnz.value, dtype=np.int32)
    data = np.zeros(nnz.value, dtype=np.float64)
    _lib.check(lib.hikf_ray_operator_3d(n3, d3, o3, n, src.ctypes.data, rcv.ctypes.data, indptr.ctypes.data,
                                        indices.ctypes.data, data.ctypes.data, ctypes.byref(nnz)))
    return scipy.sparse.csr_matrix((data, indices, indptr), shape=(n, grid.m))


def build_ray_operator_3d_device(grid: Grid3D, acq: Acquisition3D):
    import torch

    from .filters import DeviceCSR, _dev
    src, rcv = (np.ascontiguousarray(a, dtype=float) for a in acq.ray_endpoints())
    n = src.shape[0]
    n3, d3, o3 = _grid_args(grid)
    dev = _dev()
    cap = n * (grid.nx + grid.ny + grid.nz)
    indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    indices = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    data = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
    nnz = ctypes.c_int64(0)
    _lib.check(_lib.load().hikf_ray_operator_3d_device(n3, d3, o3, n, src.ctypes.data, rcv.ctypes.data,
                                                       indptr.data_ptr(), indices.data_ptr(), data.data_ptr(), cap,
                                                       ctypes.byref(nnz), _lib.stream_ptr()))
    k = nnz.value
    return DeviceCSR.from_device(indptr, indices[:k].clone(), data[:k].clone(), (n, grid.m))


@dataclass(frozen=True)
class KernelSpec3:
    family: str
    variance: float = 1.0
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0

    def __post_init__(self):
        if self.family not in ("gaussian", "exponential"):
            raise ValueError("3D kernels: family must be 'gaussian' or 'exponential'")
        if not self.variance >= 0:
            raise ValueError("variance must be >= 0")
        if not (self.lx > 0 and self.ly > 0 and self.lz > 0):
            raise ValueError("length scales must be > 0")

    def to_c(self) -> "_lib.HikfKernel3":
        return _lib.HikfKernel3(_lib.FAMILY_CODE[self.family], float(self.variance), float(self.lx),
                                float(self.ly), float(self.lz))


class FmmTree3D:
    """Octree bbFMM over 3D points (csrc/fmm3d.cu); one Chebyshev order per level."""

    is_3d = True

    def __init__(self, points, kernel: KernelSpec3, n_cheb: int = 5, max_leaf_points: int = 128):
        _lib.require_cuda()
        xyz = np.ascontiguousarray(getattr(points, "coords", points), dtype=np.float64)
        if xyz.ndim != 2 or xyz.shape[1] != 3:
            raise ValueError("coords must have shape (m, 3)")
        self.m = xyz.shape[0]
        self.kernel = kernel
        self._handle = ctypes.c_void_p()
        kc = kernel.to_c()
        _lib.check(_lib.load().hikf_tree3_create(xyz.ctypes.data, self.m, ctypes.byref(kc), int(n_cheb),
                                                 int(max_leaf_points), _lib.stream_ptr(), ctypes.byref(self._handle)),
                   "3D tree build failed")
        m, depth, n, nl = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        lo, size = (ctypes.c_double * 3)(), ctypes.c_double()
        _lib.check(_lib.load().hikf_tree3_info(self._handle, ctypes.byref(m), ctypes.byref(depth), ctypes.byref(n),
                                               ctypes.byref(nl), lo, ctypes.byref(size)))
        self.depth, self.n_cheb, self.n_leaves = int(depth.value), int(n.value), int(nl.value)
        self.root_lo, self.root_size = np.array(list(lo)), float(size.value)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                _lib.load().hikf_tree3_destroy(h)
            except Exception:
                pass
            self._handle = None

    def export(self) -> dict:
        out = {"order": np.zeros(self.m, dtype=np.int64)}
        for k in ("leaf_keys", "leaf_starts", "leaf_counts"):
            out[k] = np.zeros(self.n_leaves, dtype=np.int64)
        _lib.check(_lib.load().hikf_tree3_export(self._handle, *(out[k].ctypes.data for k in
                                                                   ("order", "leaf_keys", "leaf_starts",
                                                                    "leaf_counts"))))
        return out

    def matmat(self, V):
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        is_t = isinstance(V, torch.Tensor)
        Vt = (V if is_t else torch.as_tensor(np.asarray(V, dtype=np.float64))).to(dev, torch.float64).contiguous()
        if Vt.ndim != 2 or Vt.shape[0] != self.m:
            raise ValueError(f"expected matrix with {self.m} rows, got shape {tuple(Vt.shape)}")
        U = torch.empty_like(Vt)
        _lib.check(_lib.load().hikf_tree3_matmat(self._handle, Vt.data_ptr(), Vt.shape[1], U.data_ptr(),
                                                 _lib.stream_ptr()))
        return U if is_t else U.cpu().numpy()


def build_tree3d(points, kernel: KernelSpec3, n_cheb: int = 5, max_leaf_points: int = 128) -> FmmTree3D:
    return FmmTree3D(points, kernel, n_cheb, max_leaf_points)
