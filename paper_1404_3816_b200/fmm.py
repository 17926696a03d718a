"""Black-box FMM tree on the B200: drop-in for the reference hikf.fmm.

Same public surface as the reference (fmm.py:38-54 FmmConfig, :92-367
FmmTree, :370-374 build_tree): the tree is built and applied by
libhikf_b200.so (quadtree build, box sort, interpolation and M2L operators,
P2P/P2M/M2M/M2L/L2L/L2P kernels), Python only validates and marshals.

``FmmTree.matmat`` accepts a numpy array (returns numpy, like the reference)
or a CUDA torch tensor (returns a CUDA tensor, no host round trip).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .kernels import to_c


@dataclass(frozen=True)
class FmmConfig:
    """Tree/expansion parameters (fmm.py:38-54)."""

    n_cheb: int = 5
    max_leaf_points: int = 64
    tolerance_hint: float | None = None

    def __post_init__(self):
        if not (2 <= self.n_cheb <= 12):
            raise ValueError("n_cheb must lie in [2, 12]")
        if self.max_leaf_points < 1:
            raise ValueError("max_leaf_points must be >= 1")


def _coords_of(points) -> np.ndarray:
    c = getattr(points, "coords", points)
    c = np.ascontiguousarray(np.asarray(c, dtype=np.float64))
    if c.ndim != 2 or c.shape[1] != 2:
        raise ValueError("coords must have shape (m, 2)")
    if c.shape[0] < 1:
        raise ValueError("need at least one point")
    if not np.all(np.isfinite(c)):
        raise ValueError("coordinates must be finite")
    return c


class FmmTree:
    """Immutable operator state for fast kernel products; built by build_tree."""

    def __init__(self, points, kernel, config: FmmConfig):
        lib = _lib.load()
        _lib.require_cuda()
        self.points = points
        self.kernel = kernel
        self.config = config
        xy = _coords_of(points)
        self.m = xy.shape[0]
        self._handle = ctypes.c_void_p()
        ck = to_c(kernel)
        _lib.check(lib.hikf_tree_create(xy.ctypes.data, self.m, ctypes.byref(ck), int(config.n_cheb),
                                        int(config.max_leaf_points), _lib.stream_ptr(), ctypes.byref(self._handle)),
                   "tree build failed")
        m = ctypes.c_int64()
        depth = ctypes.c_int32()
        orders = (ctypes.c_int32 * 21)()
        lo = (ctypes.c_double * 2)()
        size = ctypes.c_double()
        nl = ctypes.c_int64()
        npairs = ctypes.c_int64()
        _lib.check(lib.hikf_tree_info(self._handle, ctypes.byref(m), ctypes.byref(depth), orders, lo,
                                      ctypes.byref(size), ctypes.byref(nl), ctypes.byref(npairs)))
        self.depth = int(depth.value)
        self.root_lo = np.array([lo[0], lo[1]])
        self.root_size = float(size.value)
        self.n_leaves = int(nl.value)
        self.n_near_pairs = int(npairs.value)
        self._orders = {lev: int(orders[lev]) for lev in range(2, self.depth + 1)} if self.depth >= 2 else {}

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                _lib.load().hikf_tree_destroy(h)
            except Exception:
                pass
            self._handle = None

    # ------------------------------------------------------------------
    # parity exports (integer tree data and operators)
    # ------------------------------------------------------------------

    def export(self) -> dict:
        """order / leaf ranges / near leaf pairs as numpy int64 arrays."""
        lib = _lib.load()
        L, P = self.n_leaves, self.n_near_pairs
        out = {k: np.zeros(n, dtype=np.int64) for k, n in
               (("order", self.m), ("leaf_ids", L), ("leaf_starts", L), ("leaf_counts", L),
                ("near_t", P), ("near_s", P))}
        _lib.check(lib.hikf_tree_export(self._handle, *(out[k].ctypes.data for k in
                                                          ("order", "leaf_ids", "leaf_starts", "leaf_counts",
                                                           "near_t", "near_s"))))
        return out

    def m2l_op(self, lev: int, dx: int, dy: int) -> np.ndarray:
        q = self._orders[lev] ** 2
        out = np.zeros((q, q))
        _lib.check(_lib.load().hikf_tree_export_op(self._handle, 0, lev, dx, dy, out.ctypes.data))
        return out

    def shift_op(self, lev: int, cx: int, cy: int) -> np.ndarray:
        out = np.zeros((self._orders[lev + 1] ** 2, self._orders[lev] ** 2))
        _lib.check(_lib.load().hikf_tree_export_op(self._handle, 1, lev, cx, cy, out.ctypes.data))
        return out

    def interp_weights(self) -> np.ndarray:
        out = np.zeros((self.m, self._orders[self.depth] ** 2))
        _lib.check(_lib.load().hikf_tree_export_op(self._handle, 2, 0, 0, 0, out.ctypes.data))
        return out

    def m2l_pairs(self, lev: int, dx: int, dy: int):
        lib = _lib.load()
        cnt = ctypes.c_int64(0)
        _lib.check(lib.hikf_tree_m2l_pairs(self._handle, lev, dx, dy, None, None, ctypes.byref(cnt)))
        t = np.zeros(cnt.value, dtype=np.int64)
        s = np.zeros(cnt.value, dtype=np.int64)
        _lib.check(lib.hikf_tree_m2l_pairs(self._handle, lev, dx, dy, t.ctypes.data, s.ctypes.data,
                                           ctypes.byref(cnt)))
        return t, s

    # ------------------------------------------------------------------
    # application (fmm.py:318-367)
    # ------------------------------------------------------------------

    def matvec(self, v):
        is_t = isinstance(v, torch.Tensor)
        shape = tuple(v.shape) if is_t else np.shape(v)
        if shape != (self.m,):
            raise ValueError(f"expected vector of length {self.m}, got shape {shape}")
        out = self.matmat(v[:, None])
        return out[:, 0]

    def matmat(self, V):
        if isinstance(V, torch.Tensor):
            return self._matmat_device(V)
        V = np.asarray(V, dtype=float)
        if V.ndim != 2 or V.shape[0] != self.m:
            raise ValueError(f"expected matrix with {self.m} rows, got shape {V.shape}")
        dev = _lib.require_cuda()
        Vd = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
        return self._matmat_device(Vd).cpu().numpy()

    def _matmat_device(self, V: torch.Tensor) -> torch.Tensor:
        if V.ndim != 2 or V.shape[0] != self.m:
            raise ValueError(f"expected matrix with {self.m} rows, got shape {tuple(V.shape)}")
        if not V.is_cuda:
            raise ValueError("device matmat needs a CUDA tensor")
        V = V.to(torch.float64)
        if V.stride(1) != 1 or (V.shape[1] > 1 and V.stride(0) < V.shape[1]):
            V = V.contiguous()
        k = V.shape[1]
        U = torch.empty((self.m, k), dtype=torch.float64, device=V.device)
        if k:
            _lib.check(_lib.load().hikf_tree_matmat(self._handle, V.data_ptr(), max(V.stride(0), k), k,
                                                    U.data_ptr(), k, _lib.stream_ptr()))
        return U

    def matmat_csrT(self, H) -> torch.Tensor:
        """C = tree @ H^T for a scipy CSR H (n x m), H^T never densified on the host."""
        from .filters import DeviceCSR
        Hd = DeviceCSR.of(H)
        if Hd.shape[1] != self.m:
            raise ValueError("operator columns do not match the tree's point count")
        U = torch.empty((self.m, Hd.shape[0]), dtype=torch.float64, device="cuda")
        _lib.check(_lib.load().hikf_tree_matmat_csrT(self._handle, Hd.shape[0], Hd.indptr.data_ptr(),
                                                     Hd.indices.data_ptr(), Hd.data.data_ptr(), U.data_ptr(),
                                                     _lib.stream_ptr()))
        return U


def build_tree(points, kernel, config: FmmConfig | None = None) -> FmmTree:
    """Build the quadtree and all translation operators on the GPU (fmm.py:370-374)."""
    if config is None:
        config = FmmConfig()
    return FmmTree(points, kernel, config)
