"""CPU oracle for the 3D configurations (BASELINE cfg3 / cfg5) -- TEST
INFRASTRUCTURE ONLY (tests/, smoke() and bench.py's cpu_baseline may use it;
the product path never does).

PARITY UNPINNED.  The reference ``hikf`` package is 2D and isotropic only
(SURVEY 8(d), 8(f) rank 2): there is no reference output for a 3D grid, a 3D
ray tracer, an octree or an anisotropic kernel.  This module states the 3D
algorithms as the direct extension of the reference's 2D rules, and is itself
checked against exact dense algebra (the direct-sum Q H^T) in
tests/test_oracle3d.py.  The CUDA path is checked against it.

Rules carried over from 2D, one more axis each:

* cells: row-major with x fastest, then y, then z (grids.py:47-52);
* ray tracing (tomography.py:76-108): breakpoints at the x / y / z plane
  crossings strictly inside (0, 1) plus {0, 1}, np.unique; a segment of
  positive length goes to the cell of its midpoint, a midpoint exactly on a
  plane goes to the lower cell; length = sqrt(dx^2 + dy^2 + dz^2);
* octree (fmm.py:95-164): cube root box lo = min, size = max extent *
  (1 + 1e-12); uniform depth = smallest with every leaf <= max_leaf, stopping
  when 8^(depth+1) > max(32768, 8 m); split-plane points go low; box key
  (bx G + by) G + bz, stable sort, np.unique;
* Chebyshev: the reference's 1D nodes and weights (fmm.py:57-78), tensor
  product over 3 axes, coefficient index (ix n + iy) n + iz;
* M2L offsets in [-3, 3]^3 with max |o| >= 2 whose parents are adjacent per
  axis (fmm.py:280-312); operator K(t_nodes, o h + t_nodes);
* one Chebyshev order at every level (the 2D order raising of fmm.py:206-244
  is not carried over: with n^3 coefficients it would multiply the M2L cost).

Anisotropic kernel: K(x, y) = variance exp(-(|A (x - y)|)^p) with
A = diag(1/lx, 1/ly, 1/lz).  The whole FMM runs on the scaled points A x with
the isotropic unit-length kernel, so boxes are cubes in the metric of the
kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse

from .hikf_oracle import cheb_nodes, cheb_weights

MAX_DEPTH = 10


@dataclass(frozen=True)
class Kern3:
    """variance exp(-(r')^p), r' = |(dx/lx, dy/ly, dz/lz)|; family gaussian (p = 2) / exponential (p = 1)."""

    family: str
    variance: float = 1.0
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0

    @property
    def p(self) -> float:
        return {"gaussian": 2.0, "exponential": 1.0}[self.family]

    def scale(self, xyz: np.ndarray) -> np.ndarray:
        return np.column_stack([xyz[:, 0] / self.lx, xyz[:, 1] / self.ly, xyz[:, 2] / self.lz])

    def of_r(self, r: np.ndarray) -> np.ndarray:
        """K at scaled distance r (numpy's p == 1 / 2 fast paths: copy / square)."""
        t = r * r if self.p == 2.0 else r
        return self.variance * np.exp(-t)


def dist3(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """|a_i - b_j| with the operation order ((dx dx + dy dy) + dz dz) then sqrt."""
    d = a[:, None, :] - b[None, :, :]
    return np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])


# ----------------------------------------------------------------------------
# grid, stations, rays
# ----------------------------------------------------------------------------


def cell_centers_3d(nx, ny, nz, dx, dy, dz, x0=0.0, y0=0.0, z0=0.0) -> np.ndarray:
    xs = x0 + (np.arange(nx) + 0.5) * dx
    ys = y0 + (np.arange(ny) + 0.5) * dy
    zs = z0 + (np.arange(nz) + 0.5) * dz
    return np.column_stack([np.tile(xs, ny * nz), np.tile(np.repeat(ys, nx), nz), np.repeat(zs, nx * ny)])


def face_stations(k: int, x: float, ylo: float, yhi: float, zlo: float, zhi: float, seed) -> np.ndarray:
    """k stations on the plane x = const: one per cell of the first k cells
    (row-major, y fastest) of an a x b lattice (a = ceil(sqrt(k)), b =
    ceil(k / a)) over [ylo, yhi] x [zlo, zhi], uniformly jittered inside its
    cell with PCG64(seed)."""
    a = int(math.ceil(math.sqrt(k)))
    b = int(math.ceil(k / a))
    rng = np.random.default_rng(seed)
    u = rng.random((a * b, 2))
    idx = np.arange(a * b)
    iy, iz = idx % a, idx // a
    y = ylo + (iy + u[:, 0]) * ((yhi - ylo) / a)
    z = zlo + (iz + u[:, 1]) * ((zhi - zlo) / b)
    return np.column_stack([np.full(a * b, float(x)), y, z])[:k]


def crosswell_3d(ns: int, nr: int, seed: int, extent=(0.0, 1.0, 0.0, 1.0, 0.0, 1.0)):
    """Sources on the x = xmin face, receivers on x = xmax (seeds [seed, 1] and
    [seed, 2]); rays source-major like tomography.py:38-43."""
    x0, x1, y0, y1, z0, z1 = extent
    src = face_stations(ns, x0, y0, y1, z0, z1, [seed, 1])
    rcv = face_stations(nr, x1, y0, y1, z0, z1, [seed, 2])
    return np.repeat(src, nr, axis=0), np.tile(rcv, (ns, 1))


def trace_3d(n3, d3, o3, p0, p1):
    """Cells and lengths along one straight ray in an nx x ny x nz grid."""
    d = p1 - p0
    length = math.sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2])
    if length == 0.0:
        raise ValueError("zero-length ray")
    cuts = [np.array([0.0, 1.0])]
    for ax in range(3):
        if d[ax] != 0.0:
            t = (o3[ax] + np.arange(1, n3[ax]) * d3[ax] - p0[ax]) / d[ax]
            cuts.append(t[(t > 0.0) & (t < 1.0)])
    t = np.unique(np.concatenate(cuts))
    seg = np.diff(t) * length
    keep = seg > 0.0
    mid = (0.5 * (t[:-1] + t[1:]))[keep]
    idx = []
    for ax in range(3):
        u = (p0[ax] + mid * d[ax] - o3[ax]) / d3[ax]
        c = np.floor(u).astype(np.int64)
        c[(u == c) & (c > 0)] -= 1
        idx.append(np.clip(c, 0, n3[ax] - 1))
    return (idx[2] * n3[1] + idx[1]) * n3[0] + idx[0], seg[keep]


def ray_operator_3d(n3, d3, src, rcv, o3=(0.0, 0.0, 0.0)) -> scipy.sparse.csr_matrix:
    rows, cols, vals = [], [], []
    for r, (a, b) in enumerate(zip(src, rcv)):
        c, s = trace_3d(n3, d3, o3, a, b)
        rows.append(np.full(len(c), r))
        cols.append(c)
        vals.append(s)
    H = scipy.sparse.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                shape=(len(src), n3[0] * n3[1] * n3[2])).tocsr()
    H.sum_duplicates()
    return H


def plumes_3d(centers: np.ndarray, steps: int, plumes) -> np.ndarray:
    """Sum of constant-amplitude 3D Gaussian blobs; plumes = [(x_start, yc, zc, width, dx_step)];
    row 0 is zero (tomography.py:177-178)."""
    F = np.zeros((steps + 1, len(centers)))
    for t in range(1, steps + 1):
        for (xs, yc, zc, w, step) in plumes:
            cx = xs + step * (t - 1)
            r2 = (centers[:, 0] - cx) ** 2 + (centers[:, 1] - yc) ** 2 + (centers[:, 2] - zc) ** 2
            F[t] += np.exp(-r2 / (2 * w * w))
    return F


# ----------------------------------------------------------------------------
# octree bbFMM
# ----------------------------------------------------------------------------


def box_of_3d(c: np.ndarray, lo: np.ndarray, size: float, depth: int):
    G = 1 << depth
    h = size / G
    out = []
    for d in range(3):
        u = (c[:, d] - lo[d]) / h
        b = np.floor(u).astype(np.int64)
        b[(u == b) & (b > 0)] -= 1
        out.append(np.clip(b, 0, G - 1))
    return out


def choose_depth_3d(c, lo, size, leaf_cap: int) -> int:
    m = len(c)
    for depth in range(MAX_DEPTH):
        bx, by, bz = box_of_3d(c, lo, size, depth)
        G = 1 << depth
        if np.bincount((bx * G + by) * G + bz).max() <= leaf_cap:
            return depth
        if 8 ** (depth + 1) > max(32768, 8 * m):
            return depth
    return MAX_DEPTH


def _offsets():
    return [(a, b, c) for a in range(-3, 4) for b in range(-3, 4) for c in range(-3, 4)
            if max(abs(a), abs(b), abs(c)) >= 2]


class OracleTree3D:
    """Uniform-depth octree bbFMM over the scaled points (dense expansions)."""

    def __init__(self, xyz: np.ndarray, k: Kern3, n_cheb: int, max_leaf: int):
        self.k = k
        self.n = n_cheb
        self.pts = k.scale(np.asarray(xyz, dtype=float))
        self.m = len(self.pts)
        lo = self.pts.min(axis=0)
        hi = self.pts.max(axis=0)
        self.lo = lo
        self.size = float((hi - lo).max()) * (1.0 + 1e-12)
        self.depth = choose_depth_3d(self.pts, lo, self.size, max_leaf)
        G = 1 << self.depth
        bx, by, bz = box_of_3d(self.pts, lo, self.size, self.depth)
        key = (bx * G + by) * G + bz
        self.order = np.argsort(key, kind="stable")
        self.leaf_ids, self.leaf_starts, self.leaf_counts = np.unique(key[self.order], return_index=True,
                                                                     return_counts=True)
        self.key = key

    # -- operators --
    def _nodes3(self, h: float) -> np.ndarray:
        nd = cheb_nodes(self.n) * (h / 2.0)
        n = self.n
        return np.column_stack([np.repeat(nd, n * n), np.tile(np.repeat(nd, n), n), np.tile(nd, n * n)])

    def interp(self) -> np.ndarray:
        """W2 (m x n^3), original point order: S_ix(xi) S_iy(eta) S_iz(zeta) in the point's leaf."""
        G = 1 << self.depth
        h = self.size / G
        bx, by, bz = box_of_3d(self.pts, self.lo, self.size, self.depth)
        ctr = self.lo + (np.column_stack([bx, by, bz]) + 0.5) * h
        loc = (self.pts - ctr) / (h / 2.0)
        w = [cheb_weights(loc[:, d], self.n) for d in range(3)]
        n = self.n
        return np.einsum("pi,pj,pk->pijk", w[0], w[1], w[2]).reshape(self.m, n ** 3)

    def shift(self) -> dict:
        """Child -> parent interpolation kron(Bx, By, Bz) per child parity (fmm.py:264-278)."""
        xs = cheb_nodes(self.n)
        out = {}
        for cx in (0, 1):
            for cy in (0, 1):
                for cz in (0, 1):
                    B = [cheb_weights((xs + 2 * c - 1) / 2.0, self.n) for c in (cx, cy, cz)]
                    out[(cx, cy, cz)] = np.einsum("ia,jb,kc->ijkabc", *B).reshape(self.n ** 3, self.n ** 3)
        return out

    def m2l(self, lev: int) -> dict:
        h = self.size / (1 << lev)
        t = self._nodes3(h)
        ops = {}
        for o in _offsets():
            s = t + np.array(o, dtype=float) * h
            ops[o] = self.k.of_r(dist3(t, s))
        return ops

    # -- product --
    def near_matmat(self, V: np.ndarray) -> np.ndarray:
        G = 1 << self.depth
        U = np.zeros((self.m, V.shape[1]))
        leaf_of = {int(k): i for i, k in enumerate(self.leaf_ids)}
        for li, key in enumerate(self.leaf_ids):
            bx, rem = divmod(int(key), G * G)
            by, bz = divmod(rem, G)
            t = self.order[self.leaf_starts[li]:self.leaf_starts[li] + self.leaf_counts[li]]
            src = []
            for ox in (-1, 0, 1):
                for oy in (-1, 0, 1):
                    for oz in (-1, 0, 1):
                        x, y, z = bx + ox, by + oy, bz + oz
                        if min(x, y, z) < 0 or max(x, y, z) >= G:
                            continue
                        s = leaf_of.get((x * G + y) * G + z)
                        if s is None:
                            continue
                        src.append(self.order[self.leaf_starts[s]:self.leaf_starts[s] + self.leaf_counts[s]])
            src = np.concatenate(src)
            U[t] += self.k.of_r(dist3(self.pts[t], self.pts[src])) @ V[src]
        return U

    def matmat(self, V: np.ndarray) -> np.ndarray:
        V = np.asarray(V, dtype=float)
        U = self.near_matmat(V)
        D = self.depth
        if D < 2:
            return U
        k = V.shape[1]
        q = self.n ** 3
        W2 = self.interp()
        bx, by, bz = box_of_3d(self.pts, self.lo, self.size, D)
        G = 1 << D
        w = {D: np.zeros((G, G, G, q, k))}
        np.add.at(w[D], (bx, by, bz), np.einsum("pa,pk->pak", W2, V))
        shifts = self.shift()
        for lev in range(D - 1, 1, -1):
            Gp = 1 << lev
            wp = np.zeros((Gp, Gp, Gp, q, k))
            child = w[lev + 1]
            for (cx, cy, cz), C in shifts.items():
                wp += np.einsum("xyzak,ab->xyzbk", child[cx::2, cy::2, cz::2], C)
            w[lev] = wp
        loc = None
        for lev in range(2, D + 1):
            Gl = 1 << lev
            L = np.zeros((Gl, Gl, Gl, q, k))
            ops = self.m2l(lev)
            W = w[lev]
            idx = np.arange(Gl)
            for o, M in ops.items():
                tx = idx[(idx + o[0] >= 0) & (idx + o[0] < Gl)]
                ty = idx[(idx + o[1] >= 0) & (idx + o[1] < Gl)]
                tz = idx[(idx + o[2] >= 0) & (idx + o[2] < Gl)]
                for x in tx:
                    for y in ty:
                        for z in tz:
                            s = (x + o[0], y + o[1], z + o[2])
                            if max(abs((x >> 1) - (s[0] >> 1)), abs((y >> 1) - (s[1] >> 1)),
                                   abs((z >> 1) - (s[2] >> 1))) > 1:
                                continue
                            L[x, y, z] += M @ W[s]
            if loc is not None:
                for (cx, cy, cz), C in shifts.items():
                    L[cx::2, cy::2, cz::2] += np.einsum("ab,xyzbk->xyzak", C, loc)
            loc = L
        U += np.einsum("pa,pak->pk", W2, loc[bx, by, bz])
        return U

    def dense_matmat(self, V: np.ndarray) -> np.ndarray:
        """Exact Q V with the dense Gram (r = 0 -> K(0))."""
        return self.k.of_r(dist3(self.pts, self.pts)) @ V
