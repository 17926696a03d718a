"""Seeded input recipes shared by the golden generator and the tests.

Nothing here imports the reference or the product: it only builds numpy
inputs (point clouds, charges, SPD matrices, BASELINE scenario parameters)
so that ``make_golden.py`` (reference side) and ``tests/`` (oracle and CUDA
side) see byte-identical inputs.
"""

from __future__ import annotations

import numpy as np

# BASELINE.json configs; seed = [seed, 0] as experiment.py:166
CFG1 = dict(name="cfg1", N=64, ns=8, nr=8, family="exponential", L=0.3, R=1e-2, T=20, order=4, leaf=64, seed=0)
CFG2 = dict(name="cfg2", N=256, ns=16, nr=16, family="gaussian", L=0.2, R=1e-3, T=100, order=5, leaf=64, seed=0)
CFG4 = dict(name="cfg4", N=1024, ns=32, nr=32, family="exponential", L=0.25, R=1e-3, T=50, order=6, leaf=64, seed=0)
# a small far-field-exercising scenario (depth 3, two far levels)
SMALL = dict(name="small", N=24, ns=4, nr=5, family="gaussian", L=0.2, R=1e-3, T=10, order=5, leaf=16, seed=3)


def plume_fields(centers: np.ndarray, steps: int, x0=0.2, yc=0.5, width=0.1, dxs=0.01) -> np.ndarray:
    """Constant-amplitude Gaussian plume moving +dxs per step; row 0 is zero."""
    F = np.zeros((steps + 1, len(centers)))
    for t in range(1, steps + 1):
        cx = x0 + dxs * (t - 1)
        F[t] = np.exp(-((centers[:, 0] - cx) ** 2 + (centers[:, 1] - yc) ** 2) / (2 * width * width))
    return F


def charges(m: int, k: int) -> np.ndarray:
    return np.random.default_rng(12).standard_normal((m, k))


def _grid(nx, ny, dx, dy):
    xs = (np.arange(nx) + 0.5) * dx
    ys = (np.arange(ny) + 0.5) * dy
    return np.column_stack([np.tile(xs, ny), np.repeat(ys, nx)])


def _edge_cloud() -> np.ndarray:
    """Random points plus exact split-line hits, corners and 70 coincident points."""
    rng = np.random.default_rng(21)
    pts = [rng.random((560, 2))]
    pts.append(np.array([[0.0, 0.0], [1.0, 1.0], [1.0, 0.0], [0.0, 1.0]]))
    size = 1.0 * (1.0 + 1e-12)
    for G in (2, 4, 8, 16):
        h = size / G
        k = np.arange(1, G)
        pts.append(np.column_stack([k * h, np.full(len(k), 0.37)]))
        pts.append(np.column_stack([np.full(len(k), 0.61), k * h]))
    pts.append(np.tile([[0.3125, 0.6875]], (70, 1)))
    return np.concatenate(pts)


def tree_cases() -> dict:
    """name -> (points, kernel dict, n_cheb, max_leaf_points, n charge columns)."""
    cloud = np.random.default_rng(11).random((1500, 2)) * 10.0
    return {
        "cloud_gauss7": (cloud, dict(family="gaussian", variance=1.0, length_scale=2.0), 7, 64, 2),
        "cloud_exp4": (cloud, dict(family="exponential", variance=0.5, length_scale=3.0), 4, 64, 3),
        "cloud_log5": (cloud, dict(family="logarithm", log_amplitude=-1.0), 5, 64, 2),
        "single_leaf": (np.random.default_rng(16).random((30, 2)),
                        dict(family="gaussian", length_scale=0.2), 3, 64, 2),
        "depth1": (np.random.default_rng(17).random((100, 2)),
                   dict(family="exponential", length_scale=0.5), 4, 32, 2),
        "grid_cfg1": (_grid(64, 64, 1 / 64, 1 / 64), dict(family="exponential", length_scale=0.3), 4, 64, 3),
        "grid_30x28": (_grid(30, 28, 1.0, 1.0), dict(family="exponential", variance=1e-2, length_scale=4.0), 7, 64, 2),
        "edges_gauss": (_edge_cloud(), dict(family="gaussian", length_scale=0.3), 5, 64, 2),
        "edges_log": (_edge_cloud(), dict(family="logarithm", log_amplitude=-0.5), 4, 64, 2),
        "rect_empty": (np.column_stack([np.random.default_rng(19).random(2000) * 10.0,
                                        np.random.default_rng(20).random(2000)]),
                       dict(family="gaussian", length_scale=1.0), 5, 64, 2),
    }


def spd_case():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((12, 12))
    A = A @ A.T + 12 * np.eye(12)
    B = np.random.default_rng(1).standard_normal((12, 3))
    return A, B


def update_cases():
    """(state dict, dense H, r, z) hand and random cases for hikf_update."""
    out = []
    # scalar hand values: gain 1/2, posterior variance 1/2 (tests/test_filters.py:184-191)
    out.append((dict(mean=np.zeros(1), cross_cov=np.array([[1.0]]), variance=np.array([1.0]),
                     HC=np.array([[1.0]])), np.array([[1.0]]), 1.0, np.array([2.0])))
    # consistent random state from a dense P (m = 9, n = 4)
    rng = np.random.default_rng(31)
    m, n = 9, 4
    A = rng.standard_normal((m, m))
    P = A @ A.T + m * np.eye(m)
    H = rng.standard_normal((n, m))
    C = P @ H.T
    out.append((dict(mean=rng.standard_normal(m), cross_cov=C, variance=np.diag(P).copy(), HC=H @ C),
                H, 0.3, rng.standard_normal(n)))
    return out


def sketch_vectors(m: int, n: int):
    """Seeded probe vectors for the column / row sketches of m x n fixtures."""
    rng = np.random.default_rng(77)
    return rng.standard_normal(m), rng.standard_normal(n)
