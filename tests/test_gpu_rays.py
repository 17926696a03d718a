"""Device ray operator (hikf_ray_operator_device): the CSR
traced on the GPU must be bit-identical -- pattern AND lengths -- to the
reference's build_ray_operator (tomography.py:76-133, golden fixtures made by
the reference) and to the host restatement, including grazing rays along
gridlines, rays through cell corners, vertical/horizontal rays, rays on the
boundary and random interior segments; the filter must accept it as H.
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import hikf_oracle as O
from tests.golden import cases

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _same(Hd, Hh):
    A = Hd.to_scipy()
    assert A.shape == Hh.shape
    assert np.array_equal(A.indptr.astype(np.int64), Hh.indptr.astype(np.int64))
    assert np.array_equal(A.indices.astype(np.int64), Hh.indices.astype(np.int64))
    assert np.array_equal(A.data.view(np.uint64), np.asarray(Hh.data, dtype=np.float64).view(np.uint64))


@pytest.mark.parametrize("cfg,fixture", [(cases.SMALL, "small_rays.npz"), (cases.CFG1, "cfg1.npz"),
                                         (cases.CFG2, "cfg2.npz"), (cases.CFG4, "cfg4_pins.npz")])
def test_device_ray_operator_matches_reference(cfg, fixture):
    from paper_1404_3816_b200 import Grid2D, tomography
    g = dict(np.load(os.path.join(G, fixture)))
    N = cfg["N"]
    grid = Grid2D(nx=N, ny=N, dx=1.0 / N, dy=1.0 / N)
    acq = tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0)
    Hd = tomography.build_ray_operator_device(grid, acq)
    H = Hd.to_scipy()
    if "H_indices" in g:
        assert np.array_equal(H.indptr.astype(np.int64), g["H_indptr"])
        assert np.array_equal(H.indices.astype(np.int64), g["H_indices"])
        assert np.array_equal(H.data, g["H_data"])
    else:
        assert H.nnz == int(g["H_nnz"])
        assert _sha(H.indptr.astype(np.int64), H.indices.astype(np.int64)) == g["H_pattern_sha"].item().decode()
        assert _sha(H.data) == g["H_data_sha"].item().decode()
    _same(Hd, tomography.build_ray_operator(grid, acq))


def test_device_ray_operator_edge_cases():
    from paper_1404_3816_b200 import Grid2D, tomography
    grid = Grid2D(nx=7, ny=5, dx=0.5, dy=0.25, origin=(-1.0, 2.0))
    x0, y0 = grid.origin
    x1, y1 = x0 + 7 * 0.5, y0 + 5 * 0.25
    src = [[x0, y0 + 0.25], [x0, y0], [x0 + 1.0, y0], [x0, y0], [x1, y1], [x0 + 0.5, y0 + 0.5], [x0, y1], [x0, y0]]
    rcv = [[x1, y0 + 0.25], [x1, y1], [x0 + 1.0, y1], [x0 + 0.5, y0 + 0.25], [x0, y0], [x0 + 1.5, y0 + 1.0],
           [x1, y1], [x0, y1]]
    # horizontal on a gridline, corner-to-corner, vertical on a gridline, one-cell diagonal,
    # reversed direction, diagonal through interior corners, top boundary, left boundary
    rng = np.random.default_rng(7)
    for _ in range(64):
        src.append([rng.uniform(x0, x1), rng.uniform(y0, y1)])
        rcv.append([rng.uniform(x0, x1), rng.uniform(y0, y1)])
    src, rcv = np.array(src), np.array(rcv)
    acq_pairs = [(src[i:i + 1], rcv[i:i + 1]) for i in range(len(src))]
    for s, r in acq_pairs:  # one ray at a time (the Acquisition is a source x receiver product)
        acq = tomography.Acquisition(s, r)
        _same(tomography.build_ray_operator_device(grid, acq), tomography.build_ray_operator(grid, acq))
    # the oracle (a restatement of tomography.py) on all rays at once
    Ho = O.ray_operator(7, 5, 0.5, 0.25, src, rcv, x0=x0, y0=y0)
    Hd = np.vstack([tomography.build_ray_operator_device(grid, tomography.Acquisition(s, r)).to_scipy().toarray()
                    for s, r in acq_pairs])
    assert np.array_equal(Hd, Ho.toarray())
    with pytest.raises(ValueError):
        tomography.build_ray_operator_device(grid, tomography.Acquisition(np.array([[x0, y0]]), np.array([[x0, y0]])))
    with pytest.raises(ValueError):
        tomography.build_ray_operator_device(grid, tomography.Acquisition(np.array([[x0 - 1, y0]]),
                                                                          np.array([[x1, y1]])))


def test_device_ray_operator_random_acquisitions_and_filter():
    """Many-station products on a non-square grid + the operator used as H by the filter."""
    import torch

    from paper_1404_3816_b200 import Grid2D, filters, tomography
    grid = Grid2D(nx=61, ny=45, dx=1.0 / 61, dy=1.0 / 45)
    rng = np.random.default_rng(3)
    src = np.column_stack([np.zeros(9), np.sort(rng.uniform(0, 1, 9))])
    rcv = np.column_stack([np.full(11, 1.0), np.sort(rng.uniform(0, 1, 11))])
    src[3] = [0.0, 1.0 / 45 * 7]  # a station exactly on a gridline
    acq = tomography.Acquisition(src, rcv)
    Hd = tomography.build_ray_operator_device(grid, acq)
    Hh = tomography.build_ray_operator(grid, acq)
    _same(Hd, Hh)
    # H from the device feeds the precompute without a host round trip; same C_Q as the host H
    import types

    import paper_1404_3816_b200 as P
    kern = P.KernelSpec("exponential", variance=1.0, length_scale=0.3)
    tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=5, max_leaf_points=48))
    a = filters.hikf_precompute_fmm(types.SimpleNamespace(H=Hd, m=grid.m), tree)
    b = filters.hikf_precompute_fmm(types.SimpleNamespace(H=Hh, m=grid.m), tree)
    assert torch.equal(a.C_Q_t, b.C_Q_t) and torch.equal(a.HC_Q_t, b.HC_Q_t)


def test_device_ray_operator_large_grid():
    """Largest supported grid (nx + ny = 4096) against the host restatement."""
    from paper_1404_3816_b200 import Grid2D, tomography
    grid = Grid2D(nx=2048, ny=2048, dx=1.0 / 2048, dy=1.0 / 2048)
    acq = tomography.default_acquisition(grid, 8, 16, 0.0, 1.0)
    _same(tomography.build_ray_operator_device(grid, acq), tomography.build_ray_operator(grid, acq))
    with pytest.raises(ValueError):
        tomography.build_ray_operator_device(Grid2D(nx=2049, ny=2048), acq)
