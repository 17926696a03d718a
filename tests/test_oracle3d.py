"""The 3D oracle (oracle/hikf_oracle3d.py) against exact algebra.  There is no
reference output for 3D (the reference is 2D and isotropic), so the pins are:
the octree FMM against the dense direct sum, the ray operator against its
geometric invariants (row sums = ray lengths, grazing rays to the lower cell,
agreement with a fine point sampling of each ray)."""

import math

import numpy as np
import pytest

from oracle import hikf_oracle3d as O3


def test_ray_operator_3d_invariants():
    n3, d3 = (6, 5, 4), (1.0 / 6, 1.0 / 5, 1.0 / 4)
    src, rcv = O3.crosswell_3d(5, 4, seed=3)
    H = O3.ray_operator_3d(n3, d3, src, rcv)
    lengths = np.sqrt(((rcv - src) ** 2).sum(axis=1))
    np.testing.assert_allclose(np.asarray(H.sum(axis=1)).ravel(), lengths, rtol=1e-14)
    assert (H.data > 0).all()
    # sampling check: each ray's length per cell vs 20000 midpoint samples
    for r in range(0, len(src), 7):
        s = (np.arange(20000) + 0.5) / 20000
        p = src[r] + s[:, None] * (rcv[r] - src[r])
        idx = [np.clip(np.floor(p[:, a] / d3[a]).astype(int), 0, n3[a] - 1) for a in range(3)]
        cell = (idx[2] * n3[1] + idx[1]) * n3[0] + idx[0]
        approx = np.bincount(cell, minlength=np.prod(n3)) * (lengths[r] / 20000)
        np.testing.assert_allclose(H[r].toarray().ravel(), approx, atol=3 * lengths[r] / 20000)


def test_ray_operator_3d_grazing_and_errors():
    n3, d3 = (4, 4, 4), (0.25, 0.25, 0.25)
    # along x on the plane y = 0.5, z = 0.25: the lower cells (j = 1, k = 0)
    H = O3.ray_operator_3d(n3, d3, np.array([[0.0, 0.5, 0.25]]), np.array([[1.0, 0.5, 0.25]]))
    assert set(H.indices) == {(0 * 4 + 1) * 4 + i for i in range(4)}
    np.testing.assert_allclose(H.data, 0.25)
    # body diagonal through the cell corners: one cell per step, length sqrt(3)/4
    H = O3.ray_operator_3d(n3, d3, np.array([[0.0, 0.0, 0.0]]), np.array([[1.0, 1.0, 1.0]]))
    assert sorted(H.indices) == [(i * 4 + i) * 4 + i for i in range(4)]
    np.testing.assert_allclose(H.data, math.sqrt(3) / 4, rtol=1e-15)
    with pytest.raises(ValueError):
        O3.trace_3d(n3, d3, (0, 0, 0), np.zeros(3), np.zeros(3))


def test_face_stations_are_seeded_and_inside():
    a = O3.face_stations(24, 0.0, 0.0, 1.0, 0.0, 1.0, [0, 1])
    b = O3.face_stations(24, 0.0, 0.0, 1.0, 0.0, 1.0, [0, 1])
    assert np.array_equal(a, b) and a.shape == (24, 3)
    assert (a[:, 0] == 0.0).all() and (a[:, 1:] > 0).all() and (a[:, 1:] < 1).all()
    src, rcv = O3.crosswell_3d(24, 20, seed=0)
    assert src.shape == (480, 3) and rcv.shape == (480, 3) and (rcv[:, 0] == 1.0).all()


@pytest.mark.parametrize("fam,ls,order,tol", [("exponential", (0.3, 0.3, 0.3), 4, 3e-4),
                                              ("gaussian", (0.3, 0.3, 0.3), 4, 1e-3),
                                              ("exponential", (0.4, 0.4, 0.1), 5, 1e-4)])
def test_octree_fmm_against_direct_sum(fam, ls, order, tol):
    N = 12
    xyz = O3.cell_centers_3d(N, N, N, 1 / N, 1 / N, 1 / N)
    k = O3.Kern3(fam, 1.0, *ls)
    t = O3.OracleTree3D(xyz, k, order, 32)
    assert t.depth >= 2
    V = np.random.default_rng(0).standard_normal((len(xyz), 2))
    U = t.matmat(V)
    D = t.dense_matmat(V)
    assert np.linalg.norm(U - D) / np.linalg.norm(D) <= tol
    # the tree: leaves partition the points, stable order by box key
    assert t.leaf_counts.sum() == len(xyz) and (t.leaf_counts <= 32).all()
    assert np.all(np.diff(t.key[t.order]) >= 0)
