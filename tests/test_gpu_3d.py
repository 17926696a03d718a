"""3D path (BASELINE cfg3 / cfg5) on the GPU against the 3D oracle
(oracle/hikf_oracle3d.py, itself checked against exact algebra; parity with the
reference is unpinned because the reference is 2D only):

* ray operator: host and device bit-identical to the oracle;
* octree: order / leaves bit-identical to the oracle;
* Q V and Q H^T: the oracle's FMM to reassociation roundoff, the exact direct
  sum to the FMM's own truncation error (also at the cfg3 shape, on columns);
* a short filter run against the oracle's update loop.
"""

import numpy as np
import pytest

from oracle import hikf_oracle as O
from oracle import hikf_oracle3d as O3

pytestmark = pytest.mark.gpu


def _same_csr(A, B):
    assert A.shape == B.shape
    assert np.array_equal(A.indptr.astype(np.int64), B.indptr.astype(np.int64))
    assert np.array_equal(A.indices.astype(np.int64), B.indices.astype(np.int64))
    assert np.array_equal(np.asarray(A.data, dtype=np.float64).view(np.uint64),
                          np.asarray(B.data, dtype=np.float64).view(np.uint64))


@pytest.mark.parametrize("N,ns,nr,seed", [(8, 5, 4, 3), (64, 24, 20, 0), (20, 7, 9, 5)])
def test_ray_operator_3d_bit_exact(N, ns, nr, seed):
    from paper_1404_3816_b200 import space3d as S
    grid = S.Grid3D(N, N, N, 1.0 / N, 1.0 / N, 1.0 / N)
    acq = S.crosswell_3d(grid, ns, nr, seed)
    src, rcv = O3.crosswell_3d(ns, nr, seed)
    assert np.array_equal(acq.ray_endpoints()[0], src) and np.array_equal(acq.ray_endpoints()[1], rcv)
    Ho = O3.ray_operator_3d((N, N, N), (1.0 / N,) * 3, src, rcv)
    Hh = S.build_ray_operator_3d(grid, acq)
    _same_csr(Hh, Ho)
    _same_csr(S.build_ray_operator_3d_device(grid, acq).to_scipy(), Ho)


def test_ray_operator_3d_grazing_device():
    from paper_1404_3816_b200 import space3d as S
    grid = S.Grid3D(4, 4, 4, 0.25, 0.25, 0.25)
    pts = [([0.0, 0.5, 0.25], [1.0, 0.5, 0.25]), ([0.0, 0.0, 0.0], [1.0, 1.0, 1.0]),
           ([0.5, 0.0, 0.5], [0.5, 1.0, 0.5]), ([0.1, 0.2, 0.3], [0.9, 0.7, 0.35])]
    for a, b in pts:
        acq = S.Acquisition3D(np.array([a]), np.array([b]))
        Ho = O3.ray_operator_3d((4, 4, 4), (0.25,) * 3, np.array([a]), np.array([b]))
        _same_csr(S.build_ray_operator_3d_device(grid, acq).to_scipy(), Ho)
        _same_csr(S.build_ray_operator_3d(grid, acq), Ho)
    with pytest.raises(ValueError):
        S.build_ray_operator_3d(grid, S.Acquisition3D(np.array([[0.0, 0.0, 0.0]]), np.array([[0.0, 0.0, 0.0]])))


# (family, length scales, order, leaf, N, FMM truncation tolerance vs the direct sum)
CASES = [("exponential", (0.3, 0.3, 0.3), 4, 32, 12, 1e-3), ("gaussian", (0.3, 0.3, 0.3), 3, 16, 10, 1e-2),
         ("exponential", (0.4, 0.4, 0.1), 5, 32, 12, 1e-4)]


@pytest.mark.parametrize("fam,ls,order,leaf,N,tol", CASES)
def test_octree_and_matmat_against_oracle(fam, ls, order, leaf, N, tol):
    from paper_1404_3816_b200 import space3d as S
    xyz = O3.cell_centers_3d(N, N, N, 1 / N, 1 / N, 1 / N)
    k3 = O3.Kern3(fam, 1.0, *ls)
    ot = O3.OracleTree3D(xyz, k3, order, leaf)
    tree = S.build_tree3d(xyz, S.KernelSpec3(fam, 1.0, *ls), n_cheb=order, max_leaf_points=leaf)
    ex = tree.export()
    assert tree.depth == ot.depth
    assert np.array_equal(ex["order"], ot.order)
    assert np.array_equal(ex["leaf_keys"], ot.leaf_ids)
    assert np.array_equal(ex["leaf_starts"], ot.leaf_starts)
    assert np.array_equal(ex["leaf_counts"], ot.leaf_counts)
    V = np.random.default_rng(1).standard_normal((len(xyz), 70))  # > one 64-column chunk
    U = tree.matmat(V)
    Uo = ot.matmat(V)
    assert O.rel_fro(U, Uo) <= 1e-12
    D = ot.dense_matmat(V)
    assert O.rel_fro(U, D) <= tol


def test_precompute3_and_filter_against_oracle():
    import torch

    from paper_1404_3816_b200 import filters as flt
    from paper_1404_3816_b200 import space3d as S
    N, ns, nr, T, R = 12, 4, 5, 6, 1e-3
    grid = S.Grid3D(N, N, N, 1 / N, 1 / N, 1 / N)
    acq = S.crosswell_3d(grid, ns, nr, 0)
    H = S.build_ray_operator_3d(grid, acq)
    xyz = grid.cell_centers().coords
    k3 = O3.Kern3("exponential", 1.0, 0.4, 0.4, 0.2)
    tree = S.build_tree3d(xyz, S.KernelSpec3("exponential", 1.0, 0.4, 0.4, 0.2), n_cheb=4, max_leaf_points=32)
    model = type("M3", (), dict(H=H, m=grid.m, n=H.shape[0], alpha=0.0, initial_mean=np.zeros(grid.m)))()
    pre = flt.hikf_precompute_fmm(model, tree)
    ot = O3.OracleTree3D(xyz, k3, 4, 32)
    CQ = ot.matmat(H.T.toarray())
    assert O.rel_fro(pre.C_Q, CQ) <= 1e-12
    HCQ = np.asarray(H @ CQ)
    assert O.rel_fro(pre.HC_Q, 0.5 * (HCQ + HCQ.T)) <= 1e-12
    np.testing.assert_array_equal(pre.diag_Q, np.ones(grid.m))
    fields = O3.plumes_3d(xyz, T, [(0.2, 0.5, 0.5, 0.08, 0.005)])
    obs = O.observations(H, fields, R, [0, 0])
    st = flt.hikf_init(model)
    ost = O.init_state(H, grid.m)
    opre = O.Pre(CQ, 0.5 * (HCQ + HCQ.T), np.ones(grid.m))
    for t in range(T):
        st = flt.hikf_update(flt.hikf_predict(st, pre), H, R, obs[t])
        ost = O.update(O.predict(ost, opre), H, R, obs[t])
    assert O.rel_fro(st.mean, ost.mean) <= 1e-9
    assert O.rel_fro(st.variance, ost.variance) <= 1e-9
    assert O.rel_fro(st.cross_cov, ost.cross_cov) <= 1e-9
    del torch


@pytest.mark.slow
def test_cfg3_shape_qht_columns_against_direct_sum():
    """cfg3 (64^3 cells, 24 x 20 jittered rays, exponential 0.3, order 5, leaf 128):
    Q H^T on 4 columns against the exact direct sum on the GPU."""
    import torch

    from paper_1404_3816_b200 import space3d as S
    N = 64
    grid = S.Grid3D(N, N, N, 1 / N, 1 / N, 1 / N)
    acq = S.crosswell_3d(grid, 24, 20, 0)
    H = S.build_ray_operator_3d(grid, acq)
    assert H.shape == (480, N ** 3)
    xyz = grid.cell_centers().coords
    tree = S.build_tree3d(xyz, S.KernelSpec3("exponential", 1.0, 0.3, 0.3, 0.3), n_cheb=5, max_leaf_points=128)
    model = type("M3", (), dict(H=H, m=grid.m, n=480, alpha=0.0, initial_mean=np.zeros(grid.m)))()
    from paper_1404_3816_b200 import filters as flt
    pre = flt.hikf_precompute_fmm(model, tree)
    X = torch.as_tensor(xyz / 0.3, device="cuda")
    for j in (0, 131, 277, 479):
        cells = H.indices[H.indptr[j]:H.indptr[j + 1]]
        h = torch.as_tensor(H.data[H.indptr[j]:H.indptr[j + 1]], device="cuda")
        r = torch.cdist(X, X[torch.as_tensor(cells, device="cuda").long()])
        exact = (torch.exp(-r) @ h).cpu().numpy()
        assert O.rel_fro(pre.C_Q_t[:, j].cpu().numpy(), exact) <= 1e-4
