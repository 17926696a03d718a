"""Pin the CPU oracle (oracle/hikf_oracle.py) to the reference's golden outputs.

The fixtures were produced by the real reference (tests/golden/make_golden.py);
integer/index data must match bit for bit, floats to reassociation roundoff.
"""

import hashlib
import os

import numpy as np
import pytest
import scipy.sparse

from oracle import hikf_oracle as O
from tests.golden import cases

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    path = os.path.join(G, name)
    if not os.path.exists(path):
        pytest.skip(f"fixture {name} not generated")
    return dict(np.load(path))


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _kern(spec):
    return O.Kern(spec["family"], spec.get("variance", 1.0), spec.get("length_scale", 1.0),
                  None, spec.get("log_amplitude"))


def _m2l_digest(tree):
    keys, counts, h = [], [], hashlib.sha256()
    for key in sorted(tree.m2l_pairs):
        t, s = tree.m2l_pairs[key]
        keys.append(key)
        counts.append(len(t))
        h.update(np.asarray(t, dtype=np.int64).tobytes())
        h.update(np.asarray(s, dtype=np.int64).tobytes())
    return np.array(keys, dtype=np.int64), np.array(counts, dtype=np.int64), h.hexdigest()


def check_tree_ints(tree, g, prefix="tree_"):
    assert tree.depth == int(g[prefix + "depth"])
    assert tree.size == float(g[prefix + "root_size"])
    assert np.array_equal(tree.lo, g[prefix + "root_lo"])
    assert np.array_equal(tree.order, g[prefix + "order"])
    assert np.array_equal(tree.leaf_ids, g[prefix + "leaf_ids"])
    assert np.array_equal(tree.leaf_starts, g[prefix + "leaf_starts"])
    assert np.array_equal(tree.leaf_counts, g[prefix + "leaf_counts"])
    near = tree.near_csr()
    near.sort_indices()
    assert near.nnz == int(g[prefix + "near_nnz"])
    assert np.array_equal(near.indptr.astype(np.int64), g[prefix + "near_indptr"])
    assert _sha(near.indptr.astype(np.int64), near.indices.astype(np.int64)) == g[prefix + "near_pattern_sha"].item().decode()
    if tree.depth >= 2:
        assert sorted(tree.orders.items()) == [tuple(r) for r in g[prefix + "orders"].tolist()]
        keys, counts, digest = _m2l_digest(tree)
        assert np.array_equal(keys, g[prefix + "m2l_keys"])
        assert np.array_equal(counts, g[prefix + "m2l_counts"])
        assert digest == g[prefix + "m2l_pairs_sha"].item().decode()
        n2 = tree.orders[tree.depth] ** 2
        idx = (tree.key[:, None] * n2 + np.arange(n2)[None, :]).ravel().astype(np.int64)
        assert _sha(idx) == g[prefix + "interp_indices_sha"].item().decode()
    return near


@pytest.mark.parametrize("name", list(cases.tree_cases()))
def test_oracle_tree_matches_reference(name):
    pts, spec, n_cheb, leaf, nvec = cases.tree_cases()[name]
    g = _load(f"tree_{name}.npz")
    tree = O.OracleTree(pts, _kern(spec), n_cheb, leaf)
    near = check_tree_ints(tree, g)
    # float operators: same formulas, so equal to roundoff
    if "op_near_data" in g:
        np.testing.assert_allclose(near.data, g["op_near_data"], rtol=1e-13, atol=1e-300)
    if tree.depth >= 2:
        np.testing.assert_allclose(tree.w2, g["op_interp_data"], rtol=0, atol=1e-14)
        for key, val in g.items():
            if key.startswith("op_m2l_"):
                lev, dx, dy = (int(v) for v in key[len("op_m2l_"):].split("_"))
                np.testing.assert_allclose(tree.m2l_ops[(lev, dx, dy)], val, rtol=1e-14, atol=1e-300)
            if key.startswith("op_shift_"):
                lev, c = key[len("op_shift_"):].split("_")
                np.testing.assert_allclose(tree.shift[int(lev)][(int(c[0]), int(c[1]))], val, rtol=0, atol=1e-14)
    U = tree.matmat(g["V"])
    assert O.rel_fro(U, g["U"]) <= 1e-13


def test_oracle_spd_solve():
    g = _load("spd_solve.npz")
    np.testing.assert_allclose(O.spd_solve(g["A"], g["B"]), g["X"], rtol=1e-13)
    with pytest.raises(O.OracleDecompositionError):
        O.spd_solve(np.diag([1.0, -1.0]), np.ones(2))
    with pytest.raises(ValueError):
        O.spd_solve(np.array([[2.0, 1.0], [0.0, 2.0]]), np.ones(2))


def test_oracle_update_cases():
    g = _load("update_cases.npz")
    for i, (st, Hm, r, z) in enumerate(cases.update_cases()):
        out = O.update(O.State(st["mean"], st["cross_cov"], st["variance"], st["HC"]),
                       scipy.sparse.csr_matrix(Hm), r, z)
        for k in ("mean", "cross_cov", "variance", "HC"):
            np.testing.assert_allclose(getattr(out, k), g[f"c{i}_{k}"], rtol=1e-12, atol=1e-14)
    # negative posterior variance is an error (tests/test_filters.py:233-244)
    bad = O.State(np.zeros(1), np.array([[3.0]]), np.array([1.0]), np.array([[4.0]]))
    with pytest.raises(O.OracleConsistencyError):
        O.update(bad, scipy.sparse.csr_matrix(np.array([[1.0]])), 0.0, np.array([0.0]))


def _scenario(cfg):
    N = cfg["N"]
    xy = O.cell_centers(N, N, 1.0 / N, 1.0 / N)
    src, rcv = O.crosswell_stations(cfg["ns"], cfg["nr"], 0.0, 1.0, 0.0, 1.0)
    H = O.ray_operator(N, N, 1.0 / N, 1.0 / N, src, rcv)
    return xy, H


@pytest.mark.parametrize("fixture,cfg", [("small_rays.npz", cases.SMALL), ("cfg1.npz", cases.CFG1)])
def test_oracle_filter_matches_reference(fixture, cfg):
    g = _load(fixture)
    xy, H = _scenario(cfg)
    # ray operator: bit-exact pattern, values to roundoff
    assert np.array_equal(H.indptr.astype(np.int64), g["H_indptr"])
    assert np.array_equal(H.indices.astype(np.int64), g["H_indices"])
    np.testing.assert_allclose(H.data, g["H_data"], rtol=1e-15, atol=0)
    fields = cases.plume_fields(xy, cfg["T"])
    obs = O.observations(H, fields, cfg["R"], [cfg["seed"], 0])
    np.testing.assert_array_equal(obs, g["obs"])
    kern = O.Kern(cfg["family"], 1.0, cfg["L"])
    tree = O.OracleTree(xy, kern, cfg["order"], cfg["leaf"])
    check_tree_ints(tree, g)
    pre = O.precompute(H, tree)
    assert O.rel_fro(pre.C_Q, g["C_Q"]) <= 1e-14
    st = O.init_state(H, len(xy))
    for t in range(cfg["T"]):
        st = O.update(O.predict(st, pre), H, cfg["R"], g["obs"][t])
    assert O.rel_fro(st.mean, g["final_mean"]) <= 1e-11
    assert O.rel_fro(st.variance, g["final_variance"]) <= 1e-11
    assert O.rel_fro(st.cross_cov, g["final_cross_cov"]) <= 1e-11


def test_oracle_cfg4_pins():
    """cfg4 (m = 1,048,576): tree depth/orders and the ray-operator pattern."""
    g = _load("cfg4_pins.npz")
    cfg = cases.CFG4
    N = cfg["N"]
    xy = O.cell_centers(N, N, 1.0 / N, 1.0 / N)
    lo = xy.min(axis=0)
    size = float(max(xy.max(axis=0) - lo)) * (1.0 + 1e-12)
    assert size == float(g["root_size"])
    depth = O.choose_depth(xy, lo, size, cfg["leaf"])
    assert depth == int(g["depth"])
    orders = O.select_orders(O.Kern(cfg["family"], 1.0, cfg["L"]), cfg["order"], depth, size)
    assert sorted(orders.items()) == [tuple(r) for r in g["orders"].tolist()]
    src, rcv = O.crosswell_stations(cfg["ns"], cfg["nr"], 0.0, 1.0, 0.0, 1.0)
    H = O.ray_operator(N, N, 1.0 / N, 1.0 / N, src, rcv)
    assert H.nnz == int(g["H_nnz"])
    assert _sha(H.indptr.astype(np.int64), H.indices.astype(np.int64)) == g["H_pattern_sha"].item().decode()
    assert _sha(H.data) == g["H_data_sha"].item().decode()


DENSE_CASES = [("small", cases.SMALL), ("cfg1", cases.CFG1),
               ("small_log", dict(cases.SMALL, N=16, ns=3, nr=4, family="logarithm", T=6))]


@pytest.mark.parametrize("name,cfg", DENSE_CASES)
def test_oracle_dense_precompute_matches_reference(name, cfg):
    """hikf_precompute_dense (filters.py:108-115) and the filter run on it."""
    g = _load("dense_cases.npz")
    xy, H = _scenario(cfg)
    kern = (O.Kern("logarithm", log_amplitude=-0.5) if cfg["family"] == "logarithm"
            else O.Kern(cfg["family"], 1.0, cfg["L"]))
    pre = O.precompute_dense(H, xy, kern)
    assert O.rel_fro(pre.C_Q, g[f"{name}_C_Q"]) <= 1e-14
    assert O.rel_fro(pre.HC_Q, g[f"{name}_HC_Q"]) <= 1e-14
    np.testing.assert_array_equal(pre.diag_Q, g[f"{name}_diag_Q"])
    if cfg["family"] == "logarithm":
        return
    st = O.init_state(H, len(xy))
    for t in range(cfg["T"]):
        st = O.update(O.predict(st, pre), H, cfg["R"], g[f"{name}_obs"][t])
    assert O.rel_fro(st.mean, g[f"{name}_final_mean"]) <= 1e-11
    assert O.rel_fro(st.variance, g[f"{name}_final_variance"]) <= 1e-11
    assert O.rel_fro(st.cross_cov, g[f"{name}_final_cross_cov"]) <= 1e-11


def test_oracle_cfg4_proxy_tree_and_qht_columns():
    """cfg4-proxy (m = 262,144, n = 1024, order 6, depth 6; make_golden.py --proxy):
    the oracle's tree integers and the ray operator bit-exact, and its bbFMM
    Q H^T on 2 of the reference's 8 sampled columns (matmat is
    column-independent, fmm.py:325-367) to reassociation roundoff."""
    g = _load("cfg4_proxy.npz")
    N, ns, nr, order, leaf = 512, 32, 32, 6, 64
    xy = O.cell_centers(N, N, 1.0 / N, 1.0 / N)
    src, rcv = O.crosswell_stations(ns, nr, 0.0, 1.0, 0.0, 1.0)
    H = O.ray_operator(N, N, 1.0 / N, 1.0 / N, src, rcv)
    assert H.nnz == int(g["H_nnz"])
    assert _sha(H.indptr.astype(np.int64), H.indices.astype(np.int64)) == g["H_pattern_sha"].item().decode()
    assert _sha(H.data) == g["H_data_sha"].item().decode()
    tree = O.OracleTree(xy, O.Kern("exponential", 1.0, 0.25), order, leaf)
    check_tree_ints(tree, g)
    rows, cols = g["rows"], g["cols"]
    pick = [0, 7]  # first ray and one interior ray of the sampled columns
    U = tree.matmat(np.ascontiguousarray(H[cols[pick]].T.toarray()))
    assert O.rel_fro(U[rows], g["C_Q_sample"][:, pick]) <= 1e-13
    np.testing.assert_allclose(U.sum(axis=0), g["C_Q_colsum"][cols[pick]], rtol=1e-13)
