"""Parity at BASELINE-sized problems.

* cfg4-proxy (m = 262,144, n = 1024, order 6, depth 6): the largest
  BASELINE-shaped case the real reference runs in the build container's RAM.
  Fixture ``cfg4_proxy.npz`` (make_golden.py --proxy) holds the reference's
  tree integers, C_Q / HC_Q fingerprints, and the state after all T = 50
  filter steps: the full final mean, variance and HC, per-step means on a row
  sample, and every column's norm plus seeded sketches of the final cross
  covariance.
* cfg4 itself (m = 1,048,576, n = 1024): the reference needs > 62 GB for it,
  so the GPU Q H^T is checked column-wise against the oracle's bbFMM
  (matmat is column-independent, fmm.py:325-367), the near-pair and M2L
  interaction lists against the oracle's, and all 50 steps of the fused
  update (explicit and factored) against a plain torch float64 restatement of
  hikf_predict / hikf_update (filters.py:129-157: Cholesky, m-RHS solve, K HC)
  on the same device-resident C_Q.
"""

import os

import numpy as np
import pytest

from oracle import hikf_oracle as O
from tests.golden import cases
from tests.test_gpu_parity import PARITY, _Model, _gpu_scenario, _load, _record, _sha, _spec, check_tree_ints  # noqa: F401

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CFG4_PROXY = dict(name="cfg4_proxy", N=512, ns=32, nr=32, family="exponential", L=0.25, R=1e-3, T=50, order=6,
                  leaf=64, seed=0)


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1404_3816_b200 as p
    return p


def _sketch_errs(torch, A_t, g, prefix, gm, gn):
    """Relative errors of the size-independent fingerprints of an m x n device
    array against the reference's (make_golden.sketches): the worst column
    norm, the column sketch A^T g_m, the row sketch A g_n, the Frobenius norm."""
    cn = torch.linalg.norm(A_t, dim=0).cpu().numpy()
    ref_cn = g[prefix + "col_norms"]
    return {
        prefix + "col_norms": O.rel_fro(cn, ref_cn),
        prefix + "col_norms_worst_column": float(np.max(np.abs(cn - ref_cn) / ref_cn)),
        prefix + "col_sketch": O.rel_fro((A_t.T @ gm).cpu().numpy(), g[prefix + "col_sketch"]),
        prefix + "row_sketch": O.rel_fro((A_t @ gn).cpu().numpy(), g[prefix + "row_sketch"]),
        prefix + "fro": abs(float(torch.linalg.norm(A_t)) - float(g[prefix + "fro"])) / float(g[prefix + "fro"]),
    }


@pytest.fixture(scope="module")
def proxy(pkg):
    """The cfg4-proxy scenario on the device (H, tree, precompute) + the reference fixture."""
    g = _load("cfg4_proxy.npz")
    cfg = CFG4_PROXY
    grid, H = _gpu_scenario(pkg, cfg)
    kern = pkg.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
    model = _Model(grid, H, kern, cfg["R"])
    tree = pkg.build_tree(grid.cell_centers(), kern, pkg.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    pre = pkg.filters.hikf_precompute_fmm(model, tree)
    return g, cfg, grid, H, model, tree, pre


def test_cfg4_proxy_tree_and_qht_match_reference(pkg, proxy):
    """Tree integers bit-exact, and C_Q = Q H^T (all 1024 columns through their
    norms and a seeded sketch, plus a row x column sample) against the reference."""
    import torch
    g, cfg, grid, H, model, tree, pre = proxy
    assert H.nnz == int(g["H_nnz"])
    assert _sha(H.indptr.astype(np.int64), H.indices.astype(np.int64)) == g["H_pattern_sha"].item().decode()
    assert _sha(H.data) == g["H_data_sha"].item().decode()
    check_tree_ints(tree, g)
    gm_np, gn_np = cases.sketch_vectors(grid.m, H.shape[0])
    gm, gn = torch.as_tensor(gm_np).cuda(), torch.as_tensor(gn_np).cuda()
    rows, cols = g["rows"], g["cols"]
    C_Q = pre.C_Q_t
    errs = _sketch_errs(torch, C_Q, g, "C_Q_", gm, gn)
    errs.update({
        "C_Q_sample": O.rel_fro(C_Q[torch.as_tensor(rows).cuda()][:, torch.as_tensor(cols).cuda()].cpu().numpy(),
                                g["C_Q_sample"]),
        "C_Q_colsum": O.rel_fro(C_Q.sum(dim=0).cpu().numpy(), g["C_Q_colsum"]),
        "HC_Q_block": O.rel_fro(pre.HC_Q[:64, :64], g["HC_Q_block"]),
        "HC_Q_fro": abs(np.linalg.norm(pre.HC_Q) - float(g["HC_Q_fro"])) / float(g["HC_Q_fro"]),
        "HC_Q_col_norms_max": float(np.max(np.abs(np.linalg.norm(pre.HC_Q, axis=0) - g["HC_Q_col_norms"]) /
                                           g["HC_Q_col_norms"])),
    })
    _record("cfg4_proxy_qht", errs)
    for k, v in errs.items():
        assert v <= (1e-13 if "worst_column" not in k else 1e-12), (k, v)


@pytest.mark.parametrize("representation", ["explicit", "factored"])
def test_cfg4_proxy_50_steps_match_reference(pkg, proxy, representation):
    """All T = 50 predict/update steps of the cfg4-proxy (m = 262,144, n = 1024)
    in run_hikf's order (experiment.py:232-236, filters.py:129-157) against the
    real reference: the full final mean, variance and HC, the per-step means on
    a row sample, and the final cross covariance through every column's norm, a
    seeded column / row sketch, a row x column sample and its Frobenius norm.
    North-star gate: relative Frobenius <= 1e-9 (PARITY); the margins are
    recorded in gpurun_out/parity_errors.jsonl."""
    import torch
    g, cfg, grid, H, model, tree, pre = proxy
    flt = pkg.filters
    rows, cols = g["rows"], g["cols"]
    st = flt.hikf_init(model, representation=representation)
    step_means, step_norms = [], []
    for t in range(cfg["T"]):
        st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], g["obs"][t])
        step_means.append(st.mean[rows])
        step_norms.append(np.linalg.norm(st.mean))
    gm_np, gn_np = cases.sketch_vectors(grid.m, H.shape[0])
    gm, gn = torch.as_tensor(gm_np).cuda(), torch.as_tensor(gn_np).cuda()
    C = st.cross_cov_t
    errs = {
        "mean": O.rel_fro(st.mean, g["final_mean"]),
        "variance": O.rel_fro(st.variance, g["final_variance"]),
        "HC": O.rel_fro(st.HC, g["final_HC"]),
        "step_means": O.rel_fro(np.array(step_means), g["step_means_sample"]),
        "step_mean_norms_max": float(np.max(np.abs(np.array(step_norms) - g["step_mean_norms"]) /
                                            g["step_mean_norms"])),
        "cross_cov_sample": O.rel_fro(C[torch.as_tensor(rows).cuda()][:, torch.as_tensor(cols).cuda()].cpu().numpy(),
                                      g["final_cross_cov_sample"]),
    }
    errs.update(_sketch_errs(torch, C, g, "final_cross_cov_", gm, gn))
    _record(f"cfg4_proxy_50_steps_{representation}", errs)
    worst = max(errs.values())
    print(f"cfg4-proxy 50 steps ({representation}): worst {worst:.3g}, margin {PARITY / max(worst, 1e-300):.3g}x", errs)
    for k, v in errs.items():
        # a single column's own relative error is not the north-star metric: 10x looser gate
        assert v <= (PARITY if "worst_column" not in k else 10 * PARITY), (k, v)


@pytest.fixture(scope="module")
def cfg4(pkg):
    """The full cfg4 scenario on the device: H, tree, precompute."""
    cfg = cases.CFG4
    grid, H = _gpu_scenario(pkg, cfg)
    kern = pkg.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
    model = _Model(grid, H, kern, cfg["R"])
    tree = pkg.build_tree(grid.cell_centers(), kern, pkg.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    pre = pkg.filters.hikf_precompute_fmm(model, tree)
    return cfg, grid, H, model, tree, pre


def test_cfg4_pins_and_qht_columns_against_oracle(pkg, cfg4):
    """Tree depth / orders and the ray operator against the reference's cfg4
    pins; Q H^T columns against the oracle bbFMM on the same tree (the oracle
    is pinned to the reference on 12 trees and the cfg4-proxy)."""
    cfg, grid, H, model, tree, pre = cfg4
    pins = _load("cfg4_pins.npz")
    assert tree.depth == int(pins["depth"]) and tree.root_size == float(pins["root_size"])
    assert sorted(tree._orders.items()) == [tuple(r) for r in pins["orders"].tolist()]
    assert _sha(H.indptr.astype(np.int64), H.indices.astype(np.int64)) == pins["H_pattern_sha"].item().decode()
    assert _sha(H.data) == pins["H_data_sha"].item().decode()
    xy = grid.cell_centers().coords
    otree = O.OracleTree(xy, O.Kern(cfg["family"], 1.0, cfg["L"]), cfg["order"], cfg["leaf"])
    assert otree.depth == tree.depth and otree.orders == tree._orders
    ex = tree.export()
    assert np.array_equal(ex["order"], otree.order)
    assert np.array_equal(ex["leaf_ids"], otree.leaf_ids) and np.array_equal(ex["leaf_starts"], otree.leaf_starts)
    # near leaf pairs (fmm.py:166-201) bit-exact against the oracle's (145,924 pairs, 597.7 M point pairs)
    ot, os_ = otree.near_pairs
    got = np.stack([ex["near_t"], ex["near_s"]], axis=1).astype(np.int64)
    want = np.stack([np.asarray(ot), np.asarray(os_)], axis=1).astype(np.int64)
    assert got.shape == want.shape == (145924, 2)
    assert np.array_equal(got[np.lexsort(got.T[::-1])], want[np.lexsort(want.T[::-1])])
    assert int((otree.leaf_counts[want[:, 0]] * otree.leaf_counts[want[:, 1]]).sum()) == 145924 * 64 * 64  # near nnz
    # every M2L interaction list (fmm.py:299-312) against the real reference's cfg4 lists (cfg4_pins.npz,
    # FmmTree._build_m2l on the cfg4 tree) and the oracle's
    import hashlib
    keys, counts, h = [], [], hashlib.sha256()
    for lev in range(2, tree.depth + 1):
        for dx, dy in O.m2l_offsets():
            t_, s_ = tree.m2l_pairs(lev, dx, dy)
            if len(t_):
                keys.append((lev, dx, dy))
                counts.append(len(t_))
                ot_, os2 = otree.m2l_pairs[(lev, dx, dy)]
                assert np.array_equal(t_, ot_) and np.array_equal(s_, os2), (lev, dx, dy)
    for key in sorted(keys):
        t_, s_ = tree.m2l_pairs(*key)
        h.update(t_.astype(np.int64).tobytes())
        h.update(s_.astype(np.int64).tobytes())
    assert np.array_equal(np.array(sorted(keys), dtype=np.int64), pins["m2l_keys"])
    assert np.array_equal(np.array([c for _, c in sorted(zip(keys, counts))], dtype=np.int64), pins["m2l_counts"])
    assert h.hexdigest() == pins["m2l_pairs_sha"].item().decode()
    sel = np.array([0, 341, 682, 1023])  # first / interior / last rays (one horizontal on a gridline)
    U = otree.matmat(np.ascontiguousarray(H[sel].T.toarray()))
    got = pre.C_Q_t[:, sel].cpu().numpy()
    errs = {f"C_Q_col{j}": O.rel_fro(got[:, i], U[:, i]) for i, j in enumerate(sel)}
    errs["C_Q_cols"] = O.rel_fro(got, U)
    _record("cfg4_qht_vs_oracle", errs)
    assert errs["C_Q_cols"] <= 1e-13, errs
    # HC_Q = sym(H C_Q) (filters.py:103-104): symmetric to the bit, against a host restatement on the columns
    HCQ = pre.HC_Q_t.cpu().numpy()
    assert np.array_equal(HCQ, HCQ.T)
    import torch
    hrows = torch.as_tensor(H[sel].toarray()).cuda()
    HC_rows = (hrows @ pre.C_Q_t).cpu().numpy()  # (H C_Q)[sel, :]
    assert O.rel_fro(HCQ[:, sel], 0.5 * (H @ got + HC_rows.T)) <= 1e-13


def test_cfg4_50_steps_against_torch_fp64(pkg, cfg4):
    """All T = 50 steps of the cfg4 experiment (C is 8.6 GB), explicit and
    factored updates in lockstep with a plain torch float64 restatement of the
    reference's predict / update (filters.py:129-157: Cholesky of the
    symmetrised S, m-RHS cholesky_solve for K, K HC) on the same device C_Q;
    relative Frobenius errors of mean, variance, cross_cov and HC every 10
    steps (recorded), gate PARITY = 1e-9 at every checkpoint."""
    import torch
    cfg, grid, H, model, tree, pre = cfg4
    flt = pkg.filters
    T = cfg["T"]
    obs = O.observations(H, O.moving_plume(grid.cell_centers().coords, T), cfg["R"], [cfg["seed"], 0])
    Hd = torch.sparse_csr_tensor(torch.as_tensor(H.indptr, dtype=torch.int64),
                                 torch.as_tensor(H.indices, dtype=torch.int64), torch.as_tensor(H.data),
                                 size=H.shape).cuda()
    dev = pre.C_Q_t.device
    m, n = pre.C_Q_t.shape
    f64 = dict(dtype=torch.float64, device=dev)
    ref = {"mean": torch.zeros(m, **f64), "C": torch.zeros(m, n, **f64), "var": torch.zeros(m, **f64),
           "HC": torch.zeros(n, n, **f64)}
    eye = torch.eye(n, **f64)
    ex = flt.hikf_init(model)
    fa = flt.hikf_init(model, representation="factored")

    def rf(a, b):
        return float(torch.linalg.norm(a - b) / torch.linalg.norm(b))

    worst = 0.0
    for t in range(T):
        ex = flt.hikf_update(flt.hikf_predict(ex, pre), H, cfg["R"], obs[t])
        fa = flt.hikf_update(flt.hikf_predict(fa, pre), H, cfg["R"], obs[t])
        C = ref["C"] + pre.C_Q_t
        var = ref["var"] + pre.diag_Q_t
        HC = ref["HC"] + pre.HC_Q_t
        S = HC + cfg["R"] * eye
        S = 0.5 * (S + S.T)
        L = torch.linalg.cholesky(S)
        K = torch.cholesky_solve(C.T.contiguous(), L).T
        innov = torch.as_tensor(obs[t], device=dev) - Hd @ ref["mean"]
        ref["var"] = var - (K * C).sum(dim=1)
        ref["mean"] = ref["mean"] + K @ innov
        KH = torch.cholesky_solve(HC.T.contiguous(), L).T
        ref["C"] = C - K @ HC
        ref["HC"] = HC - KH @ HC
        del K, C
        if (t + 1) % 10 == 0 or t + 1 == T:
            for name, st in (("explicit", ex), ("factored", fa)):
                errs = {"mean": rf(st.mean_t, ref["mean"]), "variance": rf(st.variance_t, ref["var"]),
                        "cross_cov": rf(st.cross_cov_t, ref["C"]), "HC": rf(st.HC_t, ref["HC"])}
                _record(f"cfg4_{name}_vs_torch_step{t + 1}", errs)
                worst = max(worst, *errs.values())
                for k, v in errs.items():
                    assert v <= PARITY, (name, t + 1, k, v)
    print(f"cfg4 50 steps vs torch fp64: worst {worst:.3g}")


def test_dgemm_beyond_2_31_elements(pkg):
    """The K-GEMM shape of cfg5 and beyond: M = 2^21 + 37 rows x 1024 (2.15e9 elements per
    operand, past the int32 element range) through the CUTLASS-mainloop variant, checked
    against torch (cuBLAS) on row slices at the start, the middle and the end."""
    import torch
    from paper_1404_3816_b200 import _lib
    lib = _lib.load()
    M, N, K = (1 << 21) + 37, 1024, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(M, N, dtype=torch.float64, device="cuda")
    _lib.check(lib.hikf_dgemm(M, N, K, A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, 1.0, 0.0, 0, 30,
                              _lib.stream_ptr()))
    for r0 in (0, M // 2 - 1000, M - 4096):
        ref = A[r0:r0 + 4096] @ B
        err = float((C[r0:r0 + 4096] - ref).abs().max() / ref.abs().max())
        assert err <= 1e-14, (r0, err)
    del A, B, C
    torch.cuda.empty_cache()
