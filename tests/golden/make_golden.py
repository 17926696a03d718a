"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big | --dense | --proxy]

Every fixture is produced by the reference ``hikf`` package's own public API
(build_tree / FmmTree.matmat / hikf_precompute_fmm / hikf_init /
hikf_predict / hikf_update / spd_solve / build_ray_operator), on seeded inputs
whose recipe is restated in ``tests/golden/cases.py``.  ``--big`` also runs
cfg2 (m = 65,536, n = 256, 100 steps; about two minutes) and the cfg4
tree-order/ray-operator pins (no cfg4 matmat: it needs > 62 GB here).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np
import scipy.sparse

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

from hikf import filters as flt  # noqa: E402
from hikf.fmm import FmmConfig, FmmTree, build_tree  # noqa: E402
from hikf.grids import Grid2D, PointSet  # noqa: E402
from hikf.kernels import KernelSpec  # noqa: E402
from hikf.linalg import spd_solve  # noqa: E402
from hikf.ssm import StateSpaceModel, simulate_truth_and_data  # noqa: E402
from hikf.tomography import PlumeScenario, build_ray_operator, default_acquisition  # noqa: E402

from golden import cases  # noqa: E402  (tests/golden/cases.py)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def tree_ints(tree: FmmTree) -> dict:
    """Integer / index data of a reference tree (SURVEY 8(c) bit-exact list)."""
    out = {
        "depth": np.int64(tree.depth),
        "root_lo": np.asarray(tree.root_lo, dtype=float),
        "root_size": np.float64(tree.root_size),
        "order": tree._order.astype(np.int64),
        "leaf_ids": tree._leaf_ids.astype(np.int64),
        "leaf_starts": tree._leaf_starts.astype(np.int64),
        "leaf_counts": tree._leaf_counts.astype(np.int64),
        "near_indptr": tree.near.indptr.astype(np.int64),
        "near_nnz": np.int64(tree.near.nnz),
        "near_pattern_sha": np.bytes_(sha(*_near_pattern(tree))),
    }
    if tree.depth >= 2:
        levs = sorted(tree._orders)
        out["orders"] = np.array([[lev, tree._orders[lev]] for lev in levs], dtype=np.int64)
        keys, counts, digest = [], [], hashlib.sha256()
        for key in sorted(tree._m2l_pairs):
            t, s = tree._m2l_pairs[key]
            keys.append(key)
            counts.append(len(t))
            digest.update(np.asarray(t, dtype=np.int64).tobytes())
            digest.update(np.asarray(s, dtype=np.int64).tobytes())
        out["m2l_keys"] = np.array(keys, dtype=np.int64)
        out["m2l_counts"] = np.array(counts, dtype=np.int64)
        out["m2l_pairs_sha"] = np.bytes_(digest.hexdigest())
        out["interp_indices_sha"] = np.bytes_(sha(tree._interp.indices.astype(np.int64)))
    return out


def _near_pattern(tree):
    """Row-sorted near pattern: (row, col) pairs in canonical order."""
    nr = tree.near.copy()
    nr.sort_indices()
    return nr.indptr.astype(np.int64), nr.indices.astype(np.int64)


PINNED_OFFSETS = {(2, 0), (-3, 2), (0, -2), (3, 3)}


def tree_small_floats(tree: FmmTree) -> dict:
    """Operators of a small tree, to pin the oracle's float restatement."""
    out = {}
    if tree.depth >= 2:
        for lev in range(2, tree.depth + 1):
            for (l, dx, dy), M in tree._m2l_ops.items():
                if l == lev and (dx, dy) in PINNED_OFFSETS:
                    out[f"m2l_{lev}_{dx}_{dy}"] = M
        for lev, ops in tree._shift.items():
            for (cx, cy), C in ops.items():
                out[f"shift_{lev}_{cx}{cy}"] = C
        out["interp_data"] = tree._interp.data.reshape(tree.m, -1)
    nr = tree.near.copy()
    nr.sort_indices()
    if nr.nnz <= 150_000:
        out["near_data"] = nr.data
    return out


def scenario(cfg: dict):
    """Reference objects for one BASELINE-style crosswell scenario."""
    N = cfg["N"]
    grid = Grid2D(nx=N, ny=N, dx=1.0 / N, dy=1.0 / N)
    acq = default_acquisition(grid, cfg["ns"], cfg["nr"], source_x=0.0, receiver_x=1.0)
    H = build_ray_operator(grid, acq)
    kern = KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
    model = StateSpaceModel(grid=grid, H=H, q_kernel=kern, r_variance=cfg["R"], alpha=cfg.get("alpha", 0.0))
    fields = cases.plume_fields(grid.cell_centers().coords, cfg["T"])
    record = simulate_truth_and_data(model, PlumeScenario(fields), seed=[cfg["seed"], 0])
    return grid, H, kern, model, record


def run_filter(cfg: dict, full: bool) -> dict:
    """One BASELINE-style scenario through the reference (experiment.py:232-236
    loop order).  Besides the final state: the mean after every step (all rows
    when m <= 4096, else every 16th row), and for C_Q and the final cross
    covariance every column's norm plus seeded column / row sketches; ``full``
    stores both arrays whole, else 32 evenly spaced full columns of each."""
    grid, H, kern, model, record = scenario(cfg)
    t0 = time.perf_counter()
    tree = build_tree(grid.cell_centers(), kern, FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    t_tree = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = flt.hikf_precompute_fmm(model, tree)
    t_pre = time.perf_counter() - t0
    state = flt.hikf_init(model)
    rows = np.arange(grid.m) if grid.m <= 4096 else np.arange(0, grid.m, 16)
    step_means = []
    t0 = time.perf_counter()
    for t in range(cfg["T"]):
        state = flt.hikf_update(flt.hikf_predict(state, pre), H, model.r_variance, record.observations[t])
        step_means.append(state.mean[rows])
    t_on = time.perf_counter() - t0
    print(f"  {cfg['name']}: depth {tree.depth} orders {getattr(tree, '_orders', {})} tree {t_tree:.2f}s precompute {t_pre:.2f}s online {t_on:.2f}s", flush=True)
    out = {f"tree_{k}": v for k, v in tree_ints(tree).items()}
    gm, gn = cases.sketch_vectors(grid.m, H.shape[0])
    out.update({f"C_Q_{k}": v for k, v in sketches(pre.C_Q, gm, gn).items()})
    out.update({f"final_cross_cov_{k}": v for k, v in sketches(state.cross_cov, gm, gn).items()})
    out.update({
        "H_indptr": H.indptr.astype(np.int64), "H_indices": H.indices.astype(np.int64),
        "H_data": H.data, "obs": record.observations,
        "final_mean": state.mean, "final_variance": state.variance,
        "cross_cov_fro": np.float64(np.linalg.norm(state.cross_cov)),
        "HC_Q": pre.HC_Q, "final_HC": state.HC,
        "step_rows": rows, "step_means": np.array(step_means),
    })
    if full:
        out["C_Q"] = pre.C_Q
        out["final_cross_cov"] = state.cross_cov
    else:
        cols = np.arange(0, H.shape[0], max(1, H.shape[0] // 32))
        out["cols"] = cols
        out["C_Q_cols"] = pre.C_Q[:, cols]
        out["final_cross_cov_cols"] = state.cross_cov[:, cols]
    return out


def alpha_cases() -> dict:
    """hikf_init with alpha = 0.5 (filters.py:118-126: C_0 = alpha H^T, var_0 =
    alpha, HC_0 = alpha H H^T) through the whole filter, small and cfg1."""
    out = {}
    for base in (cases.SMALL, cases.CFG1):
        cfg = dict(base, alpha=0.5)
        o = run_filter(cfg, full=True)
        for k in ("obs", "final_mean", "final_variance", "final_HC", "final_cross_cov", "step_means", "C_Q"):
            out[f"{base['name']}_{k}"] = o[k]
    return out


def dense_cases() -> dict:
    """hikf_precompute_dense (filters.py:108-115) + the filter on it: the
    reference's exact-algebra path (run_hikf mode "dense", experiment.py:224)."""
    out = {}
    log_case = dict(cases.SMALL, name="small_log", N=16, ns=3, nr=4, family="logarithm", T=6)
    for cfg in (cases.SMALL, cases.CFG1, log_case):
        name = cfg["name"]
        grid, H, kern, model, record = scenario(cfg) if cfg["family"] != "logarithm" else _log_scenario(cfg)
        pre = flt.hikf_precompute_dense(model)
        out.update({f"{name}_C_Q": pre.C_Q, f"{name}_HC_Q": pre.HC_Q, f"{name}_diag_Q": pre.diag_Q})
        if cfg["family"] == "logarithm":  # conditionally PD only: precompute pinned, no filter run
            continue
        state = flt.hikf_init(model)
        for t in range(cfg["T"]):
            state = flt.hikf_update(flt.hikf_predict(state, pre), H, model.r_variance, record.observations[t])
        out.update({f"{name}_obs": record.observations, f"{name}_final_mean": state.mean,
                    f"{name}_final_variance": state.variance, f"{name}_final_cross_cov": state.cross_cov,
                    f"{name}_final_HC": state.HC})
        print(f"  dense {name}: m {model.m} n {H.shape[0]}", flush=True)
    return out


def _log_scenario(cfg: dict):
    N = cfg["N"]
    grid = Grid2D(nx=N, ny=N, dx=1.0 / N, dy=1.0 / N)
    acq = default_acquisition(grid, cfg["ns"], cfg["nr"], source_x=0.0, receiver_x=1.0)
    H = build_ray_operator(grid, acq)
    kern = KernelSpec("logarithm", log_amplitude=-0.5)
    model = StateSpaceModel(grid=grid, H=H, q_kernel=kern, r_variance=cfg["R"], alpha=0.0)
    fields = cases.plume_fields(grid.cell_centers().coords, cfg["T"])
    record = simulate_truth_and_data(model, PlumeScenario(fields), seed=[cfg["seed"], 0])
    return grid, H, kern, model, record


CFG4_PROXY = dict(name="cfg4_proxy", N=512, ns=32, nr=32, family="exponential", L=0.25, R=1e-3, T=50, order=6, leaf=64,
                  seed=0)


def sketches(A: np.ndarray, gm: np.ndarray, gn: np.ndarray) -> dict:
    """Size-independent fingerprints of an m x n array: every column's norm,
    A^T g_m (one number per column) and A g_n (one number per row)."""
    return {"col_norms": np.linalg.norm(A, axis=0), "col_sketch": A.T @ gm, "row_sketch": A @ gn,
            "fro": np.float64(np.linalg.norm(A))}


def cfg4_proxy() -> dict:
    """SURVEY 8(d) cfg4-proxy (m = 262,144, n = 1024, order 6, depth 6): the
    largest BASELINE-shaped case the reference runs in this container's RAM.
    Full reference precompute + all T = 50 filter steps (experiment.py:232-236
    order: predict then update).  Stored: the full final mean, variance and HC,
    per-step means on a row sample, and for C_Q and the final cross_cov every
    column's norm, a seeded column / row sketch, a row x column sample and the
    Frobenius norm (the arrays themselves are 2 GB each)."""
    cfg = CFG4_PROXY
    grid, H, kern, model, record = scenario(cfg)
    t0 = time.perf_counter()
    tree = build_tree(grid.cell_centers(), kern, FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    t_tree = time.perf_counter() - t0
    out = {f"tree_{k}": v for k, v in tree_ints(tree).items()}
    t0 = time.perf_counter()
    pre = flt.hikf_precompute_fmm(model, tree)
    t_pre = time.perf_counter() - t0
    rows = np.arange(0, grid.m, 64)
    cols = np.arange(0, H.shape[0], H.shape[0] // 8)
    gm, gn = cases.sketch_vectors(grid.m, H.shape[0])
    out.update({f"C_Q_{k}": v for k, v in sketches(pre.C_Q, gm, gn).items()})
    out.update({
        "H_nnz": np.int64(H.nnz),
        "H_pattern_sha": np.bytes_(sha(H.indptr.astype(np.int64), H.indices.astype(np.int64))),
        "H_data_sha": np.bytes_(sha(H.data)),
        "rows": rows, "cols": cols,
        "C_Q_sample": pre.C_Q[np.ix_(rows, cols)], "C_Q_colsum": pre.C_Q.sum(axis=0),
        "HC_Q_block": pre.HC_Q[:64, :64], "HC_Q_fro": np.float64(np.linalg.norm(pre.HC_Q)),
        "HC_Q_col_norms": np.linalg.norm(pre.HC_Q, axis=0),
    })
    state = flt.hikf_init(model)
    step_means, step_norms, step_s = [], [], []
    for t in range(cfg["T"]):
        t0 = time.perf_counter()
        state = flt.hikf_update(flt.hikf_predict(state, pre), H, model.r_variance, record.observations[t])
        step_s.append(time.perf_counter() - t0)
        step_means.append(state.mean[rows])
        step_norms.append(np.linalg.norm(state.mean))
        print(f"    step {t}: {step_s[-1]:.1f}s", flush=True)
    t_on = float(np.sum(step_s))
    out.update({f"final_cross_cov_{k}": v for k, v in sketches(state.cross_cov, gm, gn).items()})
    out.update({
        "obs": record.observations[:cfg["T"]],
        "step_means_sample": np.array(step_means), "step_mean_norms": np.array(step_norms),
        "final_mean": state.mean, "final_variance": state.variance, "final_HC": state.HC,
        "final_cross_cov_sample": state.cross_cov[np.ix_(rows, cols)],
        "ref_seconds": np.array([t_tree, t_pre, t_on]), "ref_step_seconds": np.array(step_s),
    })
    print(f"  cfg4_proxy: depth {tree.depth} orders {tree._orders} tree {t_tree:.1f}s precompute {t_pre:.1f}s "
          f"online {t_on:.1f}s ({cfg['T']} steps)", flush=True)
    return out


def cfg4_pins():
    """cfg4: tree depth / orders, the ray operator, and the M2L interaction
    lists of the real reference (FmmTree._build_m2l on the cfg4 tree skeleton;
    the near field and the full build need > 62 GB here)."""
    N = 1024
    grid = Grid2D(nx=N, ny=N, dx=1.0 / N, dy=1.0 / N)
    H = build_ray_operator(grid, default_acquisition(grid, 32, 32, source_x=0.0, receiver_x=1.0))
    t = object.__new__(FmmTree)
    t.points = grid.cell_centers()
    t.kernel = KernelSpec("exponential", variance=1.0, length_scale=0.25)
    t.config = FmmConfig(n_cheb=6, max_leaf_points=64)
    t.m = grid.m
    lo, hi = t.points.bounding_box
    t.root_lo = lo
    t.root_size = float(max(hi - lo)) * (1.0 + 1e-12)
    t.depth = t._choose_depth(t.points.coords, lo, t.root_size)
    t._select_orders()
    t._build_m2l()
    keys, counts, digest = [], [], hashlib.sha256()
    for key in sorted(t._m2l_pairs):
        tt, ss = t._m2l_pairs[key]
        keys.append(key)
        counts.append(len(tt))
        digest.update(np.asarray(tt, dtype=np.int64).tobytes())
        digest.update(np.asarray(ss, dtype=np.int64).tobytes())
    np.savez_compressed(
        os.path.join(HERE, "cfg4_pins.npz"),
        depth=np.int64(t.depth), root_size=np.float64(t.root_size),
        orders=np.array(sorted(t._orders.items()), dtype=np.int64),
        H_indptr=H.indptr.astype(np.int64), H_nnz=np.int64(H.nnz),
        H_pattern_sha=np.bytes_(sha(H.indptr.astype(np.int64), H.indices.astype(np.int64))),
        H_data_sum=np.float64(H.data.sum()), H_data_sha=np.bytes_(sha(H.data)),
        m2l_keys=np.array(keys, dtype=np.int64), m2l_counts=np.array(counts, dtype=np.int64),
        m2l_pairs_sha=np.bytes_(digest.hexdigest()),
    )
    print(f"cfg4: depth {t.depth} orders {t._orders} nnz(H) {H.nnz} m2l keys {len(keys)} pairs {sum(counts)}")


def main(big: bool):
    if "--proxy" in sys.argv:  # only the cfg4-proxy fixture (about 13 minutes, ~16 GB RSS)
        np.savez_compressed(os.path.join(HERE, "cfg4_proxy.npz"), **cfg4_proxy())
        return
    if "--filters" in sys.argv:  # only the filter-run fixtures (small, cfg1, cfg2, alpha = 0.5; ~3 minutes)
        np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **run_filter(cases.CFG1, full=True))
        np.savez_compressed(os.path.join(HERE, "small_rays.npz"), **run_filter(cases.SMALL, full=True))
        np.savez_compressed(os.path.join(HERE, "alpha_cases.npz"), **alpha_cases())
        np.savez_compressed(os.path.join(HERE, "cfg2.npz"), **run_filter(cases.CFG2, full=False))
        return
    if "--cfg4pins" in sys.argv:  # only the cfg4 pins (seconds)
        cfg4_pins()
        return
    if "--dense" in sys.argv:  # only the dense-path fixtures (other fixtures untouched)
        np.savez_compressed(os.path.join(HERE, "dense_cases.npz"), **dense_cases())
        return
    os.makedirs(HERE, exist_ok=True)
    # 1) tree / matmat fixtures over the point-set cases
    for name, (pts, spec, n_cheb, leaf, nvec) in cases.tree_cases().items():
        ref_spec = KernelSpec(spec["family"], variance=spec.get("variance", 1.0),
                              length_scale=spec.get("length_scale", 1.0),
                              log_amplitude=spec.get("log_amplitude"))
        tree = build_tree(PointSet(pts), ref_spec, FmmConfig(n_cheb=n_cheb, max_leaf_points=leaf))
        V = cases.charges(len(pts), nvec)
        out = {f"tree_{k}": v for k, v in tree_ints(tree).items()}
        out.update({f"op_{k}": v for k, v in tree_small_floats(tree).items()})
        out["V"] = V
        out["U"] = tree.matmat(V)
        np.savez_compressed(os.path.join(HERE, f"tree_{name}.npz"), **out)
        print(f"tree_{name}: depth {tree.depth} orders {getattr(tree, '_orders', {})}", flush=True)

    # 2) spd_solve fixtures (linalg.py:18-37)
    A, B = cases.spd_case()
    np.savez_compressed(os.path.join(HERE, "spd_solve.npz"), A=A, B=B, X=spd_solve(A, B))

    # 3) hand-value filter cases (filters.py:138-157)
    hv = {}
    for i, (st, Hm, r, z) in enumerate(cases.update_cases()):
        s = flt.HikfState(mean=st["mean"], cross_cov=st["cross_cov"], variance=st["variance"], HC=st["HC"])
        o = flt.hikf_update(s, scipy.sparse.csr_matrix(Hm), r, z)
        for k in ("mean", "cross_cov", "variance", "HC"):
            hv[f"c{i}_{k}"] = getattr(o, k)
    np.savez_compressed(os.path.join(HERE, "update_cases.npz"), **hv)

    # 4) the BASELINE crosswell scenarios
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **run_filter(cases.CFG1, full=True))
    np.savez_compressed(os.path.join(HERE, "small_rays.npz"), **run_filter(cases.SMALL, full=True))
    np.savez_compressed(os.path.join(HERE, "alpha_cases.npz"), **alpha_cases())
    if big:
        np.savez_compressed(os.path.join(HERE, "cfg2.npz"), **run_filter(cases.CFG2, full=False))
        cfg4_pins()



if __name__ == "__main__":
    main("--big" in sys.argv)
