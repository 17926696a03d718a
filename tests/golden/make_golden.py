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
    model = StateSpaceModel(grid=grid, H=H, q_kernel=kern, r_variance=cfg["R"], alpha=0.0)
    fields = cases.plume_fields(grid.cell_centers().coords, cfg["T"])
    record = simulate_truth_and_data(model, PlumeScenario(fields), seed=[cfg["seed"], 0])
    return grid, H, kern, model, record


def run_filter(cfg: dict, full: bool) -> dict:
    grid, H, kern, model, record = scenario(cfg)
    t0 = time.perf_counter()
    tree = build_tree(grid.cell_centers(), kern, FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    t_tree = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = flt.hikf_precompute_fmm(model, tree)
    t_pre = time.perf_counter() - t0
    state = flt.hikf_init(model)
    t0 = time.perf_counter()
    for t in range(cfg["T"]):
        state = flt.hikf_update(flt.hikf_predict(state, pre), H, model.r_variance, record.observations[t])
    t_on = time.perf_counter() - t0
    print(f"  {cfg['name']}: depth {tree.depth} orders {getattr(tree, '_orders', {})} tree {t_tree:.2f}s precompute {t_pre:.2f}s online {t_on:.2f}s", flush=True)
    out = {f"tree_{k}": v for k, v in tree_ints(tree).items()}
    out.update({
        "H_indptr": H.indptr.astype(np.int64), "H_indices": H.indices.astype(np.int64),
        "H_data": H.data, "obs": record.observations,
        "final_mean": state.mean, "final_variance": state.variance,
        "C_Q_fro": np.float64(np.linalg.norm(pre.C_Q)),
        "cross_cov_fro": np.float64(np.linalg.norm(state.cross_cov)),
        "HC_Q": pre.HC_Q, "final_HC": state.HC,
    })
    if full:
        out["C_Q"] = pre.C_Q
        out["final_cross_cov"] = state.cross_cov
    else:
        cols = np.arange(0, H.shape[0], max(1, H.shape[0] // 4))
        out["cols"] = cols
        out["C_Q_cols"] = pre.C_Q[:, cols]
        out["final_cross_cov_cols"] = state.cross_cov[:, cols]
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


CFG4_PROXY = dict(name="cfg4_proxy", N=512, ns=32, nr=32, family="exponential", L=0.25, R=1e-3, T=3, order=6, leaf=64,
                  seed=0)


def cfg4_proxy() -> dict:
    """SURVEY 8(d) cfg4-proxy (m = 262,144, n = 1024, order 6, depth 6): the
    largest BASELINE-shaped case the reference runs in this container's RAM.
    Full reference precompute + 3 filter steps; stored on a row sample
    (every 64th state row) and 8 of the 1024 columns to keep the fixture small."""
    cfg = CFG4_PROXY
    grid, H, kern, model, record = scenario(cfg)
    t0 = time.perf_counter()
    tree = build_tree(grid.cell_centers(), kern, FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    t_tree = time.perf_counter() - t0
    out = {f"tree_{k}": v for k, v in tree_ints(tree).items()}
    t0 = time.perf_counter()
    pre = flt.hikf_precompute_fmm(model, tree)
    t_pre = time.perf_counter() - t0
    state = flt.hikf_init(model)
    t0 = time.perf_counter()
    for t in range(cfg["T"]):
        state = flt.hikf_update(flt.hikf_predict(state, pre), H, model.r_variance, record.observations[t])
    t_on = time.perf_counter() - t0
    rows = np.arange(0, grid.m, 64)
    cols = np.arange(0, H.shape[0], H.shape[0] // 8)
    out.update({
        "H_nnz": np.int64(H.nnz),
        "H_pattern_sha": np.bytes_(sha(H.indptr.astype(np.int64), H.indices.astype(np.int64))),
        "H_data_sha": np.bytes_(sha(H.data)),
        "obs": record.observations[:cfg["T"]], "rows": rows, "cols": cols,
        "C_Q_sample": pre.C_Q[np.ix_(rows, cols)], "C_Q_fro": np.float64(np.linalg.norm(pre.C_Q)),
        "C_Q_colsum": pre.C_Q.sum(axis=0),
        "HC_Q_block": pre.HC_Q[:64, :64], "HC_Q_fro": np.float64(np.linalg.norm(pre.HC_Q)),
        "final_mean": state.mean[rows], "final_mean_fro": np.float64(np.linalg.norm(state.mean)),
        "final_variance": state.variance[rows],
        "final_cross_cov_sample": state.cross_cov[np.ix_(rows, cols)],
        "final_cross_cov_fro": np.float64(np.linalg.norm(state.cross_cov)),
        "final_HC_block": state.HC[:64, :64], "final_HC_fro": np.float64(np.linalg.norm(state.HC)),
        "ref_seconds": np.array([t_tree, t_pre, t_on]),
    })
    print(f"  cfg4_proxy: depth {tree.depth} orders {tree._orders} tree {t_tree:.1f}s precompute {t_pre:.1f}s "
          f"online {t_on:.1f}s ({cfg['T']} steps)", flush=True)
    return out


def main(big: bool):
    if "--proxy" in sys.argv:  # only the cfg4-proxy fixture (about 5 minutes, ~16 GB RSS)
        np.savez_compressed(os.path.join(HERE, "cfg4_proxy.npz"), **cfg4_proxy())
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
    if big:
        np.savez_compressed(os.path.join(HERE, "cfg2.npz"), **run_filter(cases.CFG2, full=False))
        # cfg4: tree orders + ray operator pattern only
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
        np.savez_compressed(
            os.path.join(HERE, "cfg4_pins.npz"),
            depth=np.int64(t.depth), root_size=np.float64(t.root_size),
            orders=np.array(sorted(t._orders.items()), dtype=np.int64),
            H_indptr=H.indptr.astype(np.int64), H_nnz=np.int64(H.nnz),
            H_pattern_sha=np.bytes_(sha(H.indptr.astype(np.int64), H.indices.astype(np.int64))),
            H_data_sum=np.float64(H.data.sum()), H_data_sha=np.bytes_(sha(H.data)),
        )
        print(f"cfg4: depth {t.depth} orders {t._orders} nnz(H) {H.nnz}")


if __name__ == "__main__":
    main("--big" in sys.argv)
