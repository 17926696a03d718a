"""Dense exact-algebra precompute (hikf_precompute_dense, filters.py:108-115)
and the device-resident experiment loop (run_hikf, experiment.py:219-242) on
the GPU, against fixtures made by the reference (tests/golden/dense_cases.npz,
cfg1.npz, small_rays.npz)."""

import os

import numpy as np
import pytest

from oracle import hikf_oracle as O
from tests.golden import cases

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
LOG = dict(cases.SMALL, name="small_log", N=16, ns=3, nr=4, family="logarithm", T=6)


def _scenario(cfg, obs, T=None):
    import paper_1404_3816_b200 as P
    from paper_1404_3816_b200 import experiment as E
    N = cfg["N"]
    grid = P.Grid2D(nx=N, ny=N, dx=1.0 / N, dy=1.0 / N)
    H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
    kern = (P.KernelSpec("logarithm", log_amplitude=-0.5) if cfg["family"] == "logarithm"
            else P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"]))
    model = E.StateSpaceModel(grid=grid, H=H, q_kernel=kern, r_variance=cfg["R"], alpha=0.0)
    T = cfg["T"] if T is None else T
    rec = E.SimulatedRecord(truth=np.zeros((T, grid.m)), observations=np.asarray(obs)[:T])
    return E.Scenario(model=model, record=rec,
                      fmm_config=P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))


@pytest.mark.parametrize("name,cfg", [("small", cases.SMALL), ("cfg1", cases.CFG1), ("small_log", LOG)])
def test_dense_precompute_matches_reference(name, cfg):
    from paper_1404_3816_b200 import filters as flt
    g = dict(np.load(os.path.join(G, "dense_cases.npz")))
    scn = _scenario(cfg, np.zeros((cfg["T"], 1)))
    pre = flt.hikf_precompute_dense(scn.model)
    assert O.rel_fro(pre.C_Q, g[f"{name}_C_Q"]) <= 1e-13
    assert O.rel_fro(pre.HC_Q, g[f"{name}_HC_Q"]) <= 1e-13
    np.testing.assert_array_equal(pre.diag_Q, g[f"{name}_diag_Q"])


def test_dense_and_fmm_precompute_agree():
    """test_filters.py:130-136: FMM C_Q against the dense oracle path.  At the
    cfg1 order (4) the FMM truncation error must be the reference's own
    (golden FMM C_Q vs golden dense C_Q); at n_cheb = 7 it must meet the
    reference test's atol = 1e-6 max|C_Q|."""
    import paper_1404_3816_b200 as P
    from paper_1404_3816_b200 import filters as flt
    cfg = cases.CFG1
    scn = _scenario(cfg, np.zeros((1, 1)), T=1)
    dense = flt.hikf_precompute_dense(scn.model)
    tree = P.build_tree(scn.model.grid.cell_centers(), scn.model.q_kernel, scn.fmm_config)
    fast = flt.hikf_precompute_fmm(scn.model, tree)
    ref_err = O.rel_fro(np.load(os.path.join(G, "cfg1.npz"))["C_Q"], np.load(os.path.join(G, "dense_cases.npz"))["cfg1_C_Q"])
    assert abs(O.rel_fro(fast.C_Q, dense.C_Q) - ref_err) <= 1e-9 * ref_err + 1e-13
    tree7 = P.build_tree(scn.model.grid.cell_centers(), scn.model.q_kernel, P.FmmConfig(n_cheb=7))
    fast7 = flt.hikf_precompute_fmm(scn.model, tree7)
    assert np.allclose(fast7.C_Q, dense.C_Q, atol=1e-6 * np.abs(dense.C_Q).max())


@pytest.mark.parametrize("mode,fixture,prefix,cfg", [
    ("fmm", "small_rays.npz", "", cases.SMALL), ("fmm", "cfg1.npz", "", cases.CFG1),
    ("dense", "dense_cases.npz", "small_", cases.SMALL), ("dense", "dense_cases.npz", "cfg1_", cases.CFG1)])
def test_run_hikf_matches_reference(mode, fixture, prefix, cfg):
    from paper_1404_3816_b200 import experiment as E
    g = dict(np.load(os.path.join(G, fixture)))
    scn = _scenario(cfg, g[f"{prefix}obs"])
    run = E.run_hikf(scn, mode)
    assert run.label == "hikf" and run.means.shape == (cfg["T"], scn.model.m)
    assert run.online_seconds > 0 and run.precompute_seconds > 0
    assert run.storage == E.storage_bytes("hikf", scn.model.m, n=scn.model.n)
    assert run.effective_ranks == [None] * cfg["T"]
    assert O.rel_fro(run.means[-1], g[f"{prefix}final_mean"]) <= 1e-9
    assert O.rel_fro(run.final_variance, g[f"{prefix}final_variance"]) <= 1e-9
    if f"{prefix}step_means" in g:
        # every step's posterior mean -- what the reference's metrics_rows / write_report
        # (experiment.py:298-378) consume -- against the reference's own run
        rows = g[f"{prefix}step_rows"]
        worst = max(O.rel_fro(run.means[t][rows], g[f"{prefix}step_means"][t]) for t in range(cfg["T"]))
        assert worst <= 1e-9, worst


def test_dense_kf_matches_oracle_and_hikf():
    """kf_predict / kf_update on the device (filters.py:45-74) against the numpy
    restatement, and the reference's own equivalence test (test_filters.py:100-115):
    HiKF on the dense precompute == the dense KF (mean, variance = diag P, C = P H^T)."""
    import torch

    from paper_1404_3816_b200 import filters as flt
    cfg = cases.SMALL
    g = dict(np.load(os.path.join(G, "small_rays.npz")))
    scn = _scenario(cfg, g["obs"])
    model, H = scn.model, scn.model.H
    xy = model.grid.cell_centers().coords
    Q = flt.dense_gram(model.q_kernel, model.grid.cell_centers())
    Qo = O.dense_gram(O.Kern(cfg["family"], 1.0, cfg["L"]), xy)
    assert O.rel_fro(Q.cpu().numpy(), Qo) <= 1e-15
    ks = flt.kf_init(model)
    mo, Po = np.zeros(model.m), np.zeros((model.m, model.m))
    pre = flt.hikf_precompute_dense(model)
    hs = flt.hikf_init(model)
    for t in range(cfg["T"]):
        ks = flt.kf_update(flt.kf_predict(ks, Q), H, cfg["R"], g["obs"][t])
        mo, Po = O.kf_update(mo, Po + Qo, H, cfg["R"], g["obs"][t])
        hs = flt.hikf_update(flt.hikf_predict(hs, pre), H, cfg["R"], g["obs"][t])
    P = ks.cov_t
    assert O.rel_fro(ks.mean, mo) <= 1e-10
    assert O.rel_fro(P.cpu().numpy(), Po) <= 1e-10
    assert torch.equal(P, P.T)
    assert O.rel_fro(hs.mean, ks.mean) <= 1e-10
    assert O.rel_fro(hs.variance, torch.diagonal(P).cpu().numpy()) <= 1e-10
    Hd = torch.as_tensor(H.toarray(), device="cuda")
    assert O.rel_fro(hs.cross_cov, (P @ Hd.T).cpu().numpy()) <= 1e-10


@pytest.mark.slow
def test_hikf_equals_dense_kf_at_cfg2():
    """HiKF == KF at the cfg2 size (m = 65,536: the dense covariance is 34 GB in
    HBM), both on the exact dense precompute, over 20 steps of the cfg2 record."""
    import torch

    from paper_1404_3816_b200 import filters as flt
    cfg = dict(cases.CFG2, T=20)
    g = dict(np.load(os.path.join(G, "cfg2.npz")))
    scn = _scenario(cfg, g["obs"])
    model, H = scn.model, scn.model.H
    pre = flt.hikf_precompute_dense(model)
    hs = flt.hikf_init(model)
    for t in range(cfg["T"]):
        hs = flt.hikf_update(flt.hikf_predict(hs, pre), H, cfg["R"], g["obs"][t])
    del pre
    Q = flt.dense_gram(model.q_kernel, model.grid.cell_centers())
    ks = flt.kf_init(model)
    for t in range(cfg["T"]):
        ks = flt.kf_update(flt.kf_predict(ks, Q), H, cfg["R"], g["obs"][t])
    del Q
    assert O.rel_fro(hs.mean, ks.mean) <= 1e-8
    assert O.rel_fro(hs.variance, torch.diagonal(ks.cov_t).cpu().numpy()) <= 1e-8
