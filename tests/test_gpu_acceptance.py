"""The reference's acceptance and hot-path property tests, run against the CUDA
path (tests/test_acceptance.py criteria 1, 2, 5, 8; test_fmm.py
order monotonicity; test_filters.py incremental HC).  The inputs follow the
reference tests' recipes (seeded random clouds and stations); the exact
answers come from direct sums here, not from fixtures.
"""

import time

import numpy as np
import pytest

from oracle import hikf_oracle as O
from tests.golden import cases
from tests.test_gpu_parity import _Model, _gpu_scenario

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1404_3816_b200 as p
    return p


def _dense_product(spec, pts, v, chunk=2000):
    """K v by direct summation on the host (oracle kernel evaluation)."""
    out = np.zeros(len(pts))
    for i in range(0, len(pts), chunk):
        out[i:i + chunk] = O.kernel_cross(spec, pts[i:i + chunk], pts) @ v
    return out


def test_fast_matvec_accuracy_criterion_1(pkg):
    """m = 10,000 uniform points, Gaussian L = 3: relative error <= 1e-8 at order 5
    and <= 1e-10 at order 7 against the direct sum (acceptance criterion 1)."""
    rng = np.random.default_rng(0)
    m = 10_000
    pts = rng.random((m, 2))
    v = rng.standard_normal(m)
    v /= np.linalg.norm(v)
    dense = _dense_product(O.Kern("gaussian", 1.0, 3.0), pts, v)
    spec = pkg.KernelSpec("gaussian", variance=1.0, length_scale=3.0)
    errs = {}
    for n_cheb in (5, 7):
        tree = pkg.build_tree(pkg.PointSet(pts), spec, pkg.FmmConfig(n_cheb=n_cheb))
        errs[n_cheb] = np.linalg.norm(tree.matvec(v) - dense) / np.linalg.norm(dense)
    assert errs[5] <= 1e-8, errs
    assert errs[7] <= 1e-10, errs


def test_higher_order_is_more_accurate(pkg):
    """Orders 3 < 5 < 7 strictly improve the FMM error on the reference's
    1500-point cloud (x10 box), Gaussian L = 1.5 (test_fmm.py:42-51)."""
    cloud = np.random.default_rng(11).random((1500, 2)) * 10.0
    v = np.random.default_rng(13).standard_normal(len(cloud))
    ref = _dense_product(O.Kern("gaussian", 1.0, 1.5), cloud, v)
    spec = pkg.KernelSpec("gaussian", length_scale=1.5)
    errs = []
    for n_cheb in (3, 5, 7):
        tree = pkg.build_tree(pkg.PointSet(cloud), spec, pkg.FmmConfig(n_cheb=n_cheb))
        errs.append(np.linalg.norm(tree.matvec(v) - ref) / np.linalg.norm(ref))
    assert errs[0] > errs[1] > errs[2], errs


def test_near_linear_scaling_criterion_2(pkg):
    """matvec time at m = 40,000 over m = 10,000 stays <= 6 (criterion 2), timed
    with CUDA events after a warm-up."""
    import torch
    rng = np.random.default_rng(0)
    spec = pkg.KernelSpec("gaussian", variance=1.0, length_scale=3.0)
    times = {}
    for m in (10_000, 40_000):
        tree = pkg.build_tree(pkg.PointSet(rng.random((m, 2))), spec, pkg.FmmConfig(n_cheb=5))
        v = torch.as_tensor(rng.standard_normal((m, 1))).cuda()
        tree.matmat(v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            tree.matmat(v)
        e1.record()
        e1.synchronize()
        times[m] = e0.elapsed_time(e1) / 5
    assert times[40_000] / times[10_000] <= 6.0, times


@pytest.mark.parametrize("device", [False, True])
def test_ray_operator_exactness_criterion_8(pkg, device):
    """1000 random rays (40 x 25 stations inside a 59 x 55 grid): row sums equal
    the ray lengths within 1e-9 and every entry is nonnegative (criterion 8),
    for the host and the device ray operator."""
    grid = pkg.Grid2D(nx=59, ny=55)
    rng = np.random.default_rng(8)
    acq = pkg.tomography.Acquisition(rng.uniform([0.0, 0.0], [59.0, 55.0], size=(40, 2)),
                                     rng.uniform([0.0, 0.0], [59.0, 55.0], size=(25, 2)))
    if device:
        H = pkg.tomography.build_ray_operator_device(grid, acq).to_scipy()
    else:
        H = pkg.tomography.build_ray_operator(grid, acq)
    src, rcv = acq.ray_endpoints()
    lengths = np.hypot(*(rcv - src).T)
    row_sums = np.asarray(H.sum(axis=1)).ravel()
    assert H.shape == (1000, grid.m)
    assert np.abs(row_sums - lengths).max() / lengths.min() <= 1e-9
    assert H.data.min() >= 0.0


@pytest.mark.parametrize("representation", ["explicit", "factored"])
def test_variance_monotone_and_incremental_hc(pkg, representation):
    """Every update lowers (never raises) the variance (criterion 5), and the
    incrementally carried HC equals H C within 1e-9 (test_filters.py:118-127),
    step by step on the cfg1 scenario."""
    flt = pkg.filters
    cfg = cases.CFG1
    grid, H = _gpu_scenario(pkg, cfg)
    kern = pkg.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
    model = _Model(grid, H, kern, cfg["R"])
    tree = pkg.build_tree(grid.cell_centers(), kern, pkg.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    pre = flt.hikf_precompute_fmm(model, tree)
    xy = grid.cell_centers().coords
    obs = O.observations(H, O.moving_plume(xy, 10), cfg["R"], [cfg["seed"], 0])
    st = flt.hikf_init(model, representation=representation)
    for t in range(10):
        prior = flt.hikf_predict(st, pre)
        prior_var = prior.variance
        st = flt.hikf_update(prior, H, cfg["R"], obs[t])
        post = st.variance
        assert np.all(post <= prior_var + 1e-12 * prior_var.max()), t
        direct = np.asarray(H @ st.cross_cov)
        assert np.abs(st.HC - direct).max() <= 1e-9 * max(np.abs(direct).max(), 1e-30), t
