"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/hikf_b200.h declares, the host-side validation
mirrors the reference's errors, and the native ray-operator producer is
bit-exact with the reference's CSR (no GPU needed for any of this)."""

import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

from tests.golden import cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "hikf_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|int64_t)\s+(hikf_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    from paper_1404_3816_b200 import _lib
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert lib.hikf_abi_version() == 1


def test_no_device_is_a_loud_error():
    import torch
    from paper_1404_3816_b200 import PointSet, KernelSpec, build_tree
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        build_tree(PointSet(np.random.default_rng(0).random((10, 2))), KernelSpec("gaussian"))


def test_host_validation_mirrors_reference():
    from paper_1404_3816_b200 import FmmConfig, KernelSpec, PointSet, Grid2D
    for bad in (dict(n_cheb=1), dict(n_cheb=13), dict(max_leaf_points=0)):
        with pytest.raises(ValueError):
            FmmConfig(**bad)
    with pytest.raises(ValueError):
        KernelSpec("matern")
    with pytest.raises(ValueError):
        KernelSpec("logarithm")
    with pytest.raises(ValueError):
        KernelSpec("gaussian", length_scale=0.0)
    with pytest.raises(ValueError):
        KernelSpec("exponential", power=2.5)
    with pytest.raises(ValueError):
        PointSet(np.zeros((3, 3)))
    with pytest.raises(ValueError):
        PointSet(np.array([[0.0, np.nan]]))
    with pytest.raises(ValueError):
        Grid2D(0, 3)


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("cfg,fixture", [(cases.SMALL, "small_rays.npz"), (cases.CFG1, "cfg1.npz"),
                                         (cases.CFG2, "cfg2.npz"), (cases.CFG4, "cfg4_pins.npz")])
def test_native_ray_operator_bit_exact(cfg, fixture):
    from paper_1404_3816_b200 import Grid2D, tomography
    g = dict(np.load(os.path.join(G, fixture)))
    N = cfg["N"]
    grid = Grid2D(nx=N, ny=N, dx=1.0 / N, dy=1.0 / N)
    H = tomography.build_ray_operator(grid, tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
    if "H_indices" in g:
        assert np.array_equal(H.indptr.astype(np.int64), g["H_indptr"])
        assert np.array_equal(H.indices.astype(np.int64), g["H_indices"])
        assert np.array_equal(H.data, g["H_data"])
    else:
        assert H.nnz == int(g["H_nnz"])
        assert _sha(H.indptr.astype(np.int64), H.indices.astype(np.int64)) == g["H_pattern_sha"].item().decode()
        assert _sha(H.data) == g["H_data_sha"].item().decode()


def test_ray_operator_edge_cases():
    from paper_1404_3816_b200 import Grid2D, tomography
    grid = Grid2D(4, 3)
    # horizontal ray on a gridline goes to the lower cell row; row sums = length
    acq = tomography.Acquisition(np.array([[0.0, 1.0]]), np.array([[4.0, 1.0]]))
    H = tomography.build_ray_operator(grid, acq)
    assert H.nnz == 4 and np.allclose(H.sum(axis=1), 4.0)
    assert set(H.indices) == {0, 1, 2, 3}
    # diagonal through one cell corner to corner
    acq = tomography.Acquisition(np.array([[0.0, 0.0]]), np.array([[1.0, 1.0]]))
    H = tomography.build_ray_operator(grid, acq)
    assert H.nnz == 1 and abs(H.data[0] - np.sqrt(2.0)) < 1e-15
    with pytest.raises(ValueError):
        tomography.build_ray_operator(grid, tomography.Acquisition(np.array([[0.0, 0.0]]), np.array([[0.0, 0.0]])))
    with pytest.raises(ValueError):
        tomography.build_ray_operator(grid, tomography.Acquisition(np.array([[-1.0, 0.0]]), np.array([[1.0, 1.0]])))
