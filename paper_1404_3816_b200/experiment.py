"""Device-resident HiKF experiment loop.

Mirror of the reference's ``experiment.run_hikf`` (experiment.py:219-242) and
the containers it needs (``StateSpaceModel`` ssm.py:22-52, ``SimulatedRecord``
ssm.py:55-60, ``Scenario`` experiment.py:49-56, ``FilterRun``
experiment.py:59-69, ``storage_bytes`` metrics.py:72-87).  Reference objects
are accepted duck-typed, so a reference ``Scenario`` runs unchanged.

Differences that are not visible in the results:

* the observations are uploaded once; each step's ``z`` is a device row;
* each step's posterior mean is snapshotted into a (T, m) device buffer (a
  device copy) and copied to the host once after the loop;
* the steps are enqueued back to back: a step's status is checked one step
  late (filters.resolve_pending) and all of them before the results are read.

The online clock covers the T predict + update steps; it closes after the
last step has finished on the device, so wall time brackets the device work.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import filters as flt
from .fmm import FmmConfig, build_tree


@dataclass(frozen=True)
class StateSpaceModel:
    """ssm.py:22-52: grid, H (CSR n x m), Q kernel, observation variance, P0 = alpha I."""

    grid: object
    H: object = field(repr=False)
    q_kernel: object
    r_variance: float
    alpha: float = 0.0
    initial_mean: np.ndarray | None = field(default=None, repr=False)

    def __post_init__(self):
        if self.H.shape[1] != self.grid.m:
            raise ValueError("operator column count must equal the grid cell count")
        if not self.r_variance >= 0:
            raise ValueError("r_variance must be >= 0")
        if not self.alpha >= 0:
            raise ValueError("alpha must be >= 0")
        mean = np.zeros(self.grid.m) if self.initial_mean is None else self.initial_mean
        mean = np.asarray(mean, dtype=float)
        if mean.shape != (self.grid.m,):
            raise ValueError("initial_mean must have length m")
        object.__setattr__(self, "initial_mean", mean)

    @property
    def m(self) -> int:
        return self.grid.m

    @property
    def n(self) -> int:
        return self.H.shape[0]


@dataclass(frozen=True)
class SimulatedRecord:
    """ssm.py:55-60: truth (T, m) at t = 1..T and observations (T, n)."""

    truth: np.ndarray = field(repr=False)
    observations: np.ndarray = field(repr=False)


@dataclass
class Scenario:
    """The fields of experiment.py:49-56 that run_hikf reads."""

    model: StateSpaceModel
    record: SimulatedRecord
    fmm_config: FmmConfig = field(default_factory=FmmConfig)


@dataclass
class FilterRun:
    """experiment.py:59-69."""

    label: str
    means: np.ndarray = field(repr=False)
    final_variance: np.ndarray | None = field(default=None, repr=False)
    effective_ranks: list = field(default_factory=list)
    final_spectrum: np.ndarray | None = field(default=None, repr=False)
    precompute_seconds: float = 0.0
    online_seconds: float = 0.0
    storage: dict = field(default_factory=dict)
    failed: str | None = None


def storage_bytes(kind: str, m: int, n: int = 0, ensemble_size: int = 0) -> dict:
    """Dominant-term payload in bytes of double precision (metrics.py:72-87)."""
    if kind == "kf":
        return {"total": 8 * m * m, "online_state": 8 * m * m}
    if kind == "hikf":
        online = 8 * (m * n + m)
        precomputed = 8 * (m * n + m)
        return {"total": online + precomputed, "online_state": online, "precomputed": precomputed}
    if kind == "enkf":
        return {"total": 8 * m * ensemble_size, "online_state": 8 * m * ensemble_size}
    raise ValueError(f"unknown filter kind {kind!r}")


def run_hikf(scn, mode: str) -> FilterRun:
    """experiment.py:219-242: precompute (tree + Q H^T, or the dense oracle path),
    then T predict/update steps with per-step mean snapshots."""
    model = scn.model
    T = scn.record.truth.shape[0]
    m = int(model.m)
    t0 = time.perf_counter()
    if mode == "dense":
        pre = flt.hikf_precompute_dense(model)
    else:
        tree = build_tree(model.grid.cell_centers(), model.q_kernel, scn.fmm_config)
        pre = flt.hikf_precompute_fmm(model, tree)
    torch.cuda.synchronize()
    precompute_seconds = time.perf_counter() - t0
    dev = pre.C_Q_t.device
    obs = torch.as_tensor(np.ascontiguousarray(scn.record.observations, dtype=np.float64)).to(dev)
    means = torch.empty((T, m), dtype=torch.float64, device=dev)
    Hd = flt.DeviceCSR.of(model.H)
    state = flt.hikf_init(model)
    # the steps are enqueued back to back (deferred step status, filters.resolve_pending);
    # the online clock closes after the last step has finished on the device and every
    # step's status has been checked
    t0 = time.perf_counter()
    for t in range(T):
        state = flt.hikf_predict(state, pre)
        state = flt.hikf_update(state, Hd, model.r_variance, obs[t])
        means[t].copy_(state.mean_t)
    flt.resolve_pending()
    torch.cuda.synchronize()
    online = time.perf_counter() - t0
    run = FilterRun(label="hikf", means=means.cpu().numpy())
    run.effective_ranks = [None] * T  # the full spectrum is not reconstructible from (C, variance)
    run.precompute_seconds = precompute_seconds
    run.online_seconds = online
    run.final_variance = state.variance.copy()
    run.storage = storage_bytes("hikf", m, n=int(model.n))
    return run
