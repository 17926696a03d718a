"""Row-sharded HiKF filter across ranks.

Each rank owns a contiguous block of state rows [r0, r1) -- C = P H^T,
variance, mean and C_Q rows -- while the n x n quantities (HC, HC_Q, S and
its factor) are replicated: every rank computes them from identical inputs
with the same deterministic kernels, so they stay bitwise equal without
communication.  The rows of the update are independent except for

  * the innovation z - H mean, which needs H mean = sum_r H[:, rows_r] mean_r:
    one all-reduce(sum) of an n-vector per step (8 KB at n = 1024), and
  * the negative-variance check of filters.py:149-153, which compares the
    global minimum posterior variance with the global maximum prior
    variance: one all-reduce(max) of two scalars.

The local step is pluggable: the default binds the CUDA kernels
(hikf_csr_spmv + hikf_update_rows of libhikf_b200.so); tests drive the same
orchestration with a host step on the gloo backend (tests/test_sharded.py).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse

from ._lib import NumericalConsistencyError


def row_block(m: int, world: int, rank: int):
    """Contiguous balanced row block [r0, r1) of rank (first m % world ranks get one more)."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def local_columns(H, r0: int, r1: int) -> scipy.sparse.csr_matrix:
    """H[:, r0:r1] as CSR with column indices relative to r0."""
    Hc = H.tocsr() if scipy.sparse.issparse(H) else scipy.sparse.csr_matrix(np.asarray(H, dtype=float))
    return Hc[:, r0:r1].tocsr()


class ShardedHikf:
    """Drive the HiKF predict/update on a row-sharded state.

    Parameters
    ----------
    comm : object with ``allreduce_sum(vec)`` and ``allreduce_max(vec)``
        returning new arrays/tensors (see TorchComm).
    step : local step backend with ``spmv(H_local, mean_local)`` and
        ``update_rows(state, Hmean, r, z) -> (new_state, (min_var, max_prior))``.
    state : the rank's local state (backend-defined container).
    """

    def __init__(self, comm, step, H, m: int, rank: int, world: int):
        self.comm = comm
        self.step = step
        self.rank, self.world = rank, world
        self.r0, self.r1 = row_block(m, world, rank)
        self.H_local = step.prepare_h(local_columns(H, self.r0, self.r1))

    def update(self, state, r_variance: float, z):
        """One predict+update of the local rows; raises like hikf_update (filters.py:149-153)."""
        partial = self.step.spmv(self.H_local, state)
        Hmean = self.comm.allreduce_sum(partial)
        new_state, (min_var, max_prior) = self.step.update_rows(state, Hmean, r_variance, z)
        # global check: min over ranks of the posterior, max over ranks of the prior variance
        mm = self.comm.allreduce_max(np.array([-min_var, max_prior]))
        gmin, gmax = -float(mm[0]), float(mm[1])
        prior_max = max(gmax, 0.0)
        if gmin < -1e-10 * max(prior_max, np.finfo(float).tiny):
            raise NumericalConsistencyError(f"posterior variance went negative beyond tolerance (min {gmin:.3e})")
        return new_state


def precompute_rows(tree, H, r0: int, r1: int, comm=None):
    """This rank's share of hikf_precompute_fmm: the C_Q rows
    [r0, r1) (hikf_precompute_rows: upward pass and M2L replicated, L2P / P2P
    for the owned rows only), diag_Q rows, and HC_Q = sym(sum over ranks of
    H[:, r0:r1] C_Q_rows) -- one n x n all-reduce (8 MB at n = 1024), or the
    local partial alone when comm is None."""
    import torch

    from . import _lib
    from .filters import DeviceCSR, _dev
    Hd = DeviceCSR.of(H)
    n = Hd.shape[0]
    if not 0 <= r0 <= r1 <= tree.m:
        raise ValueError(f"row block [{r0}, {r1}) outside [0, {tree.m}]")
    dev = _dev()
    CQ = torch.empty((r1 - r0, n), dtype=torch.float64, device=dev)
    X = torch.empty((n, n), dtype=torch.float64, device=dev)
    dQ = torch.empty((r1 - r0,), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().hikf_precompute_rows(tree._handle, n, Hd.indptr.data_ptr(), Hd.indices.data_ptr(),
                                                Hd.data.data_ptr(), int(r0), int(r1), CQ.data_ptr(), X.data_ptr(),
                                                dQ.data_ptr(), _lib.stream_ptr()))
    if comm is not None:
        X = comm.allreduce_sum(X)
        X = 0.5 * (X + X.T)
    return CQ, X, dQ


class LocalComm:
    """world = 1 stand-in for TorchComm (identity reductions)."""

    def allreduce_sum(self, x):
        return x

    def allreduce_max(self, x):
        return x


class TorchComm:
    """all-reduce helpers over a torch.distributed process group (NCCL or gloo)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group, self.device = torch, dist, group, device

    def _reduce(self, x, op):
        t = x if isinstance(x, self.torch.Tensor) else self.torch.as_tensor(np.asarray(x, dtype=np.float64))
        if self.device is not None:
            t = t.to(self.device)
        t = t.clone()
        self.dist.all_reduce(t, op=op, group=self.group)
        return t if isinstance(x, self.torch.Tensor) else t.cpu().numpy()

    def allreduce_sum(self, x):
        return self._reduce(x, self.dist.ReduceOp.SUM)

    def allreduce_max(self, x):
        return self._reduce(x, self.dist.ReduceOp.MAX)


class CudaRowStep:
    """Local step on the B200: hikf_csr_spmv for the H mean partial and
    hikf_update_rows (fused predict + update of the local rows)."""

    def __init__(self, pre_rows, n: int):
        """pre_rows: (C_Q rows, HC_Q, diag_Q rows) CUDA tensors of this rank."""
        import torch
        self.torch = torch
        self.CQ, self.HCQ, self.dQ = pre_rows
        self.n = n
        self._ws = None
        self._last = None

    def prepare_h(self, H_local):
        from .filters import DeviceCSR
        return DeviceCSR(H_local)

    def spmv(self, Hd, state):
        from . import _lib
        y = self.torch.empty(self.n, dtype=self.torch.float64, device=state["mean"].device)
        _lib.check(_lib.load().hikf_csr_spmv(self.n, Hd.indptr.data_ptr(), Hd.indices.data_ptr(),
                                             Hd.data.data_ptr(), state["mean"].data_ptr(), y.data_ptr(),
                                             _lib.stream_ptr()))
        return y

    def update_rows(self, state, Hmean, r, z):
        import ctypes
        from . import _lib
        torch = self.torch
        lib = _lib.load()
        m, n = state["C"].shape
        if self._ws is None or self._ws[0] != (m, n):
            nb = int(lib.hikf_update_workspace_bytes(m, n))
            self._ws = ((m, n), torch.empty(nb, dtype=torch.uint8, device=state["C"].device))
        ws = self._ws[1]
        zt = z if isinstance(z, torch.Tensor) else torch.as_tensor(np.asarray(z, dtype=np.float64))
        zt = zt.to(state["C"].device)
        out = {k: torch.empty_like(v) for k, v in state.items()}
        mm = (ctypes.c_double * 2)()
        # chained predict (hikf_update_chained flags): always produce the next C';
        # consume only when `state` is exactly the dict this step returned last time
        chain = 1 | (2 if state is self._last else 0)
        _lib.check(lib.hikf_update_rows(
            m, n, state["mean"].data_ptr(), state["C"].data_ptr(), state["var"].data_ptr(), state["HC"].data_ptr(),
            self.CQ.data_ptr(), self.dQ.data_ptr(), self.HCQ.data_ptr(), Hmean.data_ptr(), float(r), zt.data_ptr(),
            out["mean"].data_ptr(), out["C"].data_ptr(), out["var"].data_ptr(), out["HC"].data_ptr(),
            ws.data_ptr(), ws.numel(), mm, chain, _lib.stream_ptr()))
        self._last = out  # held, so its buffers cannot be recycled under the chained C'

        return out, (mm[0], mm[1])
