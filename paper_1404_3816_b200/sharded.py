"""Row-sharded HiKF filter across ranks.

Each rank owns a block of state rows -- C = P H^T, variance, mean and C_Q
rows -- while the n x n quantities (HC, HC_Q, S and its factor) are
replicated: every rank computes them from identical inputs with the same
deterministic kernels, so they stay bitwise equal without communication.

Row blocks are leaf-aligned (``leaf_block``): a rank owns a contiguous range
of quadtree leaves in the tree's x-major leaf order, balanced by point count,
and stores its rows in that (sorted) order.  Its Q H^T shard
(``precompute_leaves`` -> hikf_precompute_leaves) then runs P2P and the fused
leaf L2L + L2P for its own leaves only and M2L / L2L only for their
ancestors (a strip of box columns); only the cheap upward pass is
replicated.  ``row_block`` (contiguous original rows) remains for host-side
tests.

The rows of the update are independent except for

  * the innovation z - H mean, which needs H mean = sum_r H[:, rows_r] mean_r:
    one all-reduce(sum) of an n-vector per step (8 KB at n = 1024), and
  * the negative-variance check of filters.py:149-153, which compares the
    global minimum posterior variance with the global maximum prior
    variance: one all-reduce(max) of [-min var, max prior var, pivot].  With
    the CUDA step this is a device tensor reduced on the device (NCCL) and
    checked at the next host touch (the next update, ``check()`` or
    ``gather``), so a step makes no host round trip; an error of step t is
    raised by the next call, before any later state is exposed.

The local step is pluggable: the default binds the CUDA kernels
(hikf_csr_spmv + hikf_update_rows of libhikf_b200.so); tests drive the same
orchestration with a host step on the gloo backend (tests/test_sharded.py)
and the CUDA step with two gloo ranks sharing one GPU
(tests/test_gpu_sharded.py).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse

from ._lib import DecompositionError, NumericalConsistencyError


def row_block(m: int, world: int, rank: int):
    """Contiguous balanced row block [r0, r1) of rank (first m % world ranks get one more)."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def leaf_block(tree, world: int, rank: int):
    """Leaf-aligned block of rank: (leaf0, leaf1, s0, s1) -- leaves [leaf0, leaf1) of
    the tree's x-major leaf order, balanced by point count, whose points are the
    sorted positions [s0, s1) (original rows tree order[s0:s1])."""
    import ctypes

    from . import _lib
    out = (ctypes.c_int64 * 4)()
    _lib.check(_lib.load().hikf_leaf_partition(tree._handle, int(world), int(rank), out))
    return tuple(int(v) for v in out)


def local_columns(H, r0: int, r1: int = None) -> scipy.sparse.csr_matrix:
    """H[:, r0:r1] as CSR with column indices relative to r0; with r0 an index
    array (leaf-aligned rows), H[:, rows] in that order."""
    Hc = H.tocsr() if scipy.sparse.issparse(H) else scipy.sparse.csr_matrix(np.asarray(H, dtype=float))
    if r1 is None:
        return Hc[:, np.asarray(r0)].tocsr()
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

    def __init__(self, comm, step, H, m: int, rank: int, world: int, rows=None):
        """rows: this rank's original row indices in local order (leaf-aligned:
        tree order[s0:s1]); None = the contiguous row_block."""
        self.comm = comm
        self.step = step
        self.rank, self.world = rank, world
        self._pending = None
        if rows is None:
            self.r0, self.r1 = row_block(m, world, rank)
            self.rows = np.arange(self.r0, self.r1)
            self.H_local = step.prepare_h(local_columns(H, self.r0, self.r1))
        else:
            self.rows = np.asarray(rows, dtype=np.int64)
            self.r0, self.r1 = None, None
            self.H_local = step.prepare_h(local_columns(H, self.rows))

    @staticmethod
    def _raise_if_bad(mm):
        """mm = all-reduced max of [-min posterior var, max prior var, pivot] (filters.py:149-153)."""
        gmin, gmax, pivot = -float(mm[0]), float(mm[1]), int(mm[2]) if len(mm) > 2 else 0
        if pivot:
            raise DecompositionError(
                f"Cholesky factorization failed: {pivot}-th leading minor of the array is not positive definite")
        prior_max = max(gmax, 0.0)
        if gmin < -1e-10 * max(prior_max, np.finfo(float).tiny):
            raise NumericalConsistencyError(f"posterior variance went negative beyond tolerance (min {gmin:.3e})")

    def check(self):
        """Resolve the deferred check of the last step (raises on every rank)."""
        if self._pending is not None:
            mm, self._pending = self._pending, None
            self._raise_if_bad(mm.cpu().numpy() if hasattr(mm, "cpu") else mm)

    def update(self, state, r_variance: float, z):
        """One predict+update of the local rows; raises like hikf_update (filters.py:149-153) --
        for a deferred (device) check, at the next host touch."""
        self.check()
        partial = self.step.spmv(self.H_local, state)
        Hmean = self.comm.allreduce_sum(partial)
        new_state, mm = self.step.update_rows(state, Hmean, r_variance, z)
        if hasattr(mm, "is_cuda"):  # device [min var, max prior, pivot]: reduced on the device, checked later
            import torch
            red = torch.stack([-mm[0], mm[1], mm[2]])
            self._pending = self.comm.allreduce_max(red)
            return new_state
        min_var, max_prior = mm
        self._raise_if_bad(self.comm.allreduce_max(np.array([-min_var, max_prior, 0.0])))
        return new_state

    def gather(self, local, m: int):
        """Full-length (m) array in original row order from every rank's local rows
        (all-gather; checks the last step first)."""
        import torch
        self.check()
        loc = local if isinstance(local, torch.Tensor) else torch.as_tensor(np.asarray(local))
        parts = self.comm.allgather((torch.as_tensor(self.rows), loc))
        out = np.empty((m,) + tuple(loc.shape[1:]), dtype=np.float64)
        for rows, vals in parts:
            out[np.asarray(rows)] = vals.cpu().numpy() if hasattr(vals, "cpu") else np.asarray(vals)
        return out


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


def precompute_leaves(tree, H, leaf0: int, leaf1: int, comm=None):
    """This rank's leaf-aligned share of hikf_precompute_fmm (hikf_precompute_leaves):
    the C_Q rows of leaves [leaf0, leaf1) in leaf order, their diag_Q, and HC_Q =
    sym(sum over ranks of H[:, rows] C_Q_rows) (one n x n all-reduce) or the local
    partial alone when comm is None."""
    import torch

    from . import _lib
    from .filters import DeviceCSR, _dev
    Hd = DeviceCSR.of(H)
    n = Hd.shape[0]
    ex = tree.export()
    starts, counts = ex["leaf_starts"], ex["leaf_counts"]
    s0 = int(starts[leaf0]) if leaf0 < len(starts) else tree.m
    s1 = int(starts[leaf1 - 1] + counts[leaf1 - 1]) if leaf1 > leaf0 else s0
    dev = _dev()
    CQ = torch.empty((s1 - s0, n), dtype=torch.float64, device=dev)
    X = torch.empty((n, n), dtype=torch.float64, device=dev)
    dQ = torch.empty((s1 - s0,), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().hikf_precompute_leaves(tree._handle, n, Hd.indptr.data_ptr(), Hd.indices.data_ptr(),
                                                  Hd.data.data_ptr(), int(leaf0), int(leaf1), CQ.data_ptr(),
                                                  X.data_ptr(), dQ.data_ptr(), _lib.stream_ptr()))
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

    def allgather(self, obj):
        return [obj]


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
        if t.is_cuda and self.dist.get_backend(self.group) == "gloo":
            h = t.cpu()  # gloo reduces host buffers (tests sharing one GPU); NCCL stays on the device
            self.dist.all_reduce(h, op=op, group=self.group)
            t = h.to(t.device)
        else:
            self.dist.all_reduce(t, op=op, group=self.group)
        return t if isinstance(x, self.torch.Tensor) else t.cpu().numpy()

    def allgather(self, obj):
        """all_gather_object of (rows, values) pairs (host copies; end-of-run only)."""
        rows, vals = obj
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, (np.asarray(rows), vals.cpu().numpy() if hasattr(vals, "cpu") else vals),
                                    group=self.group)
        return out

    def allreduce_sum(self, x):
        return self._reduce(x, self.dist.ReduceOp.SUM)

    def allreduce_max(self, x):
        return self._reduce(x, self.dist.ReduceOp.MAX)


class CudaRowStep:
    """Local step on the B200: hikf_csr_spmv for the H mean partial and
    hikf_update_rows (fused predict + update of the local rows)."""

    def __init__(self, pre_rows, n: int, deferred: bool = True):
        """pre_rows: (C_Q rows, HC_Q, diag_Q rows) CUDA tensors of this rank; deferred:
        the per-step status stays on the device (hikf_update_rows chain bit 2)."""
        import torch
        self.torch = torch
        self.deferred = deferred
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
        # chained predict (hikf_update_chained flags): always produce the next C';
        # consume only when `state` is exactly the dict this step returned last time.
        # bit 2: deferred status -- [min var, max prior var, pivot] into a device array,
        # no host synchronisation (ShardedHikf reduces and checks it later)
        chain = 1 | (2 if state is self._last else 0)
        if self.deferred:
            chain |= 4
            mm = torch.empty(3, dtype=torch.float64, device=state["C"].device)
            mm_ptr = mm.data_ptr()
        else:
            mm = (ctypes.c_double * 2)()
            mm_ptr = mm
        _lib.check(lib.hikf_update_rows(
            m, n, state["mean"].data_ptr(), state["C"].data_ptr(), state["var"].data_ptr(), state["HC"].data_ptr(),
            self.CQ.data_ptr(), self.dQ.data_ptr(), self.HCQ.data_ptr(), Hmean.data_ptr(), float(r), zt.data_ptr(),
            out["mean"].data_ptr(), out["C"].data_ptr(), out["var"].data_ptr(), out["HC"].data_ptr(),
            ws.data_ptr(), ws.numel(), mm_ptr, chain, _lib.stream_ptr()))
        self._last = out  # held, so its buffers cannot be recycled under the chained C'
        if self.deferred:
            return out, mm
        return out, (mm[0], mm[1])
