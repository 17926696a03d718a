"""HiKF cross-covariance filter on the B200: drop-in for the HiKF part of the
reference hikf.filters (filters.py:82-157).

State and precompute objects keep their arrays as CUDA torch tensors
(``*_t`` attributes) and expose the reference's numpy fields (``mean``,
``cross_cov``, ``variance``, ``HC``; ``C_Q``, ``HC_Q``, ``diag_Q``) as lazily
copied host views, because callers such as experiment.run_hikf do
``run.means[t] = state.mean`` (experiment.py:237).

``hikf_predict`` is lazy: it returns a state that remembers "prior + pre";
``hikf_update`` on such a state runs the fused predict+update of
libhikf_b200.so, and reading a field of it materialises the predict.
"""

from __future__ import annotations

import os
import weakref

import numpy as np
import scipy.sparse
import torch

from . import _lib
from ._lib import NumericalConsistencyError  # noqa: F401  (re-export, filters.py:27-28)
from .kernels import value_at_zero  # noqa: F401

__all__ = [
    "DeviceCSR", "HikfPrecompute", "HikfState", "NumericalConsistencyError", "hikf_precompute_dense",
    "KfState", "dense_gram", "kf_init", "kf_predict", "kf_update",
    "hikf_precompute_fmm", "hikf_init", "hikf_predict", "hikf_update", "FactoredHikfState",
]


def _dev():
    return _lib.require_cuda()


def _to_dev(x, shape=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=_dev(), dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(_dev())
    t = t.contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {shape}, got {tuple(t.shape)}")
    return t


class DeviceCSR:
    """Device copy of a CSR ray operator (int32 indptr/indices, float64 data).

    Cached per host matrix object so the per-step update does not re-upload H.
    """

    _cache: dict = {}

    def __init__(self, H):
        Hc = H.tocsr() if scipy.sparse.issparse(H) else scipy.sparse.csr_matrix(np.asarray(H, dtype=float))
        Hc = Hc.copy()
        Hc.sum_duplicates()
        Hc.sort_indices()
        self.shape = Hc.shape
        self.nnz = Hc.nnz
        dev = _dev()
        self.indptr = torch.from_numpy(Hc.indptr.astype(np.int32)).to(dev)
        self.indices = torch.from_numpy(Hc.indices.astype(np.int32)).to(dev)
        self.data = torch.from_numpy(Hc.data.astype(np.float64)).to(dev)

    @classmethod
    def from_device(cls, indptr, indices, data, shape) -> "DeviceCSR":
        """Wrap device CSR arrays that are already canonical (sorted, no duplicates)."""
        self = cls.__new__(cls)
        self.shape = tuple(int(s) for s in shape)
        self.nnz = int(indices.numel())
        self.indptr, self.indices, self.data = indptr, indices, data
        return self

    def to_scipy(self) -> scipy.sparse.csr_matrix:
        return scipy.sparse.csr_matrix((self.data.cpu().numpy(), self.indices.cpu().numpy(),
                                        self.indptr.cpu().numpy()), shape=self.shape)

    def transposed(self) -> "DeviceCSR":
        """H^T as a device CSR (cols x rows), built once from the host copy and cached."""
        if getattr(self, "_T", None) is None:
            HT = self.to_scipy().T.tocsr()
            HT.sort_indices()
            self._T = DeviceCSR(HT)
        return self._T

    @staticmethod
    def _fingerprint(H):
        """Cheap identity of the host operator's contents: shape, nnz, the buffer
        addresses and a strided sample of 16 values and indices (~2 us; the update
        calls this every step), so a reallocated operator or an in-place edit such as
        H.data *= s is not served from a stale device copy."""
        if scipy.sparse.issparse(H) and H.format == "csr":
            d, ix = H.data, H.indices
            if d.size == 0:
                return (H.shape, 0, H.indptr.ctypes.data)
            step = max(1, d.size // 16)
            return (H.shape, H.nnz, d.ctypes.data, ix.ctypes.data, H.indptr.ctypes.data,
                    d[::step].tobytes(), ix[::step].tobytes())
        return None

    @classmethod
    def of(cls, H) -> "DeviceCSR":
        if isinstance(H, DeviceCSR):
            return H
        key = id(H)
        fp = cls._fingerprint(H)
        hit = cls._cache.get(key)
        if hit is not None:
            ref, hfp, dcsr = hit
            if ref() is H and fp is not None and hfp == fp:
                return dcsr
            cls._cache.pop(key, None)
        dcsr = cls(H)
        if fp is None:  # dense or non-CSR input: converted per call, not cached
            return dcsr
        try:
            ref = weakref.ref(H)
        except TypeError:  # not weak-referenceable: not cached
            return dcsr
        cls._cache[key] = (ref, fp, dcsr)
        # drop the device copy (and its cached transpose) when the host operator dies
        weakref.finalize(H, cls._cache.pop, key, None)
        return dcsr


class HikfPrecompute:
    """C_Q = Q H^T (m, n), HC_Q = sym(H C_Q) (n, n), diag_Q (m,) -- filters.py:82-88."""

    def __init__(self, C_Q, HC_Q, diag_Q):
        self.C_Q_t = _to_dev(C_Q)
        self.HC_Q_t = _to_dev(HC_Q)
        self.diag_Q_t = _to_dev(diag_Q)
        self._host = {}

    def _np(self, name):
        if name not in self._host:
            self._host[name] = getattr(self, name + "_t").cpu().numpy()
        return self._host[name]

    C_Q = property(lambda self: self._np("C_Q"))
    HC_Q = property(lambda self: self._np("HC_Q"))
    diag_Q = property(lambda self: self._np("diag_Q"))


class HikfState:
    """(mean, C = P H^T, diag P, HC = H P H^T) -- filters.py:91-96."""

    def __init__(self, mean, cross_cov, variance, HC, *, _prior=None, _pre=None):
        self._prior = _prior
        self._pre = _pre
        self._host = {}
        if _prior is None:
            self.mean_t = _to_dev(mean)
            m = self.mean_t.shape[0]
            self.cross_cov_t = _to_dev(cross_cov)
            if self.cross_cov_t.ndim != 2 or self.cross_cov_t.shape[0] != m:
                raise ValueError("cross_cov must have shape (m, n)")
            self.variance_t = _to_dev(variance, (m,))
            n = self.cross_cov_t.shape[1]
            self.HC_t = _to_dev(HC, (n, n))
        else:
            self.mean_t = _prior.mean_t  # the predict leaves the mean unchanged
            self.cross_cov_t = self.variance_t = self.HC_t = None

    @classmethod
    def _wrap(cls, mean_t, C_t, var_t, HC_t):
        """A state over device tensors the library just wrote (no copies or checks)."""
        self = cls.__new__(cls)
        self._prior = self._pre = None
        self._host = {}
        self.mean_t, self.cross_cov_t, self.variance_t, self.HC_t = mean_t, C_t, var_t, HC_t
        return self

    @property
    def pending(self) -> bool:
        return self._prior is not None and self.cross_cov_t is None

    def _materialize(self):
        """Run the (non-fused) predict kernel for a lazily predicted state."""
        if not self.pending:
            return
        p, pre = self._prior, self._pre
        m, n = p.cross_cov_t.shape
        C = torch.empty_like(p.cross_cov_t)
        v = torch.empty_like(p.variance_t)
        HC = torch.empty_like(p.HC_t)
        _lib.check(_lib.load().hikf_predict(m, n, p.cross_cov_t.data_ptr(), p.variance_t.data_ptr(),
                                            p.HC_t.data_ptr(), pre.C_Q_t.data_ptr(), pre.diag_Q_t.data_ptr(),
                                            pre.HC_Q_t.data_ptr(), C.data_ptr(), v.data_ptr(), HC.data_ptr(),
                                            _lib.stream_ptr()))
        self.cross_cov_t, self.variance_t, self.HC_t = C, v, HC

    def _np(self, name):
        resolve_pending()  # host data of a deferred step: its status is checked first (may raise)
        if name not in self._host:
            if name != "mean":
                self._materialize()
            self._host[name] = getattr(self, name + "_t").cpu().numpy()
        return self._host[name]

    mean = property(lambda self: self._np("mean"))
    cross_cov = property(lambda self: self._np("cross_cov"))
    variance = property(lambda self: self._np("variance"))
    HC = property(lambda self: self._np("HC"))

    @property
    def shape(self):
        src = self._prior if self.pending else self
        return tuple(src.cross_cov_t.shape)


class FactoredHikfState(HikfState):
    """A HikfState whose cross covariance is kept factored, C = C_Q N (N n x n).

    Every cross covariance of a filter started from C_0 = alpha H^T with alpha
    = 0 lies in the column space of C_Q (C' = C + C_Q, C_new = r C' S^-1), so
    the state carries N instead of the m x n C; mean, variance and HC are
    explicit and computed every step exactly as in filters.py:138-157 (same
    consistency check).  ``cross_cov`` / ``cross_cov_t`` materialise C_Q N with
    one device GEMM on first access.  Opt-in: ``hikf_init(model,
    representation="factored")``; see update.cu ("factored representation")
    and DESIGN.md section 5.  With C_0 = alpha H^T (alpha != 0) the state also
    carries A: C = alpha H^T A + C_Q N."""

    def __init__(self, mean, N, variance, HC, pre, *, A=None, alpha0=0.0, Hd=None, _prior=None, _pre=None):
        self._prior = _prior
        self._pre = _pre
        self._host = {}
        self._C = None
        if _prior is None:
            self.mean_t, self.N_t, self.variance_t, self.HC_t = mean, N, variance, HC
            self._cq_pre = pre
            # C_0 = alpha0 H^T (filters.py:118-126): C = alpha0 H^T A + C_Q N
            self.A_t, self.alpha0, self._Hd = A, float(alpha0), Hd
        else:
            self.mean_t = _prior.mean_t
            self.N_t = self.variance_t = self.HC_t = None
            self._cq_pre = _pre
            self.A_t, self.alpha0, self._Hd = _prior.A_t, _prior.alpha0, _prior._Hd

    @property
    def pending(self) -> bool:
        return self._prior is not None and self.N_t is None

    def _materialize(self):
        """Predicted state read before its update: N + I, var + diag_Q, HC + HC_Q."""
        if not self.pending:
            return
        p, pre = self._prior, self._pre
        n = p.N_t.shape[0]
        self.N_t = p.N_t + torch.eye(n, dtype=torch.float64, device=p.N_t.device)
        self.variance_t = p.variance_t + pre.diag_Q_t
        self.HC_t = p.HC_t + pre.HC_Q_t

    @property
    def cross_cov_t(self) -> torch.Tensor:
        self._materialize()
        if self._C is None:
            m, n = self.mean_t.shape[0], self.N_t.shape[0]
            if self._cq_pre is None:  # no C_Q term yet
                C = torch.zeros((m, n), dtype=torch.float64, device=self.mean_t.device)
            else:
                C = torch.empty((m, n), dtype=torch.float64, device=self.mean_t.device)
                _lib.check(_lib.load().hikf_dgemm(m, n, n, self._cq_pre.C_Q_t.data_ptr(), n, self.N_t.data_ptr(), n,
                                                  C.data_ptr(), n, 1.0, 0.0, 0, -1, _lib.stream_ptr()))
            if self.A_t is not None and self.alpha0 != 0.0:  # + alpha0 H^T A
                HT = self._Hd.transposed()
                _lib.check(_lib.load().hikf_csr_spmm_add(m, n, HT.indptr.data_ptr(), HT.indices.data_ptr(),
                                                         HT.data.data_ptr(), self.A_t.data_ptr(), self.alpha0,
                                                         C.data_ptr(), _lib.stream_ptr()))
            self._C = C
        return self._C

    @property
    def shape(self):
        src = self._prior if self.pending else self
        return (int(src.mean_t.shape[0]), int(src.N_t.shape[0]))


def _model_H(model):
    return model.H


def hikf_precompute_fmm(model, tree) -> HikfPrecompute:
    """Form Q H^T with one device FMM product over H^T (filters.py:99-105);
    ``tree`` may also be a 3D space3d.FmmTree3D (octree, cfg3 / cfg5)."""
    H = DeviceCSR.of(_model_H(model))
    m, n = tree.m, H.shape[0]
    if H.shape[1] != m:
        raise ValueError("operator columns do not match state length")
    dev = _dev()
    C_Q = torch.empty((m, n), dtype=torch.float64, device=dev)
    HC_Q = torch.empty((n, n), dtype=torch.float64, device=dev)
    diag_Q = torch.empty((m,), dtype=torch.float64, device=dev)
    entry = _lib.load().hikf_precompute3 if getattr(tree, "is_3d", False) else _lib.load().hikf_precompute
    _lib.check(entry(tree._handle, n, H.indptr.data_ptr(), H.indices.data_ptr(),
                     H.data.data_ptr(), C_Q.data_ptr(), HC_Q.data_ptr(), diag_Q.data_ptr(),
                     _lib.stream_ptr()))
    return HikfPrecompute(C_Q, HC_Q, diag_Q)


def hikf_precompute_dense(model) -> HikfPrecompute:
    """Exact dense-algebra path (filters.py:108-115): C_Q = Q H^T with the dense
    Gram Q (kernels.py:97-117), evaluated on the device as a direct sum over the
    nonzeros of H^T (Q is never stored)."""
    import ctypes

    from .fmm import _coords_of
    from .kernels import to_c
    H = DeviceCSR.of(_model_H(model))
    xy = _coords_of(model.grid.cell_centers())
    m, n = xy.shape[0], H.shape[0]
    if H.shape[1] != m:
        raise ValueError("operator columns do not match state length")
    dev = _dev()
    C_Q = torch.empty((m, n), dtype=torch.float64, device=dev)
    HC_Q = torch.empty((n, n), dtype=torch.float64, device=dev)
    diag_Q = torch.empty((m,), dtype=torch.float64, device=dev)
    kc = to_c(model.q_kernel)
    _lib.check(_lib.load().hikf_precompute_dense(xy.ctypes.data, m, ctypes.byref(kc), n, H.indptr.data_ptr(),
                                                 H.indices.data_ptr(), H.data.data_ptr(), C_Q.data_ptr(),
                                                 HC_Q.data_ptr(), diag_Q.data_ptr(), _lib.stream_ptr()))
    return HikfPrecompute(C_Q, HC_Q, diag_Q)


def hikf_init(model, representation: str = "explicit") -> HikfState:
    """mean = mu_0, C = alpha H^T, var = alpha, HC = alpha H H^T (filters.py:118-126).

    ``representation="factored"`` returns a FactoredHikfState (C kept as alpha H^T A + C_Q N)."""
    H = DeviceCSR.of(_model_H(model))
    m, n = int(model.m), H.shape[0]
    dev = _dev()
    mean = _to_dev(model.initial_mean, (m,)).clone()
    if representation == "factored":
        z = dict(dtype=torch.float64, device=dev)
        alpha = float(model.alpha)
        if alpha == 0.0:
            return FactoredHikfState(mean, torch.zeros((n, n), **z), torch.zeros((m,), **z), torch.zeros((n, n), **z),
                                     None)
        # C_0 = alpha H^T = alpha H^T A with A = I, var = alpha, HC = alpha H H^T
        Hs = H.to_scipy()
        HHt = torch.from_numpy(np.ascontiguousarray((Hs @ Hs.T).toarray())).to(dev)
        return FactoredHikfState(mean, torch.zeros((n, n), **z), torch.full((m,), alpha, **z), alpha * HHt, None,
                                 A=torch.eye(n, **z), alpha0=alpha, Hd=H)
    if representation != "explicit":
        raise ValueError(f"unknown representation {representation!r}")
    C = torch.empty((m, n), dtype=torch.float64, device=dev)
    var = torch.empty((m,), dtype=torch.float64, device=dev)
    HC = torch.empty((n, n), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().hikf_init_state(m, n, H.indptr.data_ptr(), H.indices.data_ptr(), H.data.data_ptr(),
                                           float(model.alpha), C.data_ptr(), var.data_ptr(), HC.data_ptr(),
                                           _lib.stream_ptr()))
    return HikfState(mean, C, var, HC)


def hikf_predict(state: HikfState, pre: HikfPrecompute) -> HikfState:
    """C += C_Q, var += diag_Q, HC += HC_Q (filters.py:129-135); evaluated lazily."""
    state._materialize()
    if isinstance(state, FactoredHikfState):
        if tuple(pre.C_Q_t.shape) != state.shape:
            raise ValueError("precompute shape does not match the state")
        # C = C_Q N is expressed against the C_Q this state was built with; another
        # precompute's C_Q would silently change C (C_Q2 (N + I) instead of C_Q1 N + C_Q2)
        cq = state._cq_pre
        if cq is not None and cq is not pre and cq.C_Q_t.data_ptr() != pre.C_Q_t.data_ptr():
            raise ValueError("a factored state can only be predicted with the precompute its C_Q factor refers to")
        return FactoredHikfState(None, None, None, None, None, _prior=state, _pre=pre)
    if tuple(pre.C_Q_t.shape) != tuple(state.cross_cov_t.shape):
        raise ValueError("precompute shape does not match the state")
    return HikfState(None, None, None, None, _prior=state, _pre=pre)


_WS: dict = {}


def _workspace(m: int, n: int) -> torch.Tensor:
    dev = _dev()
    key = (m, n, dev.index)
    ws = _WS.get(key)
    if ws is None:
        nbytes = int(_lib.load().hikf_update_workspace_bytes(m, n))
        _WS.clear()  # one live workspace (the update is single-writer)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        _WS[key] = ws
    return ws


# Deferred status of the explicit update (hikf_update_chained bit 2): a step's
# Cholesky pivot and negative-variance check land in pinned host memory on the
# stream instead of a per-call synchronisation, so the host enqueues step t + 1
# while the GPU runs step t.  Each update resolves every earlier step (one step in
# flight); reading any state's host data resolves all of them.  A failed step
# raises the reference's exception (filters.py:149-153, linalg.py:30-33) from the
# next update call or from the first data access -- before any data computed
# from it is exposed.  HIKF_SYNC_STATUS=1 restores the per-call check.
_PENDING: list = []
_DEFERRED = os.environ.get("HIKF_SYNC_STATUS", "0") != "1"


def resolve_pending(keep_last: bool = False):
    """Check the deferred statuses of finished steps (all, or all but the newest)."""
    while len(_PENDING) > (1 if keep_last else 0):
        status, event = _PENDING.pop(0)
        event.synchronize()
        pivot, negvar, min_var = int(status[0]), bool(status[1]), float(status[2])
        if pivot:
            _PENDING.clear()
            raise _lib.DecompositionError(
                f"Cholesky factorization failed: {pivot}-th leading minor of the array is not positive definite")
        if negvar:
            _PENDING.clear()
            raise NumericalConsistencyError(f"posterior variance went negative beyond tolerance (min {min_var:.3e})")


def hikf_update(state: HikfState, H, r_variance: float, z) -> HikfState:
    """Kalman update of (mean, C, var, HC) against z (filters.py:138-157)."""
    Hd = DeviceCSR.of(H)
    m = state.mean_t.shape[0]
    zt = z if isinstance(z, torch.Tensor) else np.asarray(z, dtype=float)
    if Hd.shape[0] != zt.shape[0]:
        raise ValueError("observation length does not match operator rows")
    if Hd.shape[1] != m:
        raise ValueError("operator columns do not match state length")
    n = Hd.shape[0]
    if n == 0:
        return state
    zt = _to_dev(zt, (n,))
    if isinstance(state, FactoredHikfState):
        return _update_factored(state, Hd, float(r_variance), zt)
    fused = state.pending
    src = state._prior if fused else state
    pre = state._pre if fused else None
    if tuple(src.cross_cov_t.shape) != (m, n):
        raise ValueError("cross covariance shape does not match (m, n)")
    dev = _dev()
    mean = torch.empty((m,), dtype=torch.float64, device=dev)
    C = torch.empty((m, n), dtype=torch.float64, device=dev)
    var = torch.empty((m,), dtype=torch.float64, device=dev)
    HC = torch.empty((n, n), dtype=torch.float64, device=dev)
    ws = _workspace(m, n)
    # chained predict (hikf_update_chained): every fused update also produces the
    # next step's C' = C_new + C_Q; it is consumed only when this prior is exactly
    # the state the previous update returned (states are immutable) with the same
    # precompute, so a stale C' can never be used
    chain = 1 if fused else 0
    if fused and _CHAIN and _CHAIN["state"]() is src and _CHAIN["pre"]() is pre:
        chain |= 2
    _CHAIN.clear()
    # the host copy of the posterior mean (what run_hikf reads every step) is
    # filled inside the call into pinned memory owned by the new state
    mean_host = torch.empty((m,), dtype=torch.float64, pin_memory=True)
    status = None
    if _DEFERRED:
        chain |= 4
        status = torch.empty((4,), dtype=torch.float64, pin_memory=True)
    _lib.check(_lib.load().hikf_update_chained(
        m, n, state.mean_t.data_ptr(), src.cross_cov_t.data_ptr(), src.variance_t.data_ptr(), src.HC_t.data_ptr(),
        _lib.ptr(pre.C_Q_t) if fused else None, _lib.ptr(pre.diag_Q_t) if fused else None,
        _lib.ptr(pre.HC_Q_t) if fused else None,
        Hd.indptr.data_ptr(), Hd.indices.data_ptr(), Hd.data.data_ptr(), float(r_variance), zt.data_ptr(),
        mean.data_ptr(), C.data_ptr(), var.data_ptr(), HC.data_ptr(), ws.data_ptr(), ws.numel(),
        _lib.ptr(status) if status is not None else None, chain, mean_host.data_ptr(), _lib.stream_ptr()))
    out = HikfState._wrap(mean, C, var, HC)
    out._pinned = mean_host
    out._host["mean"] = mean_host.numpy()
    if status is not None:
        ev = torch.cuda.Event()
        ev.record()
        _PENDING.append((status.numpy(), ev))
        resolve_pending(keep_last=True)
    if fused:
        _CHAIN.update(state=weakref.ref(out), pre=weakref.ref(pre))
    return out


_CHAIN: dict = {}


def _update_factored(state: FactoredHikfState, Hd: DeviceCSR, r: float, zt: torch.Tensor) -> FactoredHikfState:
    """hikf_update on a factored state (libhikf_b200 hikf_update_factored)."""
    fused = state.pending
    src = state._prior if fused else state
    pre = state._pre if fused else src._cq_pre
    m, n = state.shape
    if src.N_t.shape != (n, n) or src.mean_t.shape != (m,):
        raise ValueError("factored state shape does not match (m, n)")
    if Hd.shape[0] != n:  # the explicit path's check (filters.py:31-37 via the cross-covariance shape)
        raise ValueError("observation operator rows do not match the state")
    if pre is None:
        raise ValueError("a factored state needs hikf_predict (C_Q) before its first update")
    dev = _dev()
    mean = torch.empty((m,), dtype=torch.float64, device=dev)
    N = torch.empty((n, n), dtype=torch.float64, device=dev)
    var = torch.empty((m,), dtype=torch.float64, device=dev)
    HC = torch.empty((n, n), dtype=torch.float64, device=dev)
    with_a = src.A_t is not None and src.alpha0 != 0.0
    A_out = torch.empty((n, n), dtype=torch.float64, device=dev) if with_a else None
    HT = src._Hd.transposed() if with_a else None
    lib = _lib.load()
    key = (m, n, dev.index, "factored")
    ws = _WS.get(key)
    if ws is None:
        _WS.clear()
        ws = torch.empty(int(lib.hikf_update_factored_workspace_bytes(m, n)), dtype=torch.uint8, device=dev)
        _WS[key] = ws
    _CHAIN.clear()
    mean_host = torch.empty((m,), dtype=torch.float64, pin_memory=True)
    _lib.check(lib.hikf_update_factored(
        m, n, src.mean_t.data_ptr(), src.N_t.data_ptr(), src.variance_t.data_ptr(), src.HC_t.data_ptr(),
        pre.C_Q_t.data_ptr(), _lib.ptr(pre.diag_Q_t) if fused else None, _lib.ptr(pre.HC_Q_t) if fused else None,
        1 if fused else 0, Hd.indptr.data_ptr(), Hd.indices.data_ptr(), Hd.data.data_ptr(), r, zt.data_ptr(),
        mean.data_ptr(), N.data_ptr(), var.data_ptr(), HC.data_ptr(), ws.data_ptr(), ws.numel(), None,
        mean_host.data_ptr(), src.alpha0 if with_a else 0.0, _lib.ptr(src.A_t) if with_a else None,
        _lib.ptr(A_out), _lib.ptr(HT.indptr) if with_a else None, _lib.ptr(HT.indices) if with_a else None,
        _lib.ptr(HT.data) if with_a else None, _lib.stream_ptr()))
    out = FactoredHikfState(mean, N, var, HC, pre, A=A_out, alpha0=src.alpha0 if with_a else 0.0,
                            Hd=src._Hd if with_a else None)
    out._pinned = mean_host
    out._host["mean"] = mean_host.numpy()
    return out


# ----------------------------------------------------------------------
# dense Kalman filter (filters.py:45-74) -- the exact-algebra oracle path
# ----------------------------------------------------------------------


class KfState:
    """mean (m,) and the dense covariance (m, m) as CUDA tensors (``*_t``), numpy on access."""

    def __init__(self, mean, cov):
        self.mean_t, self.cov_t = mean, cov

    mean = property(lambda self: self.mean_t.cpu().numpy())
    cov = property(lambda self: self.cov_t.cpu().numpy())


def dense_gram(spec, points) -> torch.Tensor:
    """G[i, j] = K(|x_i - x_j|) on the device (kernels.py:97-117), r = 0 -> value_at_zero."""
    import ctypes

    from .fmm import _coords_of
    from .kernels import to_c
    xy = _coords_of(points)
    m = xy.shape[0]
    G = torch.empty((m, m), dtype=torch.float64, device=_dev())
    kc = to_c(spec)
    _lib.check(_lib.load().hikf_dense_gram(xy.ctypes.data, m, ctypes.byref(kc), G.data_ptr(), _lib.stream_ptr()))
    return G


def kf_init(model) -> KfState:
    """mean = mu_0, cov = alpha I (filters.py:51-53)."""
    m = int(model.m)
    dev = _dev()
    return KfState(_to_dev(model.initial_mean, (m,)).clone(),
                   float(model.alpha) * torch.eye(m, dtype=torch.float64, device=dev))


def kf_predict(state: KfState, Q) -> KfState:
    """cov + Q (filters.py:56-59)."""
    Qt = Q if isinstance(Q, torch.Tensor) else torch.as_tensor(np.asarray(Q, dtype=np.float64))
    Qt = Qt.to(state.cov_t.device)
    if tuple(Qt.shape) != tuple(state.cov_t.shape):
        raise ValueError("Q shape does not match covariance")
    out = torch.empty_like(state.cov_t)
    _lib.check(_lib.load().hikf_kf_predict(out.shape[0], state.cov_t.data_ptr(), Qt.contiguous().data_ptr(),
                                           out.data_ptr(), _lib.stream_ptr()))
    return KfState(state.mean_t, out)


def kf_update(state: KfState, H, r_variance: float, z) -> KfState:
    """Dense Kalman update (filters.py:62-74)."""
    Hd = DeviceCSR.of(H)
    m = state.mean_t.shape[0]
    zt = z if isinstance(z, torch.Tensor) else np.asarray(z, dtype=float)
    if Hd.shape[0] != zt.shape[0] or Hd.shape[1] != m:
        raise ValueError("observation / operator shape mismatch")
    n = Hd.shape[0]
    if n == 0:
        return state
    zt = _to_dev(zt, (n,))
    mean = torch.empty_like(state.mean_t)
    cov = torch.empty_like(state.cov_t)
    lib = _lib.load()
    ws = torch.empty(int(lib.hikf_kf_workspace_bytes(m, n)), dtype=torch.uint8, device=mean.device)
    _lib.check(lib.hikf_kf_update(m, n, state.mean_t.data_ptr(), state.cov_t.data_ptr(), Hd.indptr.data_ptr(),
                                  Hd.indices.data_ptr(), Hd.data.data_ptr(), float(r_variance), zt.data_ptr(),
                                  mean.data_ptr(), cov.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr()))
    return KfState(mean, cov)

