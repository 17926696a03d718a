"""SPD solve on the GPU: drop-in for the reference hikf.linalg.spd_solve
(linalg.py:18-37) -- same symmetry check, Cholesky failure mapped to
DecompositionError, ValueError on a non-square or asymmetric A."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import DecompositionError  # noqa: F401  (linalg.py:14-15)


def spd_solve(A, B):
    """Solve A X = B for symmetric positive definite A via Cholesky."""
    host = not isinstance(A, torch.Tensor)
    At = torch.as_tensor(np.asarray(A, dtype=float)) if host else A
    if At.ndim != 2 or At.shape[0] != At.shape[1]:
        raise ValueError("A must be square")
    Bt = torch.as_tensor(np.asarray(B, dtype=float)) if not isinstance(B, torch.Tensor) else B
    vec = Bt.ndim == 1
    if vec:
        Bt = Bt[:, None]
    n, k = At.shape[0], Bt.shape[1]
    if Bt.shape[0] != n:
        raise ValueError("B rows do not match A")
    dev = _lib.require_cuda()
    Ad = At.to(device=dev, dtype=torch.float64).contiguous()
    Bd = Bt.to(device=dev, dtype=torch.float64).contiguous()
    X = torch.empty((n, k), dtype=torch.float64, device=dev)
    lib = _lib.load()
    ws = torch.empty(int(lib.hikf_spd_solve_workspace_bytes(n, k)), dtype=torch.uint8, device=dev)
    info = ctypes.c_int64(0)
    _lib.check(lib.hikf_spd_solve(n, k, Ad.data_ptr(), Bd.data_ptr(), X.data_ptr(), ws.data_ptr(), ws.numel(),
                                  ctypes.byref(info), _lib.stream_ptr()))
    if vec:
        X = X[:, 0]
    return X.cpu().numpy() if host else X
