"""ctypes binding of libhikf_b200.so (include/hikf_b200.h).

The shared library is the product: every numeric call of this package goes
through it.  There is no CPU fallback -- if the library or a CUDA device is
missing, calls raise immediately.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhikf_b200.so")

HIKF_OK = 0
HIKF_BAD_ARGUMENT = 1
HIKF_NOT_PD = 2
HIKF_NEGATIVE_VARIANCE = 3
HIKF_CUDA_ERROR = 4
HIKF_ASYMMETRIC = 5
HIKF_NO_DEVICE = 6

FAMILY_CODE = {"gaussian": 0, "exponential": 1, "logarithm": 2}


class DecompositionError(RuntimeError):
    """A matrix factorization failed (linalg.py:14-15)."""


class NumericalConsistencyError(RuntimeError):
    """A tracked quantity left its guaranteed range (filters.py:27-28)."""


class HikfKernel(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32),
        ("variance", ctypes.c_double),
        ("length_scale", ctypes.c_double),
        ("power", ctypes.c_double),
        ("log_amplitude", ctypes.c_double),
    ]


class HikfKernel3(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32),
        ("variance", ctypes.c_double),
        ("lx", ctypes.c_double),
        ("ly", ctypes.c_double),
        ("lz", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); every symbol declared in include/hikf_b200.h
SIGNATURES = {
    "hikf_abi_version": (ctypes.c_int, []),
    "hikf_last_error": (ctypes.c_int, [ctypes.c_char_p, _SZ]),
    "hikf_tree_create": (ctypes.c_int, [_P, _I64, ctypes.POINTER(HikfKernel), _I32, _I64, _P, ctypes.POINTER(_P)]),
    "hikf_tree_destroy": (ctypes.c_int, [_P]),
    "hikf_release_cached_memory": (ctypes.c_int, []),
    "hikf_tree_info": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "hikf_tree_export": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "hikf_tree_export_op": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _P]),
    "hikf_tree_m2l_pairs": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P, _P]),
    "hikf_tree_matmat": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _I64, _P]),
    "hikf_tree_matmat_csrT": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _P]),
    "hikf_precompute": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "hikf_init_state": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _D, _P, _P, _P, _P]),
    "hikf_predict": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "hikf_update_workspace_bytes": (_SZ, [_I64, _I64]),
    "hikf_update": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P, _P, _P,
                                   _P, _SZ, _P, _P]),
    "hikf_update_chained": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P, _P,
                                           _P, _P, _SZ, _P, ctypes.c_int32, _P, _P]),
    "hikf_update_factored_workspace_bytes": (_SZ, [_I64, _I64]),
    "hikf_update_factored": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _D, _P, _P,
                                            _P, _P, _P, _P, _SZ, _P, _P, _D, _P, _P, _P, _P, _P, _P]),
    "hikf_csr_spmm_add": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _D, _P, _P]),
    "hikf_update_rows": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _D, _P, _P, _P, _P, _P, _P,
                                        _SZ, _P, ctypes.c_int32, _P]),
    "hikf_csr_spmv": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P]),
    "hikf_spd_solve_workspace_bytes": (_SZ, [_I64, _I64]),
    "hikf_spd_solve": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _SZ, _P, _P]),
    "hikf_ray_operator": (ctypes.c_int, [_I64, _I64, _D, _D, _D, _D, _I64, _P, _P, _P, _P, _P, _P]),
    "hikf_precompute_rows": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I64, _I64, _P, _P, _P, _P]),
    "hikf_leaf_partition": (ctypes.c_int, [_P, _I32, _I32, _P]),
    "hikf_precompute_leaves": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I64, _I64, _P, _P, _P, _P]),
    "hikf_precompute_dense": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "hikf_ray_operator_3d": (ctypes.c_int, [_P, _P, _P, _I64, _P, _P, _P, _P, _P, _P]),
    "hikf_ray_operator_3d_device": (ctypes.c_int, [_P, _P, _P, _I64, _P, _P, _P, _P, _P, _I64, _P, _P]),
    "hikf_tree3_create": (ctypes.c_int, [_P, _I64, _P, ctypes.c_int32, _I64, _P, _P]),
    "hikf_tree3_destroy": (ctypes.c_int, [_P]),
    "hikf_tree3_info": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "hikf_tree3_export": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "hikf_tree3_matmat": (ctypes.c_int, [_P, _P, _I64, _P, _P]),
    "hikf_precompute3": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "hikf_dense_gram": (ctypes.c_int, [_P, _I64, _P, _P, _P]),
    "hikf_kf_predict": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "hikf_kf_workspace_bytes": (_SZ, [_I64, _I64]),
    "hikf_kf_update": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _D, _P, _P, _P, _P, _SZ, _P]),
    "hikf_ray_operator_device": (ctypes.c_int, [_I64, _I64, _D, _D, _D, _D, _I64, _P, _P, _P, _P, _P, _I64, _P, _P]),
    "hikf_dgemm": (ctypes.c_int, [_I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _D, _D, _I32, _I32, _P]),
    "hikf_prof_enable": (ctypes.c_int, [ctypes.c_int]),
    "hikf_prof_reset": (ctypes.c_int, []),
    "hikf_prof_read": (ctypes.c_int, [_I32, _P, _P]),
    "hikf_prof_flops": (ctypes.c_int, [_I32, _P]),
    "hikf_launch_count": (_I64, []),
    "hikf_set_tuning": (ctypes.c_int, [_I32, _I32, _P]),
}

# stage ids of hikf_prof_read (csrc/prof.h)
STAGES = {"predict": 0, "factor": 1, "gemm_y": 2, "finalize": 3, "gemm_c": 4, "p2p": 5, "p2m": 6, "m2m": 7,
          "m2l": 8, "l2p": 9, "densify": 10, "l2l": 11}


def prof_read(stage: str):
    """(total ms, launches) of one stage since the last hikf_prof_reset."""
    ms = ctypes.c_double()
    cnt = ctypes.c_int64()
    load().hikf_prof_read(STAGES[stage], ctypes.byref(ms), ctypes.byref(cnt))
    return ms.value, cnt.value


def prof_flops(stage: str) -> int:
    """Useful flops a stage executed since the last hikf_prof_reset (profiling on)."""
    v = ctypes.c_uint64()
    load().hikf_prof_flops(STAGES[stage], ctypes.byref(v))
    return v.value

_lib = None


def load():
    """Load (once) and return the shared library; raises if it is missing."""
    global _lib
    if _lib is None:
        path = os.environ.get("HIKF_LIB_PATH", LIB_PATH)  # A/B timing of a second in-tree build (tools/)
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the HiKF B200 path has no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load().hikf_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception types."""
    if status == HIKF_OK:
        return
    msg = last_error() or what
    if status in (HIKF_BAD_ARGUMENT, HIKF_ASYMMETRIC):
        raise ValueError(msg)
    if status == HIKF_NOT_PD:
        raise DecompositionError(msg)
    if status == HIKF_NEGATIVE_VARIANCE:
        raise NumericalConsistencyError(msg)
    raise RuntimeError(f"libhikf_b200 failure ({status}): {msg}")


_HAVE_CUDA = False


def require_cuda() -> torch.device:
    """The current CUDA device; raises when there is none (no CPU fallback).  The
    availability probe runs until it first succeeds (it costs ~6 us per call)."""
    global _HAVE_CUDA
    if not _HAVE_CUDA:
        if not torch.cuda.is_available():
            raise RuntimeError("the HiKF B200 path needs a CUDA device; there is no CPU fallback")
        _HAVE_CUDA = True
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
