"""Time the FP64 DMMA GEMM variants of libhikf_b200 at the cfg4 update shapes
(M = 1,048,576, N = K = 1,024) against cuBLAS (torch.matmul float64)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_3816_b200 import _lib  # noqa: E402

M = int(os.environ.get("SWEEP_M", 1 << 20))
N = 1024
KK = int(os.environ.get("SWEEP_K", N))  # inner dimension (default: the update's n)
lib = _lib.load()
torch.manual_seed(0)
A = torch.randn(M, KK, dtype=torch.float64, device="cuda")
B = torch.randn(KK, N, dtype=torch.float64, device="cuda")
C = torch.randn(M, N, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {}
full = 2.0 * M * N * KK
for v in [int(x) for x in os.environ.get("SWEEP_VARIANTS", "30,32,7").split(",")]:
    t_full = timeit(lambda: lib.hikf_dgemm(M, N, KK, A.data_ptr(), KK, B.data_ptr(), N, C.data_ptr(), N, -1.0,
                                           1.0, 0, v, st))
    t_up = timeit(lambda: lib.hikf_dgemm(M, N, KK, A.data_ptr(), KK, B.data_ptr(), N, C.data_ptr(), N, 1.0, 0.0,
                                         1, v, st))
    # correctness of this variant against cuBLAS on a 4096-row slice (full and upper-triangular)
    Cs = torch.zeros(4096, N, dtype=torch.float64, device="cuda")
    lib.hikf_dgemm(4096, N, KK, A.data_ptr(), KK, B.data_ptr(), N, Cs.data_ptr(), N, 1.0, 0.0, 0, v, st)
    ref = torch.matmul(A[:4096], B)
    err_full = float(((Cs - ref).abs().max() / ref.abs().max()).item())
    lib.hikf_dgemm(4096, N, KK, A.data_ptr(), KK, B.data_ptr(), N, Cs.data_ptr(), N, 1.0, 0.0, 1, v, st)
    ref_u = None  # kmode 1 assumes B upper triangular (LiT); skip on a full random B
    err_up = None
    out[f"v{v}"] = {"full_ms": t_full, "full_tflops": full / t_full / 1e9,
                    "upper_ms": t_up, "upper_tflops": 0.5 * full / t_up / 1e9, "err_full": err_full,
                    "err_upper": err_up}
    print(v, out[f"v{v}"], flush=True)
# correctness of the default variant vs cuBLAS on a slice
ref = torch.matmul(A[:4096], B)
Cs = torch.zeros(4096, N, dtype=torch.float64, device="cuda")
lib.hikf_dgemm(4096, N, KK, A.data_ptr(), KK, B.data_ptr(), N, Cs.data_ptr(), N, 1.0, 0.0, 0, -1, st)
torch.cuda.synchronize()
out["max_rel_err_vs_cublas"] = float(((Cs - ref).abs().max() / ref.abs().max()).item())
t_cublas = timeit(lambda: torch.matmul(A, B, out=C))
out["cublas_full_ms"] = t_cublas
out["cublas_tflops"] = full / t_cublas / 1e9
print(json.dumps(out))
