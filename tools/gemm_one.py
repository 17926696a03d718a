"""Run one libhikf_b200 DGEMM (variant from argv, default 30) twice at M x 1024 x 1024
(M = GEMM_M, default 262,144): the target of an ncu capture (tools/prof_*)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_3816_b200 import _lib  # noqa: E402

v = int(sys.argv[1]) if len(sys.argv) > 1 else 30
M, N = int(os.environ.get("GEMM_M", 1 << 18)), 1024
lib = _lib.load()
A = torch.randn(M, N, dtype=torch.float64, device="cuda")
B = torch.randn(N, N, dtype=torch.float64, device="cuda")
C = torch.empty(M, N, dtype=torch.float64, device="cuda")
for _ in range(2):
    _lib.check(lib.hikf_dgemm(M, N, N, A.data_ptr(), N, B.data_ptr(), N, C.data_ptr(), N, 1.0, 0.0, 0, v,
                              _lib.stream_ptr()))
torch.cuda.synchronize()
print("ok", v, M)
