"""One fused predict+update at the cfg4 shape (m = 1048576, n = 1024) on
synthetic SPD data through the C ABI, with the profiled update inside an NVTX
range "update" so ncu can select exactly that step's kernels:

  ncu --nvtx --nvtx-include "update/" --set full ... python tools/prof_update.py

Prints the step time (CUDA events) and the stage times (hikf_prof_*)."""

import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1404_3816_b200 import _lib  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
f64 = dict(dtype=torch.float64, device=dev)
A = torch.randn(n, n, generator=g, **f64)
HC = A @ A.T / n + torch.eye(n, **f64)
HCQ = 0.1 * torch.eye(n, **f64)
C = torch.randn(m, n, generator=g, **f64) * 1e-2
CQ = torch.randn(m, n, generator=g, **f64) * 1e-2
var = torch.full((m,), 1e6, **f64)
dQ = torch.ones(m, **f64)
mean = torch.randn(m, generator=g, **f64)
z = torch.randn(n, generator=g, **f64)
# a diagonal-ish H: ray i sees cells i*k .. i*k+3
k = m // n
ip = torch.arange(0, 4 * n + 1, 4, dtype=torch.int32, device=dev)
ix = (torch.arange(n, device=dev).repeat_interleave(4) * k + torch.arange(4, device=dev).repeat(n)).to(torch.int32)
val = torch.full((4 * n,), 0.25, **f64)
outs = [torch.empty_like(t) for t in (mean, C, var, HC)]
lib = _lib.load()
ws = torch.empty(int(lib.hikf_update_workspace_bytes(m, n)), dtype=torch.uint8, device=dev)
mv = ctypes.c_double(0.0)


mode = sys.argv[3] if len(sys.argv) > 3 else "update"


def step():
    fused = mode != "nopredict"  # nopredict: update only (no fused predict), factor timed alone
    # produce the next step's C' in the GEMM epilogue, as the filter loop does (hikf_update_chained bit 0)
    _lib.check(lib.hikf_update_chained(m, n, mean.data_ptr(), C.data_ptr(), var.data_ptr(), HC.data_ptr(),
                                       CQ.data_ptr() if fused else None, dQ.data_ptr() if fused else None,
                                       HCQ.data_ptr() if fused else None, ip.data_ptr(), ix.data_ptr(),
                                       val.data_ptr(), 1e-3, z.data_ptr(), outs[0].data_ptr(), outs[1].data_ptr(),
                                       outs[2].data_ptr(), outs[3].data_ptr(), ws.data_ptr(), ws.numel(),
                                       ctypes.byref(mv), 1 if fused else 0, None, _lib.stream_ptr()))


if mode == "gemm":
    # only the two m x n x n GEMMs of the update, with the update's operands and variants:
    # Y = C' Li^T (B upper triangular, variant 10) and C_new = C' - Y P (variant 7)
    Y = torch.empty_like(C)
    LiT = torch.triu(torch.randn(n, n, generator=g, **f64)) / n
    P = torch.randn(n, n, generator=g, **f64) / n

    def step():  # noqa: F811
        _lib.check(lib.hikf_dgemm(m, n, n, C.data_ptr(), n, LiT.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, 1, 10,
                                  _lib.stream_ptr()))
        _lib.check(lib.hikf_dgemm(m, n, n, Y.data_ptr(), n, P.data_ptr(), n, outs[1].data_ptr(), n, -1.0, 1.0, 0, 7,
                                  _lib.stream_ptr()))

for _ in range(2):
    step()
torch.cuda.synchronize()
lib.hikf_prof_enable(1)
lib.hikf_prof_reset()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.nvtx.range_push("update")
e0.record()
step()
e1.record()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print(json.dumps({"mode": mode, "m": m, "n": n, "ms": e0.elapsed_time(e1), "stages_ms": {k: _lib.prof_read(k)[0] for k in _lib.STAGES}}))
