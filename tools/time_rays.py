"""Time the ray operator build at cfg4 (1024 x 1024 cells, 32 x 32 rays):
the device tracer (hikf_ray_operator_device), the native host tracer
(hikf_ray_operator) and, on a bounded sample of rays, the oracle's
restatement of the reference's per-ray Python loop (tomography.py:76-133)."""

import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1404_3816_b200 as P  # noqa: E402
from oracle import hikf_oracle as O  # noqa: E402

N = 1024
grid = P.Grid2D(nx=N, ny=N, dx=1.0 / N, dy=1.0 / N)
acq = P.tomography.default_acquisition(grid, 32, 32, 0.0, 1.0)
out = {}
for _ in range(3):
    P.tomography.build_ray_operator_device(grid, acq)
torch.cuda.synchronize()
reps = 20
t0 = time.perf_counter()
for _ in range(reps):
    Hd = P.tomography.build_ray_operator_device(grid, acq)
torch.cuda.synchronize()
out["device_ms"] = (time.perf_counter() - t0) / reps * 1e3
t0 = time.perf_counter()
for _ in range(3):
    Hh = P.tomography.build_ray_operator(grid, acq)
out["host_native_ms"] = (time.perf_counter() - t0) / 3 * 1e3
src, rcv = acq.ray_endpoints()
k = 64
t0 = time.perf_counter()
O.ray_operator(N, N, 1.0 / N, 1.0 / N, src[:k], rcv[:k])
out["oracle_ms_full_extrapolated"] = (time.perf_counter() - t0) / k * len(src) * 1e3
out["nnz"] = int(Hd.nnz)
A = Hd.to_scipy()
out["bit_identical"] = bool(np.array_equal(A.indices, Hh.indices) and np.array_equal(A.indptr, Hh.indptr)
                            and np.array_equal(A.data.view(np.uint64), Hh.data.view(np.uint64)))
print(json.dumps(out))
