"""Q H^T precompute timing (best of 4) and a C_Q digest, to check that a
kernel change is bit-identical:  python tools/qht_time.py cfg4"""
import hashlib
import sys

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_1404_3816_b200 as P  # noqa: E402
cfg = bench.CONFIGS[sys.argv[1]]
N = cfg["N"]
grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
class M: pass
model = M(); model.H, model.m = H, grid.m
kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
pre = P.filters.hikf_precompute_fmm(model, tree)
torch.cuda.synchronize()
best = 1e30
times = []
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    del pre
    e0.record(); pre = P.filters.hikf_precompute_fmm(model, tree); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
    times.append(e0.elapsed_time(e1))
h = hashlib.sha256(pre.C_Q_t.cpu().numpy().tobytes()).hexdigest()[:16]
print("runs", [round(x, 2) for x in times])
print(sys.argv[1], "ms", round(best, 2), "median", round(sorted(times)[len(times) // 2], 2), "sha", h)
