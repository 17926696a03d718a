"""Cold-start cost of the drop-in at a bench config (default cfg4): the first
build_tree + Q H^T precompute in a fresh process (CUDA context already up,
as torch has it) against the same calls warm.  Prints one JSON line.

  python tools/cold_start.py [cfg4]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1404_3816_b200 as P  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = bench.CONFIGS[args[0] if args else "cfg4"]
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
if "--preload-small" in sys.argv:  # every kernel loaded by a tiny run first: isolates the memory growth
    g1 = P.Grid2D(32, 32, 1 / 32, 1 / 32)
    H1 = P.tomography.build_ray_operator(g1, P.tomography.default_acquisition(g1, 4, 4, 0.0, 1.0))

    class M1:
        pass
    m1 = M1()
    m1.H, m1.m = H1, g1.m
    t1 = P.build_tree(g1.cell_centers(), P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"]),
                      P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=16))
    P.filters.hikf_precompute_fmm(m1, t1)
    torch.cuda.synchronize()
N = cfg["N"]
grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
t0 = time.perf_counter()
H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
t_rays = time.perf_counter() - t0


class M:
    pass


model = M()
model.H, model.m = H, grid.m
kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
out = {"rays_s": t_rays}
for tag in ("cold", "warm"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pre = P.filters.hikf_precompute_fmm(model, tree)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out[tag] = {"tree_s": t1 - t0, "qht_s": t2 - t1, "total_s": t2 - t0}
    del pre, tree
print(json.dumps(out))
