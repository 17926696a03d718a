"""Host-side cost of one fused predict+update at a small config (default cfg1):
wall time per step of the Python API loop, and a cProfile of it.

  python tools/host_overhead.py [cfg1]"""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1404_3816_b200 as P  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]
N = cfg["N"]
grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
obs = bench.plume_observations(H, grid.cell_centers().coords, cfg["T"], cfg["R"])


class M:
    pass


model = M()
model.H, model.m, model.alpha, model.initial_mean = H, grid.m, 0.0, np.zeros(grid.m)
kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
pre = P.filters.hikf_precompute_fmm(model, tree)
Zd = torch.from_numpy(obs).cuda()
st = P.filters.hikf_init(model)
flt = P.filters
for t in range(20):
    st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], Zd[t % cfg["T"]])
torch.cuda.synchronize()
K = 300
t0 = time.perf_counter()
for t in range(K):
    st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], Zd[t % cfg["T"]])
torch.cuda.synchronize()
print(f"{cfg['N']}^2 x {H.shape[0]}: {1e6 * (time.perf_counter() - t0) / K:.1f} us per step (wall)")
pr = cProfile.Profile()
pr.enable()
for t in range(K):
    st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], Zd[t % cfg["T"]])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
