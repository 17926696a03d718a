"""Time the factored update (FactoredHikfState) at cfg4: warm-up 3, 10 timed
steps; prints ms/step and the per-scope stage times (hikf_prof_*).  Env knobs:
HIKF_TRI_VARIANT (triangular GEMM tile variant), HIKF_GEMV_OVERLAP (0/1)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import numpy as np  # noqa: E402
import paper_1404_3816_b200 as P  # noqa: E402
from paper_1404_3816_b200 import _lib  # noqa: E402

cfg = bench.CONFIGS[os.environ.get("CFG", "cfg4")]
N = cfg["N"]
grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
obs = bench.plume_observations(H, grid.cell_centers().coords, cfg["T"], cfg["R"])


class Model:
    pass


model = Model()
model.H, model.m, model.alpha, model.initial_mean = H, grid.m, 0.0, np.zeros(grid.m)
kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
pre = P.filters.hikf_precompute_fmm(model, tree)
lib = _lib.load()
Zd = torch.from_numpy(obs).cuda()
st = P.filters.hikf_init(model, representation="factored")
for t in range(3):
    st = P.filters.hikf_update(P.filters.hikf_predict(st, pre), H, cfg["R"], Zd[t])
torch.cuda.synchronize()
lib.hikf_prof_reset()
lib.hikf_prof_enable(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for t in range(10):
    st = P.filters.hikf_update(P.filters.hikf_predict(st, pre), H, cfg["R"], Zd[3 + t])
e1.record()
torch.cuda.synchronize()
lib.hikf_prof_enable(0)
print(json.dumps({"env": {k: os.environ.get(k) for k in ("HIKF_TRI_VARIANT", "HIKF_GEMV_OVERLAP")},
                  "ms_per_step": e0.elapsed_time(e1) / 10,
                  "stages": {s: _lib.prof_read(s) for s in ("factor", "gemm_y", "finalize", "gemm_c")}}))
