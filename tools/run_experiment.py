"""The reference's experiment driver on the B200 path at a BASELINE config:
experiment.run_hikf (precompute = tree + Q H^T, then T predict/update steps with
per-step mean snapshots; experiment.py:219-242), with run_hikf's own clocks.
    python tools/run_experiment.py [cfg4] [--factored]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1404_3816_b200 as P  # noqa: E402
from paper_1404_3816_b200 import experiment as E  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "cfg4"
cfg = bench.CONFIGS[name]
N, T = cfg["N"], cfg["T"]
grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
xy = grid.cell_centers().coords
kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
model = E.StateSpaceModel(grid=grid, H=H, q_kernel=kern, r_variance=cfg["R"], alpha=0.0)
obs = bench.plume_observations(H, xy, T, cfg["R"])
truth = np.zeros((T, grid.m))  # run_hikf reads only the shape of the truth
scn = E.Scenario(model=model, record=E.SimulatedRecord(truth=truth, observations=obs),
                 fmm_config=P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
if "--factored" in sys.argv:
    import functools
    E.flt.hikf_init = functools.partial(P.filters.hikf_init, representation="factored")
E.run_hikf(scn, "fmm")  # warm-up (CUDA context, allocator, kernel attributes)
run = E.run_hikf(scn, "fmm")
print(json.dumps({"config": name, "factored": "--factored" in sys.argv, "steps": T,
                  "precompute_s": run.precompute_seconds, "online_s": run.online_seconds,
                  "total_s": run.precompute_seconds + run.online_seconds,
                  "steps_per_s": T / run.online_seconds}))
