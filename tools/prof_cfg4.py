"""Profiling driver (for ncu): tree build + Q H^T precompute + `--steps` fused
predict/update steps at a bench config (default cfg4).  The Q H^T kernels are
the sparse-charge path (regroup, p2m_pairs, m2m_pairs, m2l_pairs_kernel x 40
offsets x level, box_warp_kernel L2L / L2P, p2p_sparse, p2p_scatter,
spmm_rows); see tools/prof_qht.sh for the ncu selections used in profiles/."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1404_3816_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--steps", type=int, default=1)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
N = cfg["N"]
grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
obs = bench.plume_observations(H, grid.cell_centers().coords, max(args.steps, 1), cfg["R"])


class Model:
    pass


model = Model()
model.H, model.m, model.alpha, model.initial_mean = H, grid.m, 0.0, np.zeros(grid.m)
kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
pre = P.filters.hikf_precompute_fmm(model, tree)
st = P.filters.hikf_init(model)
for t in range(args.steps):
    st = P.filters.hikf_update(P.filters.hikf_predict(st, pre), H, cfg["R"], obs[t])
print("ok", float(np.abs(st.mean).max()))
