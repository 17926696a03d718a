"""Where does the e2e loop (bench.py) spend time beyond the device-resident
loop?  cfg4 filter steps with (a) device z, (b) host z, (c) host z + mean
read-back, each timed with CUDA events over 8 steps."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1404_3816_b200 as P  # noqa: E402

cfg = bench.CONFIGS["cfg4"]
N = cfg["N"]
grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
obs = bench.plume_observations(H, grid.cell_centers().coords, cfg["T"], cfg["R"])
model = type("M", (), dict(H=H, m=grid.m, alpha=0.0, initial_mean=np.zeros(grid.m)))()
kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
flt = P.filters
pre = flt.hikf_precompute_fmm(model, tree)
st = flt.hikf_init(model)
Zd = torch.from_numpy(obs).cuda()
for t in range(3):
    st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], Zd[t])
means = np.empty((8, grid.m))
for mode in ("device z", "host z", "host z + mean", "device z + mean", "device z"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for t in range(8):
        z = Zd[t] if mode.startswith("device") else obs[t]
        st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], z)
        if "mean" in mode:
            means[t] = st.mean
    e1.record()
    torch.cuda.synchronize()
    print(f"{mode:18s} {e0.elapsed_time(e1) / 8:.2f} ms/step (wall {1e3 * (time.perf_counter() - w0) / 8:.2f})")
