"""Bitwise digest of the update path (A/B checks of kernel changes that must be
bit-identical): spd_solve on seeded SPD matrices, then 10 fused steps of the
cfg2 filter; prints sha256 prefixes and the device time per step.
    HIKF_LIB_PATH=ab/libhikf_b200_old.so python tools/update_digest.py"""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1404_3816_b200 as P  # noqa: E402


def sha(*ts):
    h = hashlib.sha256()
    for t in ts:
        h.update(t.detach().cpu().numpy().tobytes())
    return h.hexdigest()[:16]


rng = np.random.default_rng(5)
out = []
for n in (37, 64, 200, 513):
    A = rng.standard_normal((n, n))
    A = A @ A.T + n * np.eye(n)
    B = rng.standard_normal((n, 7))
    out.append(sha(P.spd_solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())))
cfg = bench.CONFIGS[os.environ.get("CFG", "cfg2")]
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
for rep in ("explicit", "factored"):
    st = P.filters.hikf_init(model, representation=rep)
    for t in range(3):
        st = P.filters.hikf_update(P.filters.hikf_predict(st, pre), H, cfg["R"], obs[t])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(3, 13):
        st = P.filters.hikf_update(P.filters.hikf_predict(st, pre), H, cfg["R"], obs[t])
    e1.record()
    torch.cuda.synchronize()
    out.append(f"{rep}:{sha(st.mean_t, st.variance_t, st.HC_t)}:{e0.elapsed_time(e1) / 10:.3f}ms")
print(" ".join(out))
