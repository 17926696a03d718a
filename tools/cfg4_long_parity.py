"""Full-length parity at the full cfg4 size (m = 1,048,576, n = 1024, all 50
steps): the explicit and the factored updates against a torch float64
restatement of filters.py:129-157 (tests/test_gpu_fullsize.py's, run for the
whole experiment instead of 3 steps).  Prints one JSON line of relative
Frobenius errors every 10 steps."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_3816_b200 as P  # noqa: E402
from oracle import hikf_oracle as O  # noqa: E402
from tests.golden import cases  # noqa: E402
from tests.test_gpu_fullsize import _torch_reference_steps  # noqa: E402,F401
from tests.test_gpu_parity import _Model, _gpu_scenario  # noqa: E402

cfg = cases.CFG4
T = int(os.environ.get("STEPS", cfg["T"]))
grid, H = _gpu_scenario(P, cfg)
kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
model = _Model(grid, H, kern, cfg["R"])
tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
pre = P.filters.hikf_precompute_fmm(model, tree)
obs = O.observations(H, O.moving_plume(grid.cell_centers().coords, T), cfg["R"], [cfg["seed"], 0])
Hd = torch.sparse_csr_tensor(torch.as_tensor(H.indptr, dtype=torch.int64), torch.as_tensor(H.indices, dtype=torch.int64),
                             torch.as_tensor(H.data), size=H.shape).cuda()
flt = P.filters
dev = pre.C_Q_t.device
m, n = pre.C_Q_t.shape
f64 = dict(dtype=torch.float64, device=dev)
ref = {"mean": torch.zeros(m, **f64), "C": torch.zeros(m, n, **f64), "var": torch.zeros(m, **f64),
       "HC": torch.zeros(n, n, **f64)}
eye = torch.eye(n, **f64)
ex = flt.hikf_init(model)
fa = flt.hikf_init(model, representation="factored")


def rf(a, b):
    return float(torch.linalg.norm(a - b) / torch.linalg.norm(b))


out = []
for t in range(T):
    ex = flt.hikf_update(flt.hikf_predict(ex, pre), H, cfg["R"], obs[t])
    fa = flt.hikf_update(flt.hikf_predict(fa, pre), H, cfg["R"], obs[t])
    # reference step (filters.py:129-157)
    C = ref["C"] + pre.C_Q_t
    var = ref["var"] + pre.diag_Q_t
    HC = ref["HC"] + pre.HC_Q_t
    S = HC + cfg["R"] * eye
    S = 0.5 * (S + S.T)
    L = torch.linalg.cholesky(S)
    K = torch.cholesky_solve(C.T.contiguous(), L).T
    innov = torch.as_tensor(obs[t], device=dev) - Hd @ ref["mean"]
    ref["var"] = var - (K * C).sum(dim=1)
    ref["mean"] = ref["mean"] + K @ innov
    KH = torch.cholesky_solve(HC.T.contiguous(), L).T
    ref["C"] = C - K @ HC
    ref["HC"] = HC - KH @ HC
    del K, C
    if (t + 1) % 10 == 0 or t + 1 == T:
        row = {"step": t + 1}
        for name, st in (("explicit", ex), ("factored", fa)):
            row[name] = {"mean": rf(st.mean_t, ref["mean"]), "variance": rf(st.variance_t, ref["var"]),
                         "cross_cov": rf(st.cross_cov_t, ref["C"]), "HC": rf(st.HC_t, ref["HC"])}
        out.append(row)
        print(json.dumps(row), flush=True)
