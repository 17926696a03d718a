"""The CUDA row-sharded filter under world = 2: two gloo ranks
sharing cuda:0 each own a leaf-aligned block of rows (sharded.leaf_block),
compute their Q H^T shard with hikf_precompute_leaves (P2P / leaf L2L + L2P for
their leaves, M2L / L2L for the ancestors only) and run hikf_csr_spmv +
hikf_update_rows with the deferred on-device variance check.  The gathered
result must equal the one-rank update through the public API (filters.py:129-157)
to 1e-12, the shard's C_Q rows must equal the full precompute's bit for bit, and
a rank-local violation must raise on both ranks at the next host touch."""

import os
import socket

import numpy as np
import pytest

from oracle import hikf_oracle as O
from tests.golden import cases

pytestmark = pytest.mark.gpu

CFG = dict(cases.CFG1, T=6)


def _scenario(P):
    N = CFG["N"]
    grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
    H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, CFG["ns"], CFG["nr"], 0.0, 1.0))
    kern = P.KernelSpec(CFG["family"], variance=1.0, length_scale=CFG["L"])
    tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=CFG["order"], max_leaf_points=CFG["leaf"]))
    obs = O.observations(H, O.moving_plume(grid.cell_centers().coords, CFG["T"]), CFG["R"], [5, 0])
    return grid, H, tree, obs


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1404_3816_b200 as P
        from paper_1404_3816_b200 import sharded as SH
        grid, H, tree, obs = _scenario(P)
        m, n = grid.m, H.shape[0]
        leaf0, leaf1, s0, s1 = SH.leaf_block(tree, world, rank)
        rows = tree.export()["order"][s0:s1]
        comm = SH.TorchComm()
        CQ, HCQ, dQ = SH.precompute_leaves(tree, H, leaf0, leaf1, comm)
        step = SH.CudaRowStep((CQ, HCQ, dQ), n)
        sh = SH.ShardedHikf(comm, step, H, m, rank, world, rows=rows)
        z = lambda *s: torch.zeros(*s, dtype=torch.float64, device="cuda")  # noqa: E731
        st = {"mean": z(s1 - s0), "C": z((s1 - s0, n)), "var": z(s1 - s0), "HC": z((n, n))}
        for t in range(CFG["T"]):
            st = sh.update(st, CFG["R"], obs[t])
        mean, var = sh.gather(st["mean"], m), sh.gather(st["var"], m)
        C = sh.gather(st["C"], m)
        q.put(("ok", rank, (leaf0, leaf1, s0, s1), rows, CQ.cpu().numpy(), mean, var, C, st["HC"].cpu().numpy()))
        # a rank-local violation (rank 1's prior variance made hugely negative) must raise on
        # both ranks -- deferred: at the next host touch (check())
        bad = dict(st)
        if rank == 1:
            bad["var"] = st["var"] - 1e6
        try:
            sh.update(bad, CFG["R"], obs[0])
            sh.check()
            q.put(("no-raise", rank))
        except Exception as exc:  # NumericalConsistencyError expected on both ranks
            q.put(("raised", rank, type(exc).__name__))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_cuda_sharded_world2_leaf_blocks():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    import paper_1404_3816_b200 as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=600) for _ in range(4)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ok = sorted([m for m in msgs if m[0] == "ok"], key=lambda m: m[1])
    assert len(ok) == 2
    # leaf blocks tile the leaves and rows
    (a0, a1, r00, r01), (b0, b1, r10, r11) = ok[0][2], ok[1][2]
    assert a0 == 0 and a1 == b0 and r00 == 0 and r01 == r10
    grid, H, tree, obs = _scenario(P)
    assert b1 == tree.export()["leaf_starts"].shape[0] and r11 == grid.m
    assert np.array_equal(np.concatenate([ok[0][3], ok[1][3]]), tree.export()["order"])
    # the one-rank run through the public API
    class M:
        pass
    model = M()
    model.H, model.m, model.alpha, model.initial_mean = H, grid.m, 0.0, np.zeros(grid.m)
    pre = P.filters.hikf_precompute_fmm(model, tree)
    CQ_full = pre.C_Q
    for rk in ok:  # the shard's C_Q rows are the full precompute's rows, bit for bit
        assert np.array_equal(rk[4], CQ_full[rk[3]]), rk[1]
    st = P.filters.hikf_init(model)
    for t in range(CFG["T"]):
        st = P.filters.hikf_update(P.filters.hikf_predict(st, pre), H, CFG["R"], obs[t])
    assert np.array_equal(ok[0][8], ok[1][8])  # replicated HC bitwise equal across ranks
    for k, ref in (("mean", st.mean), ("var", st.variance), ("C", st.cross_cov)):
        got = ok[0][{"mean": 5, "var": 6, "C": 7}[k]]
        assert np.array_equal(got, ok[1][{"mean": 5, "var": 6, "C": 7}[k]])  # gathered identically
        assert O.rel_fro(got, ref) <= 1e-12, k
    assert O.rel_fro(ok[0][8], st.HC) <= 1e-12
    raised = [m for m in msgs if m[0] == "raised"]
    assert len(raised) == 2 and all(m[2] == "NumericalConsistencyError" for m in raised), msgs


@pytest.mark.parametrize("N,world", [(96, 3), (256, 4)])
def test_leaf_shards_reproduce_the_full_precompute(N, world):
    """hikf_precompute_leaves on every leaf block of a deeper tree (M2L / L2L restricted
    to the ancestors' box columns): the shards' C_Q rows are the full precompute's rows
    bit for bit, diag_Q matches, and the all-reduced HC_Q partials give HC_Q to 1e-13."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1404_3816_b200 as P
    from paper_1404_3816_b200 import sharded as SH
    cfg = dict(cases.CFG2, N=N)
    grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
    H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
    kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
    tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))

    class M:
        pass
    model = M()
    model.H, model.m = H, grid.m
    pre = P.filters.hikf_precompute_fmm(model, tree)
    order = tree.export()["order"]
    X = None
    for r in range(world):
        leaf0, leaf1, s0, s1 = SH.leaf_block(tree, world, r)
        CQ, Xr, dQ = SH.precompute_leaves(tree, H, leaf0, leaf1)
        assert torch.equal(CQ, pre.C_Q_t[torch.as_tensor(order[s0:s1], device="cuda")]), (r, tree.depth)
        assert torch.equal(dQ, pre.diag_Q_t[torch.as_tensor(order[s0:s1], device="cuda")])
        X = Xr if X is None else X + Xr
    HCQ = 0.5 * (X + X.T)
    assert float((HCQ - pre.HC_Q_t).norm() / pre.HC_Q_t.norm()) <= 1e-13
