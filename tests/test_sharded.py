"""Row-sharded filter orchestration (paper_1404_3816_b200/sharded.py) on the
CPU with world_size 2 over gloo: the per-step all-reduce of H mean and the
global variance check, driven by a host (numpy) local step that restates the
reference update on a block of rows.  The sharded run must reproduce the
unsharded oracle run (filters.py:129-157) and raise on every rank when any
rank's rows violate the variance check."""

import os
import socket

import numpy as np
import pytest
import scipy.linalg

from oracle import hikf_oracle as O
from tests.golden import cases


class HostRowStep:
    """Reference update (filters.py:129-157) restricted to a block of rows; test-only."""

    def __init__(self, pre, r0, r1):
        self.CQ = pre.C_Q[r0:r1]
        self.dQ = pre.diag_Q[r0:r1]
        self.HCQ = pre.HC_Q

    def prepare_h(self, H_local):
        return H_local

    def spmv(self, H_local, state):
        return np.asarray(H_local @ state["mean"])

    def update_rows(self, state, Hmean, r, z):
        C = state["C"] + self.CQ
        var = state["var"] + self.dQ
        HC = state["HC"] + self.HCQ
        n = HC.shape[0]
        S = HC + r * np.eye(n)
        S = 0.5 * (S + S.T)
        fac = scipy.linalg.cho_factor(S, lower=True)
        K = scipy.linalg.cho_solve(fac, C.T).T
        mean = state["mean"] + K @ (np.asarray(z) - np.asarray(Hmean))
        var_new = var - np.einsum("ij,ij->i", K, C)
        KH = scipy.linalg.cho_solve(fac, HC.T).T
        out = {"mean": mean, "C": C - K @ HC, "var": var_new, "HC": HC - KH @ HC}
        return out, (float(var_new.min()), float(var.max()))


def _scenario():
    cfg = cases.SMALL
    N = cfg["N"]
    xy = O.cell_centers(N, N, 1.0 / N, 1.0 / N)
    src, rcv = O.crosswell_stations(cfg["ns"], cfg["nr"], 0.0, 1.0, 0.0, 1.0)
    H = O.ray_operator(N, N, 1.0 / N, 1.0 / N, src, rcv)
    tree = O.OracleTree(xy, O.Kern(cfg["family"], 1.0, cfg["L"]), cfg["order"], cfg["leaf"])
    pre = O.precompute(H, tree)
    obs = O.observations(H, cases.plume_fields(xy, cfg["T"]), cfg["R"], [cfg["seed"], 0])
    return cfg, H, pre, obs


def _worker(rank, world, port, result_q):
    import torch.distributed as dist
    from paper_1404_3816_b200.sharded import ShardedHikf, TorchComm, row_block
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, H, pre, obs = _scenario()
        m, n = H.shape[1], H.shape[0]
        r0, r1 = row_block(m, world, rank)
        sh = ShardedHikf(TorchComm(), HostRowStep(pre, r0, r1), H, m, rank, world)
        st = {"mean": np.zeros(r1 - r0), "C": np.zeros((r1 - r0, n)), "var": np.zeros(r1 - r0),
              "HC": np.zeros((n, n))}
        for t in range(cfg["T"]):
            st = sh.update(st, cfg["R"], obs[t])
        result_q.put(("ok", rank, r0, r1, st["mean"], st["var"], st["C"], st["HC"]))
        # a rank-local violation must raise on every rank
        bad = dict(st)
        if rank == 1:
            bad = dict(st, var=st["var"] - 1e6)
        try:
            sh.update(bad, cfg["R"], obs[0])
            result_q.put(("no-raise", rank))
        except Exception as exc:  # NumericalConsistencyError expected on both ranks
            result_q.put(("raised", rank, type(exc).__name__))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_block_partition():
    from paper_1404_3816_b200.sharded import row_block
    for m in (1, 7, 576, 1000):
        for w in (1, 2, 3, 8):
            blocks = [row_block(m, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1


def test_sharded_world2_matches_unsharded():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(4)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ok = sorted([m for m in msgs if m[0] == "ok"], key=lambda m: m[1])
    assert len(ok) == 2
    mean = np.concatenate([m[4] for m in ok])
    var = np.concatenate([m[5] for m in ok])
    C = np.concatenate([m[6] for m in ok])
    assert np.array_equal(ok[0][7], ok[1][7])  # replicated HC stays bitwise identical
    # unsharded oracle run
    cfg, H, pre, obs = _scenario()
    st = O.init_state(H, H.shape[1])
    for t in range(cfg["T"]):
        st = O.update(O.predict(st, pre), H, cfg["R"], obs[t])
    assert O.rel_fro(mean, st.mean) <= 1e-12
    assert O.rel_fro(var, st.variance) <= 1e-12
    assert O.rel_fro(C, st.cross_cov) <= 1e-12
    assert O.rel_fro(ok[0][7], st.HC) <= 1e-12
    raised = [m for m in msgs if m[0] == "raised"]
    assert len(raised) == 2 and all(m[2] == "NumericalConsistencyError" for m in raised)
