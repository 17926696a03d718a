"""Benchmark of the B200 HiKF hot path (BASELINE.json metric):

    HiKF assimilation steps/sec  (+ Q H^T (m n)/sec of the bbFMM precompute)

on cfg4 (2D 1024 x 1024 grid, m = 1,048,576, n = 1,024 crosswell rays,
exponential kernel L = 0.25, Chebyshev order 6, leaf 64, R = 1e-3).

One "step" = hikf_predict + hikf_update (the fused predict/update of
libhikf_b200.so) on device-resident inputs; `value` = steps/s over exactly
--steps timed steps after --warmup untimed ones (CUDA events, barrier +
synchronize on both sides, max over ranks).  The state (C is 8.6 GB) is far
larger than L2 (126 MB), so no flush is needed between steps.

`e2e` is the same metric through the public Python API with host buffers:
every step uploads z (numpy, 8 n bytes) and reads the posterior mean back to
numpy (8 m bytes), exactly what experiment.run_hikf does (experiment.py:237).

`--impl reference` times the reference algorithm on the host CPU cores: the
reference is pure Python and cannot travel to the GPU box, so its numpy
restatement in oracle/ (pinned to the reference by tests/test_oracle_golden.py)
runs full-size steps of the config's scenario (CpuFilter; prior Q = I stand-in,
the step cost being independent of the values).

Multi-GPU (--gpus N under torchrun): independent replicas, one filter per
GPU ("replicas only" this round); value sums ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

# The reference arm (--impl reference) runs the CPU algorithm alone on rank 0 with every host
# thread.  torchrun exports OMP_NUM_THREADS=1 to multi-process launches, and OpenBLAS sizes its
# pool from that when numpy is first imported, so the override must precede `import numpy`.
if "--impl" in sys.argv and sys.argv[sys.argv.index("--impl") + 1:][:1] == ["reference"]:
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[_v] = str(os.cpu_count() or 1)

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(N=64, ns=8, nr=8, family="exponential", L=0.3, R=1e-2, T=20, order=4, leaf=64,
                 desc="cfg1: 2D 64x64 unit square m=4096, n=64 crosswell rays, exponential L=0.3, order 4, leaf 64"),
    "cfg2": dict(N=256, ns=16, nr=16, family="gaussian", L=0.2, R=1e-3, T=100, order=5, leaf=64,
                 desc="cfg2: 2D 256x256 m=65536, n=256 crosswell rays, gaussian L=0.2, order 5, leaf 64"),
    "cfg4": dict(N=1024, ns=32, nr=32, family="exponential", L=0.25, R=1e-3, T=50, order=6, leaf=64,
                 desc="cfg4: 2D 1024x1024 m=1048576, n=1024 crosswell rays, exponential L=0.25, order 6, leaf 64"),
    # 3D (no reference oracle: parity unpinned)
    "cfg3": dict(dim=3, N=64, ns=24, nr=20, family="exponential", ls=(0.3, 0.3, 0.3), R=1e-3, T=100, order=5,
                 leaf=128, plumes=[(0.2, 0.5, 0.5, 0.08, 0.005)],
                 desc="cfg3: 3D 64^3 m=262144, n=480 jittered crosswell rays, exponential L=0.3, order 5, leaf 128"),
    "cfg5": dict(dim=3, N=128, ns=32, nr=32, family="exponential", ls=(0.4, 0.4, 0.1), R=5e-4, T=50, order=5,
                 leaf=128, plumes=[(0.3, 0.4, 0.5, 0.06, 0.005), (0.7, 0.6, 0.5, 0.1, -0.005)],
                 desc="cfg5: 3D 128^3 m=2097152, n=1024 jittered crosswell rays, anisotropic exponential "
                      "(0.4, 0.4, 0.1), order 5, leaf 128"),
}


def cfg_m(cfg):
    return cfg["N"] ** cfg.get("dim", 2)

# FP64 roofline denominator: MEASURED_PEAKS.json has no FP64 entry; this is the
# cuBLAS DGEMM (torch.matmul float64, 8192^3) we measured on this pool's B200
# (profiles/r01_fp64_dgemm.json: 35.48 burst / 35.46 sustained TFLOP/s; the
# DMMA/DFMA issue-rate microbenchmark gives 37.0, profiles/r01_fp64_micro.json).
FP64_PEAK_TFLOPS = 35.46
FP64_PEAK_SOURCE = "measured cuBLAS DGEMM 8192^3 on B200 (profiles/r01_fp64_dgemm.json); not in MEASURED_PEAKS.json"
# DRAM traffic of one chained K-GEMM launch at cfg4 from `ncu --set full` (dram__bytes_read.sum +
# dram__bytes_write.sum); the algorithmic bytes are C' and C_Q in, C_new and the next C' out
# = 4 x 8 m n = 34.4 GB (S^-1 stays in L2).
C_GEMM_TRAFFIC_CFG4 = 17.74e9 + 17.37e9  # ncu dram read + write of the chained K GEMM (profiles/r01_ncu_kgemm_cutlass_summary.txt)


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# scenario (host inputs)
# ---------------------------------------------------------------------------

def plume_observations(H, xy, T, R, seed=0):
    """Constant-amplitude moving Gaussian plume (w = 0.1 from (0.2, 0.5), +0.01 x
    per step) and z_t = H x_t + N(0, R) from PCG64 seed [seed, 0] (ssm.py:81-113)."""
    Z = np.empty((T, H.shape[0]))
    for t in range(1, T + 1):
        x = np.exp(-((xy[:, 0] - (0.2 + 0.01 * (t - 1))) ** 2 + (xy[:, 1] - 0.5) ** 2) / (2 * 0.1 * 0.1))
        Z[t - 1] = H @ x
    rng = np.random.default_rng([seed, 0])
    return Z + math.sqrt(R) * rng.standard_normal(Z.shape)


def fmm_flops(orders, depth, k, near_pairs_pts, m):
    """Dense-formulation flops of one matmat."""
    nl = orders[depth]
    f = {"p2p": 2.0 * k * near_pairs_pts, "p2m": 2.0 * k * m * nl * nl, "l2p": 2.0 * k * m * nl * nl}
    mm = 0.0
    for lev in range(2, depth):
        mm += 2.0 * k * (4 ** (lev + 1)) * orders[lev + 1] ** 2 * orders[lev] ** 2
    f["m2m"] = mm
    f["l2l"] = mm
    return f


def m2l_flops(tree, k):
    tot = 0.0
    for lev in range(2, tree.depth + 1):
        pairs = 0
        G = 1 << lev
        for dx in range(-3, 4):
            for dy in range(-3, 4):
                if max(abs(dx), abs(dy)) < 2:
                    continue
                cnt = [0, 0]
                for d, c in ((dx, 0), (dy, 1)):
                    i = np.arange(G)
                    j = i + d
                    cnt[c] = int(np.sum((j >= 0) & (j < G) & (np.abs((j >> 1) - (i >> 1)) <= 1)))
                pairs += cnt[0] * cnt[1]
        tot += 2.0 * k * pairs * tree._orders[lev] ** 4
    return tot


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock and clock-event reasons sampled during the timed region: NVML polled
    from a thread every 10 ms (enough samples for short regions), else nvidia-smi."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.stop = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(int(self.index))
            self.stop = threading.Event()

            def poll():
                while True:
                    try:
                        self.samples.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                             float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                             int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))))
                    except Exception:
                        pass
                    if self.stop.wait(0.01):
                        break
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.stop = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.stop is not None:
            self.stop.set()
            self.thread.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        reasons = set()
        for s in load:
            for bit, name in self.REASONS.items():
                if s[2] & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in load), "sm_max_mhz": max(s[1] for s in load),
                "reasons": sorted(reasons), "samples": len(load)}


# ---------------------------------------------------------------------------
# CPU leg: the reference algorithm (oracle restatement) on a bounded sample
# ---------------------------------------------------------------------------

def host_info():
    """Host cores, RAM and the BLAS thread pool the CPU legs run with."""
    info = {"cpu_count": os.cpu_count()}
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal:"):
                    info["ram_gb"] = round(int(line.split()[1]) / 1024 ** 2, 1)
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    return info


def cpu_scenario(cfg):
    """The 2D config's scenario on the host through the oracle (oracle/hikf_oracle.py restates
    grids.py / tomography.py): cell centres, the crosswell ray operator, plume observations."""
    from oracle import hikf_oracle as O
    N = cfg["N"]
    xy = O.cell_centers(N, N, 1.0 / N, 1.0 / N)
    src, rcv = O.crosswell_stations(cfg["ns"], cfg["nr"], 0.0, 1.0, 0.0, 1.0)
    H = O.ray_operator(N, N, 1.0 / N, 1.0 / N, src, rcv)
    return xy, H, plume_observations(H, xy, cfg["T"], cfg["R"])


class CpuFilter:
    """The reference's predict + update (oracle restatement of filters.py:129-157: numpy +
    OpenBLAS / LAPACK cho_factor / cho_solve) on the FULL m x n state of the config.

    The prior is the white-noise stand-in Q = I (C_Q = H^T, HC_Q = H H^T, diag_Q = 1): the CPU
    bbFMM for the real C_Q takes ~20 min at cfg4 (see cpu_baseline.qht), and a step's cost is
    dense BLAS / LAPACK on m x n and n x n arrays, independent of the values."""

    def __init__(self, cfg, rows=None, H=None, obs=None):
        from oracle import hikf_oracle as O
        self.O = O
        if H is None:
            _, H, obs = cpu_scenario(cfg)
        m = H.shape[1]
        if rows is not None and rows < m:  # leading rows (a row sample, cross-check only)
            H = H[:, :rows].tocsr()
            m = rows
        self.H, self.obs, self.R, self.m = H, obs, cfg["R"], m
        t0 = time.perf_counter()
        Ht = np.ascontiguousarray(H.T.toarray())
        self.pre = O.Pre(Ht, np.asarray((H @ Ht)), np.ones(m))
        self.st = O.init_state(H, m)
        self.t_setup = time.perf_counter() - t0
        self.t = 0

    def step(self):
        O = self.O
        t0 = time.perf_counter()
        self.st = O.update(O.predict(self.st, self.pre), self.H, self.R, self.obs[self.t % len(self.obs)])
        self.t += 1
        return time.perf_counter() - t0


def scenario_3d(cfg):
    """3D scenario (space3d, recipe restated in oracle/hikf_oracle3d.py): grid,
    seeded jittered crosswell, ray operator, plume observations."""
    from paper_1404_3816_b200 import space3d as S
    from oracle import hikf_oracle3d as O3
    N = cfg["N"]
    grid = S.Grid3D(N, N, N, 1.0 / N, 1.0 / N, 1.0 / N)
    H = S.build_ray_operator_3d(grid, S.crosswell_3d(grid, cfg["ns"], cfg["nr"], 0))
    xyz = grid.cell_centers().coords
    F = O3.plumes_3d(xyz, cfg["T"], cfg["plumes"])
    Z = np.asarray((H @ F[1:].T).T)
    rng = np.random.default_rng([0, 0])
    return grid, H, xyz, Z + math.sqrt(cfg["R"]) * rng.standard_normal(Z.shape)


def fmm3_flops(tree, k):
    """Dense-formulation flops of the 3D product as csrc/fmm3d.cu performs it
    (expansions of every box at every level)."""
    ex = tree.export()
    q, D, G = tree.n_cheb ** 3, tree.depth, 1 << tree.depth
    keys, cnt = ex["leaf_keys"], ex["leaf_counts"]
    lut = dict(zip(keys.tolist(), cnt.tolist()))
    near = 0
    for key, c in zip(keys.tolist(), cnt.tolist()):
        bx, by, bz = key // (G * G), (key // G) % G, key % G
        for ox in (-1, 0, 1):
            for oy in (-1, 0, 1):
                for oz in (-1, 0, 1):
                    x, y, z = bx + ox, by + oy, bz + oz
                    if 0 <= x < G and 0 <= y < G and 0 <= z < G:
                        near += c * lut.get((x * G + y) * G + z, 0)
    f = {"p2p": 2.0 * k * near, "p2m": 2.0 * k * tree.m * q, "l2p": 2.0 * k * tree.m * q}
    f["m2m"] = f["l2l"] = sum(2.0 * k * 8 ** (lev + 1) * q * q for lev in range(2, D))
    m2l = 0.0
    for lev in range(2, D + 1):
        Gl = 1 << lev
        i = np.arange(Gl)
        per_axis = {}
        for d in range(-3, 4):
            j = i + d
            per_axis[d] = {c: int(np.sum((j >= 0) & (j < Gl) & (i % 2 == c) &
                                         (np.abs((j >> 1) - (i >> 1)) <= 1))) for c in (0, 1)}
        for a in range(-3, 4):
            for b in range(-3, 4):
                for c in range(-3, 4):
                    if max(abs(a), abs(b), abs(c)) < 2:
                        continue
                    m2l += sum(per_axis[a][x] * per_axis[b][y] * per_axis[c][z]
                               for x in (0, 1) for y in (0, 1) for z in (0, 1))
    f["m2l"] = 2.0 * k * q * q * m2l if D >= 2 else 0.0
    return f


def cpu_qht_sample_3d(cfg, H, xyz, cols=2):
    """Exact Q H^T columns on the host (direct sum over each ray's cells, numpy):
    the CPU baseline for the 3D precompute (the reference has no 3D path)."""
    ls = np.array(cfg["ls"])
    X = xyz / ls
    sel = np.linspace(0, H.shape[0] - 1, cols).astype(int)
    t0 = time.perf_counter()
    for j in sel:
        c = H.indices[H.indptr[j]:H.indptr[j + 1]]
        h = H.data[H.indptr[j]:H.indptr[j + 1]]
        acc = np.zeros(len(X))
        for s in range(0, len(c), 16):
            d = X[:, None, :] - X[None, c[s:s + 16], :]
            r = np.sqrt((d * d).sum(-1))
            acc += np.exp(-(r * r if cfg["family"] == "gaussian" else r)) @ h[s:s + 16]
    t = time.perf_counter() - t0
    return len(X) * cols / t, t


def cpu_qht_sample(cfg, cols=32):
    """Reference bbFMM (oracle restatement) Q H^T on `cols` columns of H^T
    (matmat is column-independent, fmm.py:325-367): (m n)/s = m cols / t."""
    from oracle import hikf_oracle as O
    N = cfg["N"]
    xy = O.cell_centers(N, N, 1.0 / N, 1.0 / N)
    src, rcv = O.crosswell_stations(cfg["ns"], cfg["nr"], 0.0, 1.0, 0.0, 1.0)
    H = O.ray_operator(N, N, 1.0 / N, 1.0 / N, src, rcv)
    t0 = time.perf_counter()
    tree = O.OracleTree(xy, O.Kern(cfg["family"], 1.0, cfg["L"]), cfg["order"], cfg["leaf"])
    t_build = time.perf_counter() - t0
    sel = np.linspace(0, H.shape[0] - 1, cols).astype(int)
    V = np.ascontiguousarray(H[sel].T.toarray())
    t0 = time.perf_counter()
    tree.matmat(V)
    t = time.perf_counter() - t0
    return N * N * cols / t, t_build, t


def arm_config(args, cfg, world, mode):
    """The `config` object of the bench line, shared by both arms (same_config)."""
    c = {"workload": cfg["desc"], "steps_per_run": cfg["T"],
         "l2": "no flush: per-step inputs (C 8.6 GB, C_Q 8.6 GB) far exceed the 126 MB L2"
         if args.config == "cfg4" else "small config: inputs may be L2-resident"}
    if mode == "sharded":
        c["parallelism"] = f"row-sharded x{world} (one n-vector all-reduce per step)"
    else:
        c["parallelism"] = f"replicas x{world}" if world > 1 else "single GPU"
    return c


def arm_mode(args, cfg, world):
    mode = args.mode
    if mode == "auto":
        mode = "sharded" if world > 1 and cfg.get("dim", 2) == 2 else "replicas"
    return mode


def run_reference(args, cfg, rank):
    """--impl reference: the reference algorithm (oracle port) on the host cores, rank 0
    only, on the full m x n state of the config.  Warm-up: the first untimed step is a full
    step (page faults, BLAS thread pool); the other W - 1 run on a 65,536-row sample so the
    whole run stays within a few minutes.  Timed: exactly K full steps."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    if cfg.get("dim", 2) != 2:
        print(json.dumps({"impl": "reference", "unavailable": "the reference is 2D only (grids.py:59-66)"}))
        return
    threads = os.cpu_count()
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=threads):
        if args.warmup > 1:
            small = CpuFilter(cfg, rows=min(65536, cfg_m(cfg)))
            for _ in range(args.warmup - 1):
                small.step()
            del small
        cf = CpuFilter(cfg)
        if args.warmup > 0:
            cf.step()
        per_step = [cf.step() for _ in range(args.steps)]
    t_step = sum(per_step) / len(per_step)
    value = 1.0 / t_step
    hi = host_info()
    sample = (f"oracle/hikf_oracle.py predict+update (numpy + OpenBLAS / LAPACK, {threads} threads) on the full "
              f"{cfg_m(cfg)} x {cfg['ns'] * cfg['nr']} state of the {args.config} scenario (crosswell rays, plume "
              f"observations); prior Q = I stand-in for C_Q (step cost independent of the values); "
              f"{args.steps} timed full steps")
    line = {
        "metric": "hikf_assimilation_steps_per_sec", "value": value, "unit": "steps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded crosswell rays + moving Gaussian plume, PCG64 noise (cfg recipe, SURVEY 8(d))",
        "config": arm_config(args, cfg, world, arm_mode(args, cfg, world)), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": threads, "kind": "port", "sample": sample,
                         "host": hi, "step_s": per_step, "setup_s": cf.t_setup},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------

def run_sharded(args, cfg, P, torch, dist, world, rank, local):
    """--mode sharded: rank r owns the state rows row_block(m, world, r);
    Q H^T rows via hikf_precompute_rows (+ one n x n all-reduce), then per step one
    all-reduce of the n-vector H mean and one of the (min, max) variance pair."""
    from paper_1404_3816_b200 import sharded as SH
    if cfg.get("dim", 2) != 2:
        raise SystemExit("--mode sharded supports the 2D configs")
    N = cfg["N"]
    grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
    H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0, 1.0))
    m, n = grid.m, H.shape[0]
    obs = plume_observations(H, grid.cell_centers().coords, cfg["T"], cfg["R"])
    kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
    dev = torch.device("cuda", local)
    comm = SH.TorchComm(device=dev) if world > 1 else SH.LocalComm()

    def barrier_sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    # leaf-aligned row block (x-major leaf range, equal point counts): rows in leaf order
    leaf0, leaf1, r0, r1 = SH.leaf_block(tree, world, rank)
    rows = tree.export()["order"][r0:r1]
    for _ in range(3):  # warm-up (the stream-ordered pool settles over the first calls)
        SH.precompute_leaves(tree, H, leaf0, leaf1, comm)
    barrier_sync()
    qht_runs = []  # median of five (the stream-ordered pool settles over the first calls)
    CQ = HCQ = dQ = None
    for _ in range(5):
        del CQ, HCQ, dQ
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        CQ, HCQ, dQ = SH.precompute_leaves(tree, H, leaf0, leaf1, comm)
        e1.record()
        barrier_sync()
        qht_runs.append(e0.elapsed_time(e1) / 1e3)
    t_qht = max_over_ranks(sorted(qht_runs)[len(qht_runs) // 2])
    step = SH.CudaRowStep((CQ, HCQ, dQ), n)
    sh = SH.ShardedHikf(comm, step, H, m, rank, world, rows=rows)
    zeros = lambda *s: torch.zeros(*s, dtype=torch.float64, device=dev)  # noqa: E731
    st = {"mean": zeros(r1 - r0), "C": zeros((r1 - r0, n)), "var": zeros(r1 - r0), "HC": zeros((n, n))}
    Zd = torch.from_numpy(obs).to(dev)
    for t in range(args.warmup):
        st = sh.update(st, cfg["R"], Zd[t % cfg["T"]])
    lib = P._lib.load()
    l0 = lib.hikf_launch_count()
    lib.hikf_prof_reset()
    lib.hikf_prof_enable(1)
    barrier_sync()
    with ClockSampler(local) as clk:
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for t in range(args.steps):
            st = sh.update(st, cfg["R"], Zd[(args.warmup + t) % cfg["T"]])
        s1.record()
        barrier_sync()
    sh.check()  # the deferred variance / pivot check of the last timed step
    lib.hikf_prof_enable(0)
    launches = int(lib.hikf_launch_count() - l0)
    t_loop = max_over_ranks(s0.elapsed_time(s1) / 1e3)
    ms_c, n_c = P._lib.prof_read("gemm_c")
    achieved = max_over_ranks(2.0 * (r1 - r0) * n * n / (ms_c / max(n_c, 1) / 1e3) / 1e12) if n_c else None
    # e2e: host z up, this rank's mean rows down, every step
    barrier_sync()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for t in range(args.steps):
        st = sh.update(st, cfg["R"], obs[(args.warmup + t) % cfg["T"]])
        st["mean"].cpu().numpy()
    c1.record()
    barrier_sync()
    t_e2e = max_over_ranks(c0.elapsed_time(c1) / 1e3)
    if rank == 0:
        line = {
            "metric": "hikf_assimilation_steps_per_sec", "value": args.steps / t_loop, "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * t_loop / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded crosswell rays + moving Gaussian plume, PCG64 noise (cfg recipe, SURVEY 8(d))",
            "config": arm_config(args, cfg, world, "sharded"), "rows_per_rank": r1 - r0,
            "qht": {"ms": 1000.0 * t_qht, "value": m * n / t_qht, "unit": "(m*n)/s",
                    "note": "leaf-aligned precompute shard: upward pass replicated; M2L / L2L for the ancestors of "
                            "the rank's leaves, P2P and the fused leaf L2L + L2P for its own leaves"},
            "e2e": {"value": args.steps / t_e2e, "unit": "steps/s", "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 8 * (r1 - r0), "api": "sharded.ShardedHikf.update (numpy z) + mean rows"},
            "roofline": {"kernel": "dgemm_rm_kernel (K = C' S^-1 on this rank's rows, fused epilogue; "
                                   "2 (m/N) n^2 flops per launch)", "bound": "fp64", "achieved": achieved,
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS if achieved else None, "traffic": None,
                         "peak_source": FP64_PEAK_SOURCE},
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-factored", action="store_true",
                    help="skip the opt-in factored-representation leg (C = C_Q N) reported under 'factored'")
    ap.add_argument("--mode", default="auto", choices=["auto", "replicas", "sharded"],
                    help="replicas: every rank runs the whole filter (weak scaling); sharded: the state rows are "
                         "split across ranks with one n-vector all-reduce per step (strong scaling, 2D configs); "
                         "auto: replicas at N = 1 (the full report), sharded at N > 1 for 2D configs")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist
    # one process per GPU; HIKF_BENCH_BACKEND=gloo with more ranks than GPUs is a
    # functional check of the multi-rank path only (timings meaningless)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("HIKF_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_1404_3816_b200 as P
    from paper_1404_3816_b200 import _lib
    lib = _lib.load()
    flt = P.filters
    mode = arm_mode(args, cfg, world)
    if mode == "sharded":
        run_sharded(args, cfg, P, torch, dist, world, rank, local)
        return

    N = cfg["N"]
    dim3 = cfg.get("dim", 2) == 3
    if dim3:
        grid, H, xy, obs = scenario_3d(cfg)
        kern = P.space3d.KernelSpec3(cfg["family"], 1.0, *cfg["ls"])
    else:
        grid = P.Grid2D(N, N, 1.0 / N, 1.0 / N)
        H = P.tomography.build_ray_operator(grid, P.tomography.default_acquisition(grid, cfg["ns"], cfg["nr"], 0.0,
                                                                                   1.0))
        xy = grid.cell_centers().coords
        obs = plume_observations(H, xy, cfg["T"], cfg["R"])
        kern = P.KernelSpec(cfg["family"], variance=1.0, length_scale=cfg["L"])
    m, n = grid.m, H.shape[0]

    class Model:
        pass

    model = Model()
    model.H, model.m, model.alpha, model.initial_mean, model.r_variance = H, m, 0.0, np.zeros(m), cfg["R"]

    def barrier_sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- tree build + Q H^T precompute (one-time; timed separately) ----
    # (a tiny build first, so lazy CUDA module loading is not charged to the tree)
    if dim3:
        P.space3d.build_tree3d(np.random.default_rng(0).random((512, 3)), kern, cfg["order"], cfg["leaf"])
    else:
        P.build_tree(P.PointSet(np.random.default_rng(0).random((256, 2))), kern)
    barrier_sync()
    t0 = time.perf_counter()
    if dim3:
        tree = P.space3d.build_tree3d(grid.cell_centers(), kern, cfg["order"], cfg["leaf"])
    else:
        tree = P.build_tree(grid.cell_centers(), kern, P.FmmConfig(n_cheb=cfg["order"], max_leaf_points=cfg["leaf"]))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    for _ in range(3):  # warm-up of the precompute (the stream-ordered pool settles over the first calls)
        flt.hikf_precompute_fmm(model, tree)
    barrier_sync()
    # median of five precomputes; the cold cost is tools/cold_start.py's (profiles/*cold_start*)
    qht_runs = []
    pre = None
    for _ in range(5):
        del pre
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pre = flt.hikf_precompute_fmm(model, tree)
        e1.record()
        barrier_sync()
        qht_runs.append(e0.elapsed_time(e1) / 1e3)
    t_qht = max_over_ranks(sorted(qht_runs)[len(qht_runs) // 2])
    # stage timers and flop counters (event pairs per stage, atomics in the kernels) on an extra
    # precompute outside the timed one
    lib.hikf_prof_reset()
    lib.hikf_prof_enable(1)
    flt.hikf_precompute_fmm(model, tree)
    barrier_sync()
    lib.hikf_prof_enable(0)
    fmm_stage = {s: _lib.prof_read(s) for s in ("densify", "p2p", "p2m", "m2m", "m2l", "l2l", "l2p")}
    fmm_useful = {s: _lib.prof_flops(s) for s in ("p2p", "p2m", "m2m", "m2l", "l2l", "l2p")}
    qht_useful = float(sum(fmm_useful.values()))
    if dim3:
        ff = fmm3_flops(tree, n)  # dense formulation; the kernels skip all-zero sources and empty boxes
    else:
        ex = tree.export()
        cnt = ex["leaf_counts"]
        near_pts = float(np.sum(cnt[ex["near_t"]] * cnt[ex["near_s"]]))
        ff = fmm_flops(tree._orders, tree.depth, n, near_pts, m) if tree.depth >= 2 else {"p2p": 2.0 * n * near_pts}
        ff["m2l"] = m2l_flops(tree, n) if tree.depth >= 2 else 0.0
    qht_flops = sum(ff.values())

    # ---- filter: warm-up, then the timed region ----
    Zd = torch.from_numpy(obs).cuda()
    st = flt.hikf_init(model)
    for t in range(args.warmup):
        st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], Zd[t % cfg["T"]])
    l0 = lib.hikf_launch_count()
    barrier_sync()
    with ClockSampler(local) as clk:
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for t in range(args.steps):
            st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], Zd[(args.warmup + t) % cfg["T"]])
        s1.record()
        barrier_sync()
    launches = int(lib.hikf_launch_count() - l0)
    t_loop = max_over_ranks(s0.elapsed_time(s1) / 1e3)
    steps_per_s = world * args.steps / t_loop
    # per-stage device times (the library's CUDA-event stage timers) from a few more steps of
    # the same loop, outside the timed region: the timers add event records to every stage
    lib.hikf_prof_reset()
    lib.hikf_prof_enable(1)
    for t in range(min(args.steps, 5)):
        st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], Zd[(args.warmup + args.steps + t) % cfg["T"]])
    torch.cuda.synchronize()
    lib.hikf_prof_enable(0)
    stage = {s: _lib.prof_read(s) for s in ("predict", "factor", "gemm_y", "finalize", "gemm_c")}

    # ---- e2e: public API with host buffers (z up, mean down, every step) ----
    barrier_sync()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    means = np.empty((args.steps, m))
    c0.record()
    for t in range(args.steps):
        z_host = obs[(args.warmup + t) % cfg["T"]]
        st = flt.hikf_update(flt.hikf_predict(st, pre), H, cfg["R"], z_host)
        means[t] = st.mean
    c1.record()
    barrier_sync()
    t_e2e = max_over_ranks(c0.elapsed_time(c1) / 1e3)

    # ---- the standalone predict add (the chained loop fuses it into the K-GEMM
    # epilogue; this is the pass every unchained update runs) ----
    pc = [torch.empty_like(x) for x in (st.cross_cov_t, st.variance_t, st.HC_t)]
    pt = []
    for _ in range(4):
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        _lib.check(lib.hikf_predict(m, n, st.cross_cov_t.data_ptr(), st.variance_t.data_ptr(), st.HC_t.data_ptr(),
                                    pre.C_Q_t.data_ptr(), pre.diag_Q_t.data_ptr(), pre.HC_Q_t.data_ptr(),
                                    pc[0].data_ptr(), pc[1].data_ptr(), pc[2].data_ptr(), _lib.stream_ptr()))
        p1.record()
        torch.cuda.synchronize()
        pt.append(p0.elapsed_time(p1) / 1e3)
    del pc

    # ---- opt-in factored representation (C = C_Q N, filters.FactoredHikfState):
    # the same predict+update steps, device-resident; the headline stays explicit ----
    fac = None
    if not args.no_factored and float(model.alpha) == 0.0:
        sf = flt.hikf_init(model, representation="factored")
        for t in range(args.warmup):
            sf = flt.hikf_update(flt.hikf_predict(sf, pre), H, cfg["R"], Zd[t % cfg["T"]])
        lib.hikf_prof_reset()
        lib.hikf_prof_enable(1)
        barrier_sync()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for t in range(args.steps):
            sf = flt.hikf_update(flt.hikf_predict(sf, pre), H, cfg["R"], Zd[(args.warmup + t) % cfg["T"]])
        f1.record()
        barrier_sync()
        lib.hikf_prof_enable(0)
        t_fac = max_over_ranks(f0.elapsed_time(f1) / 1e3)
        fst = {s: _lib.prof_read(s) for s in ("predict", "factor", "gemm_y", "finalize", "gemm_c")}
        ms_t, n_t = fst["gemm_c"]
        t_tri = ms_t / max(n_t, 1) / 1e3
        bn = 64  # column tile of the K-range-limited triangular GEMM (variant 32; k >= n0 per column tile)
        tri_flops = sum(2.0 * m * min(bn, n - n0) * (n - n0) for n0 in range(0, n, bn))
        # e2e through the public API, as the explicit leg: host z up, posterior mean down, every step
        barrier_sync()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fmeans = np.empty((args.steps, m))
        g0.record()
        for t in range(args.steps):
            sf = flt.hikf_update(flt.hikf_predict(sf, pre), H, cfg["R"], obs[(args.warmup + t) % cfg["T"]])
            fmeans[t] = sf.mean
        g1.record()
        barrier_sync()
        t_fe2e = max_over_ranks(g0.elapsed_time(g1) / 1e3)
        del fmeans
        fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fe0.record()
        C_mat = sf.cross_cov_t  # one materialisation C_Q N (a user reading cross_cov)
        fe1.record()
        torch.cuda.synchronize()
        fac = {"value": world * args.steps / t_fac, "unit": "steps/s", "ms_per_step": 1000.0 * t_fac / args.steps,
               "note": "opt-in FactoredHikfState (alpha = 0): C_t = C_Q N_t with an n x n recursion; mean, variance "
                       "(with the consistency check) and HC every step as filters.py:138-157; C materialised on "
                       "read (ms_materialize, one GEMM)",
               "ms_materialize": fe0.elapsed_time(fe1),
               "e2e": {"value": world * args.steps / t_fe2e, "unit": "steps/s", "h2d_bytes_per_step": 8 * n,
                       "d2h_bytes_per_step": 8 * m},
               "stage_ms_per_step": {k: v[0] / max(v[1], 1) for k, v in fst.items()},
               "roofline": {"kernel": "dgemm_rm_kernel KB_LOWER (rowsum((C_Q L_G)^2), no output store)",
                            "bound": "fp64", "achieved": tri_flops / t_tri / 1e12 if t_tri else None,
                            "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                            "frac": tri_flops / t_tri / 1e12 / FP64_PEAK_TFLOPS if t_tri else None,
                            "flops_per_launch": tri_flops, "triangular_ideal_flops": float(m) * n * (n + 1),
                            "algorithmic_bytes": 8.0 * m * n}}
        del sf, C_mat

    # ---- rooflines ----
    hbm, hbm_src = hbm_peak()
    ms_c, n_c = stage["gemm_c"]
    ms_y, n_y = stage["gemm_y"]
    t_c = ms_c / max(n_c, 1) / 1e3
    flops_c = 2.0 * m * n * n
    achieved = flops_c / t_c / 1e12
    t_p = min(pt[1:])
    bytes_p = 24.0 * m * n + 24.0 * m + 24.0 * n * n
    # K = C' S^-1 (2 m n^2) + n x n work: Cholesky n^3/3, inverse n^3/3, S^-1 = Li^T Li, P, R, HC_new (2 n^3 each)
    update_flops = 2.0 * m * n * n + 4 * 2.0 * n ** 3 + 2 * n ** 3 / 3.0

    line = {
        "metric": "hikf_assimilation_steps_per_sec",
        "value": steps_per_s,
        "unit": "steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * t_loop / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: seeded crosswell rays + moving Gaussian plume, PCG64 noise (cfg recipe, SURVEY 8(d))",
        "config": arm_config(args, cfg, world, mode),
        "qht": {"value": world * m * n / t_qht, "unit": "(m*n)/s", "ms": 1000.0 * t_qht,
                "runs_ms": [round(1000.0 * x, 3) for x in qht_runs], "tree_build_s": t_build,
                "precompute_incl_build_mn_per_s": m * n / (t_qht + t_build),
                "flops_dense_formulation": qht_flops,
                "flops_performed": qht_useful,
                "stage_ms": {k: v[0] for k, v in fmm_stage.items()},
                "stage_gflop_performed": {k: v / 1e9 for k, v in fmm_useful.items()},
                "roofline": {"bound": "fp64", "achieved": qht_useful / t_qht / 1e12, "peak": FP64_PEAK_TFLOPS,
                             "unit": "TFLOP/s", "frac": qht_useful / t_qht / 1e12 / FP64_PEAK_TFLOPS,
                             "note": "performed flops counted in the kernels (H^T sparsity exploited: only nonzero "
                                     "charges / expansions are multiplied); dense-formulation equivalent rate = "
                                     f"{qht_flops / t_qht / 1e12:.1f} TFLOP/s",
                             "stage_ms_note": "stage_ms are event intervals on the stages' own streams; the "
                                              "streams overlap and an interval includes waits on other streams, so "
                                              "they do not add up to ms (per-kernel times: profiles/*launches_qht*)"}},
        "roofline": {"kernel": "dgemm_rm_kernel (K = C' S^-1 -> C_new = r K, fused rowsum(K o C'), K innov and the "
                               "next step's C' = C_new + C_Q; 2 m n^2 flops per launch)", "bound": "fp64",
                     "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS,
                     "traffic": C_GEMM_TRAFFIC_CFG4 if args.config == "cfg4" else None,
                     "algorithmic_bytes": 32.0 * m * n, "peak_source": FP64_PEAK_SOURCE,
                     "share_of_step": ((ms_c / max(n_c, 1) + ms_y / max(n_y, 1)) / (1000.0 * t_loop / args.steps)
                                       if t_loop else None),
                     "update_step_flops": update_flops,
                     "update_step_frac": update_flops * args.steps / t_loop / 1e12 / FP64_PEAK_TFLOPS},
        "streaming": {"kernel": "predict add (C += C_Q, var += diag_Q, HC += HC_Q), standalone hikf_predict; "
                                "fused into the K-GEMM epilogue in the chained loop", "bound": "hbm",
                      "achieved": bytes_p / t_p / 1e9 if t_p else None, "peak": hbm, "unit": "GB/s",
                      "frac": (bytes_p / t_p / 1e9) / hbm if t_p else None, "peak_source": hbm_src},
        "stage_ms_per_step": {k: v[0] / max(v[1], 1) for k, v in stage.items()},
        "e2e": {"value": world * args.steps / t_e2e, "unit": "steps/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * m, "api": "paper_1404_3816_b200.filters.hikf_update(numpy z) + state.mean"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if fac is not None:
        line["factored"] = fac
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=os.cpu_count()):
            # (3D: no reference 3D path; the same oracle update on the 3D config's rays)
            cf = CpuFilter(cfg, H=H, obs=obs) if dim3 else CpuFilter(cfg)
            cf.step()  # first touch of the m x n buffers, BLAS pool
            t_cpu = cf.step()
            del cf
        if t_cpu is not None:
            line["cpu_baseline"] = {
                "value": 1.0 / t_cpu, "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
                "sample": f"one timed full-size predict+update step of the oracle port on the {m} x {n} state "
                          "(after one untimed step), prior Q = I stand-in for C_Q", "host": host_info()}
        try:
            if dim3:
                mn_s, tq = cpu_qht_sample_3d(cfg, H, xy, cols=2 if m <= 300000 else 1)
                line.setdefault("cpu_baseline", {"kind": "port", "cores": os.cpu_count()})["qht"] = {
                    "value": mn_s, "unit": "(m*n)/s", "sample": f"exact direct-sum Q H^T on {2 if m <= 300000 else 1} "
                                                                f"of {n} columns ({tq:.1f} s; no reference 3D path)"}
            else:
                ncol = min(32, n)
                mn_s, tb, tq = cpu_qht_sample(cfg, cols=ncol)
                line["cpu_baseline"]["qht"] = {"value": mn_s, "unit": "(m*n)/s",
                                               "sample": f"oracle bbFMM matmat on {ncol} of {n} H^T columns "
                                                         f"({tq:.1f} s; matmat is column-independent), tree build "
                                                         f"{tb:.1f} s"}
        except MemoryError:
            pass
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
