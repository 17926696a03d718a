"""Compact per-kernel summary of an ncu report (raw page CSV) -> stdout.

usage: python tools/ncu_summary.py report.ncu-rep
"""
import csv
import subprocess
import sys

KEYS = [
    ("time_ms", "gpu__time_duration.sum", 1e-6),
    ("dram_rd_GB", "dram__bytes_read.sum", 1e-9),
    ("dram_wr_GB", "dram__bytes_write.sum", 1e-9),
    ("dmma_pct", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
    ("fp64_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("fp64_cyc_pct", "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("l2_GB", "lts__t_bytes.sum", 1e-9),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("smem_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
]


def scale(v, f):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * f


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")[-70:]
        print(f"== {short}  grid={r[idx.get('Grid Size', 0)]} block={r[idx.get('Block Size', 0)]}")
        parts = []
        for label, key, f in KEYS:
            if key in idx:
                # ncu reports time in its own unit; normalise by the unit row
                v = r[idx[key]]
                u = units[idx[key]]
                x = scale(v, 1)
                if isinstance(x, float):
                    if u == "ns":
                        x *= 1e-6
                    elif u == "us":
                        x *= 1e-3
                    elif u == "ms":
                        x *= 1
                    elif u == "Kbyte":
                        x *= 1e-6
                    elif u == "Mbyte":
                        x *= 1e-3
                    elif u == "Gbyte":
                        x *= 1
                    elif u == "Tbyte":
                        x *= 1e3
                    elif u == "byte":
                        x *= 1e-9
                    parts.append(f"{label}={x:.4g}")
                else:
                    parts.append(f"{label}={v}")
        print("   " + " ".join(parts))
        stalls = []
        for h, i in idx.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            print("   stalls: " + ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
