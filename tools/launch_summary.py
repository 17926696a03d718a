"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python tools/launch_summary.py launches.csv [top]
Prints launches, total/avg device time and share of all profiled kernel time.
"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*\)$", "", name)  # drop the parameter list
    return name.replace("hikf::<unnamed>::", "").replace("hikf::", "")


def main(path, top=40):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")) * 1e-6))
    agg = defaultdict(lambda: [0, 0.0])
    for k, t in rows:
        agg[k][0] += 1
        agg[k][1] += t
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total:.3f} ms total kernel time (cold-cache, serialised)")
    print(f"{'share':>6} {'total_ms':>10} {'n':>5} {'avg_ms':>9}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{t / total:6.1%} {t:10.3f} {n:5d} {t / n:9.4f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
