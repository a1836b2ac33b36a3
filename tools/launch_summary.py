"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list by
kernel name (share of total time, launch count, average duration).

    python tools/launch_summary.py profiles/r01_launches_bench_n1.csv
"""
import csv
import sys
from collections import defaultdict


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    k, m, v, u = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = defaultdict(list)
    for r in rows[1:]:
        if r[m] == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(r[u], 1e-3)
            agg[r[k]].append(float(r[v].replace(",", "")) * scale)
    total = sum(sum(x) for x in agg.values())
    for name, xs in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{100 * sum(xs) / total:5.1f}%  n={len(xs):4d}  avg={sum(xs) / len(xs):9.2f} us  {name[:90]}")


if __name__ == "__main__":
    main()
