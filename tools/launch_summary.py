#!/usr/bin/env python
"""Per-kernel share of an ncu `--metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_summary.py gpurun_out/launches.csv [--title ...] > profiles/x.txt
"""

import argparse
import collections
import csv

UNIT = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, mi, ui, vi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        us = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    if args.title:
        print(args.title)
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:8d} {t:12.1f} {t / n:10.2f} {100 * t / tot:6.1f}%")
    print(f"{'TOTAL':60s} {sum(v[0] for v in agg.values()):8d} {tot:12.1f}")


if __name__ == "__main__":
    main()
