#!/usr/bin/env python
"""Summarise an ncu report (details + raw pages) per kernel.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--grep REGEX] [--json out.json]
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "lts__t_bytes.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]


def _ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")], "id": r[hdr.index("ID")]}
        for m in RAW:
            if m in hdr:
                d[m] = r[hdr.index(m)] + " " + units[hdr.index(m)]
        out.append(d)
    return out


def details(rep, pattern):
    rows = list(csv.reader(io.StringIO(_ncu(["-i", rep, "--page", "details", "--csv"]))))
    hdr = rows[0]
    ki, si, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Section Name", "Metric Name",
                                                 "Metric Unit", "Metric Value"))
    idi = hdr.index("ID")
    out = {}
    for r in rows[1:]:
        if pattern and not re.search(pattern, r[mi] + " " + r[si]):
            continue
        out.setdefault((r[idi], r[ki][:60]), []).append((r[si], r[mi], r[vi], r[ui]))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--grep", default="Duration|Throughput|Occupancy|Registers|Warp Cycles|"
                                       "Eligible|Bytes|Hit Rate|Stall|Active Warps")
    ap.add_argument("--json")
    args = ap.parse_args()
    r = raw(args.rep)
    for d in r:
        print(json.dumps(d))
    for (kid, k), items in details(args.rep, args.grep).items():
        print(f"== {kid} {k}")
        for s, m, v, u in items:
            print(f"   [{s}] {m}: {v} {u}")
    if args.json:
        json.dump(r, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
