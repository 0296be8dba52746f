#!/usr/bin/env python
"""Condense the ncu --page raw CSVs of the K2/K3 captures
(tools/gpu_scripts/ncu_k3.sh) into one text table: duration, issue / FP64
pipe / DRAM utilisation and the leading warp-stall reasons.

    python tools/ncu_k3_summary.py gpurun_out/k3_warp_cfg2.raw.csv ... > profiles/r2b_ncu_k3.txt
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU issue %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
]


def main():
    for path in sys.argv[1:]:
        rows = list(csv.reader(open(path)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        name = d.get("Kernel Name", ("?", ""))[0]
        print(f"== {path.split('/')[-1].replace('.raw.csv', '')}: {name[:110]}")
        for k, label in KEYS:
            if k in d:
                print(f"   {label:24s} {d[k][0]} {d[k][1]}")
        stalls = []
        for h, (v, u) in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), h.split("stalled_")[1]))
                except ValueError:
                    pass
        tot = sum(x for x, _ in stalls) or 1.0
        top = ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(stalls, reverse=True)[:6])
        print(f"   stall samples           {top}")


if __name__ == "__main__":
    main()
