#!/usr/bin/env python
"""One config's V-cycle for profiling: build the hierarchy, warm up, then
replay the captured V-cycle graph a few times (run under ncu for the
per-kernel launch list; plain run prints the graph time)."""
import os
import statistics
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def main():
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.pack import read_pack
    from paper_2409_14222_b200.solver import mg_rhs
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    pack = read_pack(os.path.join(os.path.dirname(HERE), "data", f"{name}_pack.npz"))
    hier = V.hierarchy_from_pack(pack)
    b = torch.from_numpy(mg_rhs(pack)).cuda()
    for _ in range(3):
        hier.vcycle_device(b)
    torch.cuda.synchronize()
    ts = []
    # under `ncu --profile-from-start off` only the timed replays are captured
    torch.cuda.profiler.start()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hier.vcycle_device(b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    torch.cuda.profiler.stop()
    print(f"{name}: V-cycle graph {statistics.median(ts):.3f} ms; levels "
          f"{[lv.n for lv in hier.levels]}")


if __name__ == "__main__":
    main()
