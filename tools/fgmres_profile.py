#!/usr/bin/env python
"""Host-side timing of the MG-FGMRES(30) loop per Arnoldi iteration: the
graph-launch call, the wait for the Hessenberg column (device time of the
step + D2H), and the host Givens update — to see how much of the TTS is the
host round trip.

    python tools/fgmres_profile.py [cfg2 ...]
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    names = sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import sparsela as S
    from paper_2409_14222_b200.pack import read_pack
    from paper_2409_14222_b200.solver import FgmresSolver, mg_rhs
    for name in names:
        pack = read_pack(os.path.join(ROOT, "data", f"{name}_pack.npz"))
        hier = V.hierarchy_from_pack(pack)
        b = torch.from_numpy(mg_rhs(pack)).cuda()
        solver = FgmresSolver(hier)
        solver.solve(b)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        hier.vcycle_device(b)
        ev1.record()
        torch.cuda.synchronize()
        vc = ev0.elapsed_time(ev1)
        solver.solve(b)          # first replay of each step graph uploads it
        torch.cuda.synchronize()
        S.FGMRES_PROFILE = {}
        t0 = time.perf_counter()
        _, its, conv, hist = solver.solve(b)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        prof, S.FGMRES_PROFILE = S.FGMRES_PROFILE, None
        rec = {"iterations": its, "wall_ms": wall * 1e3, "vcycle_ms": vc,
               "per_it_ms": wall * 1e3 / its,
               "launch_ms_mean": statistics.mean(prof["launch_s"]) * 1e3,
               "sync_ms_mean": statistics.mean(prof["sync_s"]) * 1e3,
               "host_ms_mean": statistics.mean(prof["host_s"]) * 1e3}
        print(name, json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in rec.items()}),
              flush=True)
        del hier, solver
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
