#!/usr/bin/env python
"""K3 probe: wall time of the batched patch factorization (extraction + guard
+ explicit inverse) on the finest level of each BASELINE config, first call
(allocations, schedule) and re-factor (median of --reps), with the LU-equivalent
GFLOP/s and the fraction of the measured FP64 peak.  ncu-friendly
(-k regex:factor_tile).

    python tools/factor_probe.py [cfg2 ...] [--reps 5] [--json out]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
FP64_PEAK_TFLOPS = 36.5   # profiles/r1_fp64_peak.json (DFMA microbenchmark on this B200)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.pack import read_pack

    out = {}
    for name in args.names:
        pack = read_pack(os.path.join(ROOT, "data", f"{name}_pack.npz"))
        lv = pack.fine
        ps = V.build_patches(lv.mixed, lv.system.bc)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        V.factor_patches(ps, lv.system)
        torch.cuda.synchronize()
        first = time.perf_counter() - t0
        ts = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            V.factor_patches(ps, lv.system)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = statistics.median(ts)
        sz = np.diff(ps.export()["offsets"]).astype(np.float64)
        lu = (2.0 / 3.0) * float((sz ** 3).sum())
        rec = {"J": int(ps.num_patches), "smax": int(sz.max()), "first_s": first, "refactor_ms": t * 1e3,
               "lu_equiv_gflops": lu / 1e9, "lu_equiv_tflops_per_s": lu / t / 1e12,
               "frac_fp64_peak": lu / t / 1e12 / FP64_PEAK_TFLOPS,
               "gj_issued_frac_fp64_peak": 3.0 * lu / t / 1e12 / FP64_PEAK_TFLOPS}
        out[name] = rec
        print(name, json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in rec.items()}),
              flush=True)
        del ps
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
