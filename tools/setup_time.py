#!/usr/bin/env python
"""Wall time of the device build_hierarchy per BASELINE config (median of 3
after a warm-up build): python tools/setup_time.py [cfg2 ...]"""
import gc
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SPEC = {"cfg2": ("th-tri", 2, 4), "cfg3": ("th-tri", 4, 3), "cfg4": ("th-quad", 3, 3),
        "cfg5": ("bdm", 3, 3)}


def main():
    import torch
    from paper_2409_14222_b200 import assembly as A
    from paper_2409_14222_b200 import mg
    mg.COARSE_CELLS_PER_SIDE = 16
    for name in sys.argv[1:] or list(SPEC):
        case, k, refs = SPEC[name]
        ts = []
        for rep in range(4):
            gc.collect()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = A.build_hierarchy(case, k, refs, nu=2, damping=0.5)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            del h
        print(f"{name} async={os.environ.get('VK_COARSE_ASYNC', '1')} build_hierarchy "
              f"first {ts[0]:.3f} s, then median {statistics.median(ts[1:]):.3f} s {ts[1:]}")


if __name__ == "__main__":
    main()
