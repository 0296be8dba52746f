#!/usr/bin/env python
"""cProfile of the device build_hierarchy of one BASELINE config (host-side
hot spots of the setup): python tools/setup_profile.py cfg5"""
import cProfile
import os
import pstats
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
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    case, k, refs = SPEC[name]
    mg.COARSE_CELLS_PER_SIDE = 16
    A.build_hierarchy(case, k, 1, nu=2, damping=0.5)          # warm-up (module loads)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    A.build_hierarchy(case, k, refs, nu=2, damping=0.5)
    torch.cuda.synchronize()
    pr.disable()
    print(f"{name}: build_hierarchy {time.perf_counter() - t0:.3f} s")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(28)


if __name__ == "__main__":
    main()
