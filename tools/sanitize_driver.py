#!/usr/bin/env python
"""Small run of the driver-layer kernels for compute-sanitizer: run_case on
every pair (error-norm point / jump / reduce kernels, device transpose, the
bulk K4a kernel on a small set), lu_factor beyond the patch kernels.

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import mg
    mg.COARSE_CELLS_PER_SIDE = 3
    for case, k in (("th-tri", 2), ("th-quad", 3), ("bdm", 2), ("rt", 1)):
        rec = V.run_case(V.RunSpec(case, k, nu=2, levels=1, rtol=1e-8))
        print(rec.csv_row())
    a = np.random.default_rng(0).standard_normal((150, 150)) + 150 * np.eye(150)
    x = V.lu_solve(V.lu_factor(a), np.ones(150))
    print("lu_factor 150:", float(np.abs(a @ x - 1).max()))


if __name__ == "__main__":
    main()
