#!/usr/bin/env python
"""Small end-to-end run of every new kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): device assembly + prolongation +
build_hierarchy (incl. the DMMA factorisation class and the coarse LU
inverse), both Chebyshev modes, fused transfer units, one FGMRES solve.

    compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L, mg
    from paper_2409_14222_b200.solver import FgmresSolver
    mg.COARSE_CELLS_PER_SIDE = 2
    for case, k, refs in (("th-tri", 4, 1), ("bdm", 3, 1), ("th-quad", 3, 1)):
        for mode in ("repeat", "degree"):
            hier = V.build_hierarchy(case, k, refs, damping=0.5, cheb_mode=mode)
            n = hier.fine.n
            b = np.random.default_rng(0).uniform(-1, 1, n)
            b[np.asarray(hier.fine.system.bc.indices)] = 0.0
            x, its, conv, hist = FgmresSolver(hier).solve(b)
            t = hier.transfers[-1]
            r = torch.empty(n, dtype=torch.float64, device="cuda")
            xc = torch.zeros(t.P.shape[1], dtype=torch.float64, device="cuda")
            bd = torch.from_numpy(b).cuda()
            xd = torch.zeros_like(bd)
            L.call("vk_residual_restrict", hier.fine.A.handle, L.ptr(bd), L.ptr(xd), L.ptr(r),
                   t.PT.handle, L.ptr(xc), L.stream_ptr())
            L.call("vk_prolong_residual", t.P.handle, L.ptr(xc), L.ptr(xd), hier.fine.A.handle,
                   L.ptr(bd), L.ptr(r), L.stream_ptr())
            torch.cuda.synchronize()
            print(case, k, mode, "its", its, "conv", conv, "smax", hier.fine.patches.max_size,
                  flush=True)


if __name__ == "__main__":
    main()
