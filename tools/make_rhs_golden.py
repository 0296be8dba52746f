#!/usr/bin/env python
"""Golden right-hand sides from the unmodified reference (imported from
/root/reference in the build container): for every small parity case of
tools/make_packs.py, the finest level's ``assembly.assemble`` rhs
(manufactured forcing load + Dirichlet lift, assembly.py:136-172, 273-285)
and the strong-BC values (spaces.py:203-220).

    python tools/make_rhs_golden.py          # -> tests/golden/rhs_golden.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

CASES = ["cfg1", "s_thtri2", "s_thtri4", "s_thquad3", "s_bdm3", "s_rt2", "s_thquad2",
         "t_thquad3_5", "t_bdm1_5", "t_rt1_5", "t_thtri3_3", "t_bdm2_3"]


def main():
    import make_packs as M
    M._ref()
    from stokesmg.assembly import ProblemConfig, assemble
    from stokesmg.meshtopo import build_structured_quad, build_structured_tri
    from stokesmg.spaces import build_mixed
    out = {}
    for name in CASES:
        case, k, n0, refs = M.CASES[name]
        n = n0 * 2 ** (refs or 0)
        mesh = (build_structured_quad if case == "th-quad" else build_structured_tri)(n)
        system = assemble(build_mixed(case, mesh, k), ProblemConfig(case, k))
        out[f"{name}_rhs"] = system.rhs
        out[f"{name}_bc_indices"] = system.bc.indices.astype(np.int64)
        out[f"{name}_bc_values"] = system.bc.values
        out[f"{name}_spec"] = np.array([n, k])
        print(name, case, k, n, system.rhs.shape[0], flush=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "rhs_golden.npz"), **out)


if __name__ == "__main__":
    main()
