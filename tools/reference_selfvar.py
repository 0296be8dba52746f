#!/usr/bin/env python
"""Reference self-reproducibility of the MG-FGMRES histories.

Runs the CPU oracle — bit-identical to the reference (tests/test_oracle.py) —
with ONE change: the coarse LU (reference mg.py:232, LAPACK getrf) is
factored with 8 OpenBLAS threads instead of 1.  Both factorizations are
equally valid; the resulting per-entry history difference is the floor below
which no independent implementation can be expected to agree with the
reference.  Writes tests/golden/reference_selfvar.json.

    python tools/reference_selfvar.py [names...]      # default: all MG cases
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "reference_selfvar.json")
NAMES = ["s_thtri2", "s_thtri4", "s_thquad3", "s_thquad2", "s_bdm3", "s_rt2",
         "cfg2", "cfg3", "cfg4", "cfg5"]


def run(name):
    from threadpoolctl import threadpool_limits
    from oracle import vanka_oracle as O
    from paper_2409_14222_b200.pack import read_pack
    d = "tests/golden" if name.startswith("s_") else "data"
    pack = read_pack(os.path.join(ROOT, d, f"{name}_pack.npz"))
    href = np.array(json.load(open(os.path.join(ROOT, "tests", "golden",
                                                f"{name}_history.json")))["history"])
    t0 = time.time()
    with threadpool_limits(1):
        h = O.build_hierarchy(pack)
    c = pack.levels[0]
    q = O.pressure_kernel(c.mixed)
    m = c.system.matrix.toarray() + np.abs(c.system.matrix.data).max() * np.outer(q, q)
    with threadpool_limits(8):
        h.coarse_factor = O.lu_factor(m)
    with threadpool_limits(1):
        b = O.mg_rhs(pack)
        nsp = O.NullspaceProjector([O.pressure_kernel(pack.fine.mixed)])
        _, its, conv, hist = O.solve_fgmres30(pack.fine.system.matrix, b,
                                              lambda v: O.v_cycle(h, v), nsp)
    k = min(len(hist), len(href))
    rel = float(np.max(np.abs(hist[:k] - href[:k]) / href[:k]))
    return name, {"history_max_rel": rel, "iterations": its, "seconds": time.time() - t0}


def main(names):
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    os.environ.setdefault("OMP_NUM_THREADS", "8")
    with ProcessPoolExecutor(max_workers=min(4, len(names))) as ex:
        for name, r in ex.map(run, names):
            res[name] = r
            print(name, r, flush=True)
    res["_recipe"] = ("oracle (== reference) with only the coarse getrf run on 8 OpenBLAS "
                      "threads instead of 1; max_j |h_j - h_ref_j| / h_ref_j")
    json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or NAMES)
