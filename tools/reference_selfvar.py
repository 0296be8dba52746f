#!/usr/bin/env python
"""Reference self-reproducibility of the MG-FGMRES histories.

Runs the CPU oracle — bit-identical to the reference (tests/test_oracle.py) —
with ONE change at a time, always in the coarse solve (reference mg.py:228-232
factors A0 + shift q q^T with LAPACK getrf, mg.py:274-279 applies getrs):

* ``getrf_t2`` / ``getrf_t4`` / ``getrf_t8``: the same getrf on 2 / 4 / 8
  OpenBLAS threads (a different blocking, an equally valid factorization);
* ``getri``: the explicit LAPACK inverse (getrf + getri) applied as a
  matrix-vector product — the shape of the device coarse solve;
* ``exact``: the coarse system solved to full accuracy (iterative refinement
  with extended-precision residuals).

Every variant is as correct as the reference's own coarse solve (they differ
by about cond(A0) * eps).  The per-entry history difference each one causes,
max_j |h_j - h_ref_j| / h_ref_j, is recorded; their maximum is the floor below
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
VARIANTS = ["getrf_t2", "getrf_t4", "getrf_t8", "getri", "exact"]


def _coarse_solver(variant, m, q):
    """x = S(rhs) replacing the reference's getrs with the variant's solve
    (the projections of mg.py:277-279 stay the oracle's)."""
    import scipy.linalg as sl
    from threadpoolctl import threadpool_limits
    from oracle import vanka_oracle as O
    if variant.startswith("getrf_t"):
        with threadpool_limits(int(variant[len("getrf_t"):])):
            fac = O.lu_factor(m)
        return lambda r: O.lu_solve(fac, r)
    with threadpool_limits(1):
        fac = O.lu_factor(m)
    if variant == "getri":
        with threadpool_limits(1):
            inv = sl.inv(m)
        return lambda r: inv @ r
    if variant == "exact":
        ml = m.astype(np.longdouble)

        def solve(r):
            x = O.lu_solve(fac, r)
            for _ in range(3):
                res = (r.astype(np.longdouble) - ml @ x.astype(np.longdouble)).astype(np.float64)
                x = x + O.lu_solve(fac, res)
            return x
        return solve
    raise ValueError(variant)


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
    b = O.mg_rhs(pack)
    nsp = O.NullspaceProjector([O.pressure_kernel(pack.fine.mixed)])
    out = {"variants": {}}
    ref_solve = O.coarse_solve
    try:
        for variant in VARIANTS:
            solve = _coarse_solver(variant, m, q)

            def coarse(hier, rhs, s=solve):            # mg.py:274-279 with S swapped
                qq = hier.coarse_kernel
                r = rhs - qq * (qq @ rhs)
                x = s(r)
                return x - qq * (qq @ x)
            O.coarse_solve = coarse
            with threadpool_limits(1):
                _, its, conv, hist = O.solve_fgmres30(pack.fine.system.matrix, b,
                                                      lambda v: O.v_cycle(h, v), nsp)
            k = min(len(hist), len(href))
            out["variants"][variant] = {
                "history_max_rel": float(np.max(np.abs(hist[:k] - href[:k]) / href[:k])),
                "iterations": its}
    finally:
        O.coarse_solve = ref_solve
    out["history_max_rel"] = max(v["history_max_rel"] for v in out["variants"].values())
    out["seconds"] = time.time() - t0
    return name, out


def main(names):
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    os.environ.setdefault("OMP_NUM_THREADS", "8")
    with ProcessPoolExecutor(max_workers=min(8, len(names))) as ex:
        for name, r in ex.map(run, names):
            res[name] = r
            print(name, json.dumps(r), flush=True)
            json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)
    res["_recipe"] = ("oracle (== reference) with only the coarse solve replaced by another "
                      "valid factorization (getrf on 2/4/8 OpenBLAS threads, the getri "
                      "inverse, an exact solve); per variant max_j |h_j - h_ref_j| / h_ref_j; "
                      "history_max_rel = the max over the variants")
    json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or NAMES)
