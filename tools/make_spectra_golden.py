#!/usr/bin/env python
"""Golden Chebyshev spectra + MG-FGMRES histories with the reference's OWN
default smoother bounds (build container only: imports the unmodified
reference from /root/reference).

For each small MG case the reference hierarchy is built exactly as
``stokesmg.mg.build_hierarchy(case, k, R, nu=2, cheb_mode=mode,
est_steps=10, seed=0)`` (``mg.py:177-233``): every non-coarse level's
``ChebyshevParams.lam`` comes from ``estimate_lambda_max`` (``sparsela.py:
194-226``) on A * apply_additive with seed ``31 * i`` (``mg.py:214-221``).
Recorded per case: the per-level lam, and the FGMRES(30) residual history /
iterations for the same RHS as ``make_packs.py`` (seeded uniform velocity
load), all with 1 BLAS thread, plus the reference's self-variation floor: the
largest max_j |h_j - h'_j| / h_j over runs that change only the coarse solve
to another valid factorization (the whole run on 8 BLAS threads; getrf on
2/4/8 threads; the getri inverse; an exact solve — cf.
tools/reference_selfvar.py).  The operators
themselves are the committed packs (same assembly).

    python tools/make_spectra_golden.py            # writes tests/golden/*_spectra.json
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

from make_packs import CASES, _ref  # noqa: E402

# (case name, chebyshev mode)
RUNS = [("s_thtri2", "repeat"), ("s_thtri4", "repeat"), ("s_thquad3", "repeat"),
        ("s_thquad2", "repeat"), ("s_bdm3", "repeat"), ("s_rt2", "repeat"),
        ("s_thtri2", "degree"), ("s_bdm3", "degree")]
EST_STEPS = 10
SEED = 0


def run(name, mode):
    _ref()
    import stokesmg.mg as mg
    from stokesmg.sparsela import fgmres, nullspace_projector

    case, k, coarse, refinements = CASES[name]
    mg.COARSE_CELLS_PER_SIDE = coarse
    t0 = time.perf_counter()
    hier = mg.build_hierarchy(case, k, refinements, nu=2, cheb_mode=mode,
                              est_steps=EST_STEPS, seed=SEED)
    t_setup = time.perf_counter() - t0
    lams = [None] + [float(lv.cheb.lam) for lv in hier.levels[1:]]

    fine = hier.fine
    a = fine.system.matrix
    nvel = fine.system.num_velocity
    b = np.zeros(a.shape[0])
    b[:nvel] = np.random.default_rng(0).uniform(-1.0, 1.0, nvel)
    b[fine.system.bc.indices] = 0.0
    nsp = nullspace_projector([mg.pressure_kernel(fine.mixed)])
    prec = mg.make_preconditioner(hier)
    pb = nsp(b.copy())
    x, base, hist, its, conv = None, None, [], 0, False
    for _ in range(20):
        x, rep = fgmres(a, b, preconditioner=prec, rtol=1e-8, max_it=30,
                        nullspace=nsp, x0=x, target_norm=base)
        if base is None:
            base = float(np.linalg.norm(pb))
            hist.extend(rep.history.tolist())
        else:
            hist.extend(rep.history[1:].tolist())
        its += rep.iterations
        if rep.converged:
            conv = True
            break
    rec = {"name": name, "mode": mode, "est_steps": EST_STEPS, "seed": SEED,
           "lam": lams, "iterations": its, "converged": conv, "history": hist,
           "setup_s": t_setup}
    rec["_hier"] = hier
    rec["_solve"] = (a, b, nsp, prec, pb)
    return rec


def coarse_variants(rec):
    """History change when only the reference's coarse solve (mg.py:274-279)
    is replaced by another valid factorization of the same coarse operator
    (cf. tools/reference_selfvar.py): getrf on 2/4/8 BLAS threads, the getri
    inverse, an exact (refined) solve."""
    import scipy.linalg as sl
    from threadpoolctl import threadpool_limits
    import stokesmg.mg as mg
    from stokesmg.sparsela import fgmres, lu_factor, lu_solve
    hier = rec["_hier"]
    a, b, nsp, prec, pb = rec["_solve"]
    c = hier.levels[0]
    q = mg.pressure_kernel(c.mixed)
    m = c.system.matrix.toarray() + np.max(np.abs(c.system.matrix.data)) * np.outer(q, q)
    href = np.asarray(rec["history"])
    with threadpool_limits(1):
        fac1 = lu_factor(m)
        inv = sl.inv(m)
    ml = m.astype(np.longdouble)

    def exact(r):
        x = lu_solve(fac1, r)
        for _ in range(3):
            res = (r.astype(np.longdouble) - ml @ x.astype(np.longdouble)).astype(np.float64)
            x = x + lu_solve(fac1, res)
        return x
    solvers = {}
    for t in (2, 4, 8):
        with threadpool_limits(t):
            f = lu_factor(m)
        solvers[f"getrf_t{t}"] = (lambda r, f=f: lu_solve(f, r))
    solvers["getri"] = lambda r: inv @ r
    solvers["exact"] = exact
    out = {}
    orig = mg.coarse_solve
    try:
        for key, solve in solvers.items():
            def coarse(h, rhs, s=solve):
                r = rhs - q * (q @ rhs)
                x = s(r)
                return x - q * (q @ x)
            mg.coarse_solve = coarse
            x, base, hist = None, None, []
            with threadpool_limits(1):
                for _ in range(20):
                    x, rep = fgmres(a, b, preconditioner=prec, rtol=1e-8, max_it=30,
                                    nullspace=nsp, x0=x, target_norm=base)
                    if base is None:
                        base = float(np.linalg.norm(pb))
                        hist.extend(rep.history.tolist())
                    else:
                        hist.extend(rep.history[1:].tolist())
                    if rep.converged:
                        break
            h = np.asarray(hist)
            k = min(len(h), len(href))
            out[key] = float(np.max(np.abs(h[:k] - href[:k]) / href[:k]))
    finally:
        mg.coarse_solve = orig
    return out


def main():
    from threadpoolctl import threadpool_limits
    out = os.path.join(ROOT, "tests", "golden")
    for name, mode in RUNS:
        with threadpool_limits(1):
            rec = run(name, mode)
        with threadpool_limits(8):
            alt = run(name, mode)
        h, h2 = np.asarray(rec["history"]), np.asarray(alt["history"])
        m = min(len(h), len(h2))
        variants = {"all_t8": float(np.max(np.abs(h[:m] - h2[:m]) / h[:m]))}
        variants.update(coarse_variants(rec))
        rec["selfvar_variants"] = variants
        rec["selfvar_history_max_rel"] = max(variants.values())
        rec["selfvar_iterations"] = alt["iterations"]
        rec.pop("_hier")
        rec.pop("_solve")
        path = os.path.join(out, f"{name}_{mode}_spectra.json")
        with open(path, "w") as fh:
            json.dump(rec, fh, indent=1)
        print(f"{name} {mode}: lam={rec['lam']} its={rec['iterations']} floor={variants}",
              flush=True)


if __name__ == "__main__":
    main()
