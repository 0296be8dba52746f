"""Golden fixtures for the experiment-driver layer (reference ``bench.py``):
``run_case`` records, ``error_norms`` of the reference's own solutions and a
``stopping_study`` table, produced by the unmodified reference.

    python tools/make_bench_golden.py     # -> tests/golden/bench_golden.npz (+ .json)

Needs /root/reference (this container only); the fixtures are committed.
"""

import io
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")

SPECS = [("th-tri", 2, 1, 2), ("th-tri", 3, 1, 1), ("th-quad", 2, 1, 2), ("th-quad", 3, 2, 2),
         ("bdm", 1, 1, 2), ("bdm", 2, 1, 2), ("rt", 1, 1, 2), ("rt", 2, 2, 1)]
STOPPING = [("th-quad", 2, 2), ("bdm", 1, 2)]


def main():
    from threadpoolctl import threadpool_limits
    import stokesmg as sm
    from stokesmg.bench import build_solver
    arrays, meta = {}, {"runs": [], "stopping": []}
    with threadpool_limits(1):
        for case, k, levels, nu in SPECS:
            spec = sm.RunSpec(case, k, nu=nu, levels=levels)
            hier = build_solver(spec)
            rec = sm.run_case(spec, hier)
            system = hier.fine.system
            nsp = sm.nullspace_projector([sm.mg.pressure_kernel(hier.fine.mixed)])
            x, rep = sm.fgmres(system.matrix, system.rhs,
                               preconditioner=sm.make_preconditioner(hier, spec.nu, spec.cheby),
                               rtol=spec.rtol, max_it=spec.max_it, nullspace=nsp)
            name = f"{case}_{k}_{levels}_{nu}"
            arrays[name + "_x"] = x
            # a non-solution vector too: the norms of a seeded perturbation
            y = x + 1e-3 * np.random.default_rng(7).standard_normal(len(x))
            arrays[name + "_y"] = y
            arrays[name + "_norms_x"] = np.array(sm.error_norms(x, hier.fine.mixed))
            arrays[name + "_norms_y"] = np.array(sm.error_norms(y, hier.fine.mixed, 1.0, 2 * k + 1))
            meta["runs"].append({
                "name": name, "case": case, "k": k, "levels": levels, "nu": nu,
                "n_dofs": rec.n_dofs, "m_dofs": rec.m_dofs, "iterations": rec.iterations,
                "converged": bool(rec.converged), "err_h1_vel_rel": rec.err_h1_vel_rel,
                "err_l2_p_abs": rec.err_l2_p_abs, "max_div": rec.max_div,
                "jump_seminorm": rec.jump_seminorm, "csv_row": rec.csv_row(),
                "history": rep.history.tolist()})
            print(name, rec.iterations, rec.err_h1_vel_rel, rec.err_l2_p_abs, rec.max_div,
                  rec.jump_seminorm, flush=True)
        for case, k, max_levels in STOPPING:
            out = io.StringIO()
            rows = sm.stopping_study(case, k, max_levels, out=out)
            meta["stopping"].append({
                "case": case, "k": k, "max_levels": max_levels, "csv": out.getvalue(),
                "rows": [[r.levels, r.required_rtol, r.err_h1_vel_rel, r.err_l2_p_abs,
                          bool(r.resolved)] for r in rows]})
            print(out.getvalue(), flush=True)
    meta["csv_columns"] = sm.bench.CSV_COLUMNS
    meta["stopping_columns"] = sm.bench.STOPPING_COLUMNS
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "bench_golden.npz"), **arrays)
    with open(os.path.join(ROOT, "tests", "golden", "bench_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
