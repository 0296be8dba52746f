"""Details of the reference's end-to-end acceptance criteria
(/root/reference/pkg/tests/test_acceptance.py criteria 2-7: iteration counts,
errors, divergences, stopping tolerances), computed by the unmodified
reference -> tests/golden/acceptance_golden.json.  CPU, about ten minutes.
"""
import functools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    from threadpoolctl import threadpool_limits
    from stokesmg.bench import RunSpec, build_solver, run_case, stopping_study

    @functools.lru_cache(maxsize=None)
    def solver(case, k, levels):
        return build_solver(RunSpec(case, k, levels=levels))

    out = {"runs": {}, "stopping": []}

    def solve(case, k, nu, levels, rtol=1e-10, max_it=100):
        key = f"{case},{k},{nu},{levels},{rtol:g},{max_it}"
        if key not in out["runs"]:
            r = run_case(RunSpec(case, k, nu=nu, levels=levels, rtol=rtol, max_it=max_it),
                         solver(case, k, levels))
            out["runs"][key] = {"iterations": r.iterations, "converged": bool(r.converged),
                                "err_h1_vel_rel": r.err_h1_vel_rel, "err_l2_p_abs": r.err_l2_p_abs,
                                "max_div": r.max_div, "jump_seminorm": r.jump_seminorm}
            print(key, out["runs"][key], flush=True)
        return out["runs"][key]

    with threadpool_limits(1):
        for case in ("bdm", "rt"):                                    # criterion 2
            for k in (1, 2, 3):
                for levels in (1, 2):
                    solve(case, k, 2, levels, max_it=200)
        solve("th-tri", 2, 2, 1)
        for case, k in [("th-tri", 2), ("th-quad", 2), ("th-quad", 3), ("bdm", 1), ("bdm", 2)]:
            for lev in (0, 1, 2):                                     # criterion 3
                solve(case, k, 2, lev, rtol=1e-12, max_it=200)
        for case, k in [("bdm", 2), ("th-quad", 3)]:                  # criterion 4
            for lev in (1, 2, 3):
                solve(case, k, 2, lev)
        for case, nu, orders in [("th-quad", 1, (2, 3, 4)), ("bdm", 2, (1, 2, 3))]:
            for k in orders:                                          # criterion 5
                solve(case, k, nu, 2)
        solve("th-tri", 4, 1, 2)                                      # criterion 6
        solve("th-quad", 4, 1, 2)
        rows = stopping_study("bdm", 2, 3)                            # criterion 7
        out["stopping"] = [[r.levels, r.required_rtol, r.err_h1_vel_rel, r.err_l2_p_abs,
                            bool(r.resolved)] for r in rows]
        for r in rows:
            solve("bdm", 2, 1, r.levels, rtol=1e-12, max_it=300)
    with open(os.path.join(ROOT, "tests", "golden", "acceptance_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
