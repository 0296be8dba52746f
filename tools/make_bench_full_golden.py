"""run_case of the unmodified reference at a BASELINE-size configuration
(coarse 16^2, 3 refinements -> 128^2, reference-default Chebyshev bounds):
-> tests/golden/bench_full_golden.json.  CPU, several minutes per spec.

    python tools/make_bench_full_golden.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")

SPECS = [("th-quad", 3, 3, 2, 1e-8), ("bdm", 2, 3, 2, 1e-8)]


def main():
    from threadpoolctl import threadpool_limits
    import stokesmg as sm
    import stokesmg.mg as mg
    mg.COARSE_CELLS_PER_SIDE = 16
    out = {"coarse": 16, "runs": []}
    with threadpool_limits(1):
        for case, k, levels, nu, rtol in SPECS:
            t0 = time.perf_counter()
            rec = sm.run_case(sm.RunSpec(case, k, nu=nu, levels=levels, rtol=rtol))
            out["runs"].append({"case": case, "k": k, "levels": levels, "nu": nu, "rtol": rtol,
                                "n_dofs": rec.n_dofs, "m_dofs": rec.m_dofs,
                                "iterations": rec.iterations, "converged": bool(rec.converged),
                                "setup_s": rec.setup_s, "solve_s": rec.solve_s,
                                "err_h1_vel_rel": float(rec.err_h1_vel_rel),
                                "err_l2_p_abs": float(rec.err_l2_p_abs),
                                "max_div": float(rec.max_div),
                                "jump_seminorm": float(rec.jump_seminorm),
                                "csv_row": rec.csv_row(),
                                "wall_s": time.perf_counter() - t0})
            print(out["runs"][-1], flush=True)
            with open(os.path.join(ROOT, "tests", "golden", "bench_full_golden.json"), "w") as fh:
                json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
