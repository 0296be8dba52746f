"""run_case records of the unmodified reference for the non-default RunSpec
fields (cheby = degree, weighting = unit, alpha, viscosity, seed):
-> tests/golden/bench_variants_golden.json.

    python tools/make_bench_variants_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")

VARIANTS = [
    dict(case="th-tri", k=2, levels=1, nu=2, cheby="degree"),
    dict(case="th-quad", k=3, levels=2, nu=3, cheby="degree"),
    dict(case="bdm", k=1, levels=2, nu=2, cheby="degree"),
    dict(case="rt", k=2, levels=1, nu=2, cheby="degree", weighting="unit"),
    dict(case="th-quad", k=2, levels=2, nu=2, weighting="unit"),
    dict(case="bdm", k=2, levels=1, nu=1, weighting="unit"),
    dict(case="bdm", k=1, levels=1, nu=2, alpha=25.0, viscosity=0.5),
    dict(case="th-tri", k=3, levels=1, nu=2, viscosity=3.0, seed=5, rtol=1e-9, max_it=40),
]


def main():
    from threadpoolctl import threadpool_limits
    import stokesmg as sm
    out = []
    with threadpool_limits(1):
        for kw in VARIANTS:
            rec = sm.run_case(sm.RunSpec(**kw))
            out.append({"spec": kw, "n_dofs": rec.n_dofs, "m_dofs": rec.m_dofs,
                        "iterations": rec.iterations, "converged": bool(rec.converged),
                        "err_h1_vel_rel": float(rec.err_h1_vel_rel),
                        "err_l2_p_abs": float(rec.err_l2_p_abs), "max_div": float(rec.max_div),
                        "jump_seminorm": float(rec.jump_seminorm), "csv_row": rec.csv_row()})
            print(out[-1]["csv_row"], flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "bench_variants_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
