"""Host logic of the experiment-driver layer (reference ``bench.py``
RunSpec / RunRecord / expand_grid): validation errors, grid expansion and the
CSV row format against rows printed by the unmodified reference
(tests/golden/bench_golden.json, tools/make_bench_golden.py)."""

import json
import os

import pytest

from conftest import GOLDEN


def _golden():
    return json.load(open(os.path.join(GOLDEN, "bench_golden.json")))


def test_runspec_validation_messages():
    from paper_2409_14222_b200 import RunSpec
    RunSpec("th-tri", 2).validate()
    RunSpec("rt", 4, nu=4, levels=5).validate()
    bad = [(RunSpec("th-quad", 1), "continuous pairs support orders 2..8"),
           (RunSpec("th-tri", 9), "continuous pairs support orders 2..8"),
           (RunSpec("bdm", 5), "normal-continuity pairs support orders 1..4"),
           (RunSpec("rt", 0), "normal-continuity pairs support orders 1..4"),
           (RunSpec("dg", 2), "unknown case 'dg'"),
           (RunSpec("bdm", 1, levels=6), "supported refinement counts are 0..5"),
           (RunSpec("bdm", 1, nu=0), "supported relaxation counts are 1..4"),
           (RunSpec("bdm", 1, rtol=0.0), "need a positive tolerance and iteration cap"),
           (RunSpec("bdm", 1, max_it=0), "need a positive tolerance and iteration cap")]
    for spec, message in bad:
        with pytest.raises(ValueError) as err:
            spec.validate()
        assert str(err.value) == message


def test_runspec_config_penalty():
    from paper_2409_14222_b200 import RunSpec
    assert RunSpec("bdm", 3).config().penalty == 90.0           # 10 k^2 (assembly.py:31-35)
    assert RunSpec("bdm", 3, alpha=7.5).config().penalty == 7.5
    assert RunSpec("th-tri", 2, viscosity=0.5).config().viscosity == 0.5


def test_expand_grid_order_and_passthrough():
    from paper_2409_14222_b200 import expand_grid
    specs = expand_grid({"case": "th-quad", "k": [2, 3], "nu": [1, 2], "levels": 1, "rtol": 1e-6,
                         "cheby": "degree"})
    assert [(s.k, s.nu, s.levels) for s in specs] == [(2, 1, 1), (2, 2, 1), (3, 1, 1), (3, 2, 1)]
    assert all(s.case == "th-quad" and s.rtol == 1e-6 and s.cheby == "degree" for s in specs)
    one = expand_grid({"case": "bdm", "k": 1})
    assert len(one) == 1 and one[0].nu == 2 and one[0].levels == 1


def test_csv_row_matches_reference_rows():
    from paper_2409_14222_b200 import RunRecord, RunSpec
    from paper_2409_14222_b200 import experiments as E
    g = _golden()
    assert E.CSV_COLUMNS == g["csv_columns"]
    assert E.STOPPING_COLUMNS == g["stopping_columns"]
    for run in g["runs"]:
        ref = run["csv_row"].split(",")
        rec = RunRecord(RunSpec(run["case"], run["k"], nu=run["nu"], levels=run["levels"]),
                        run["n_dofs"], run["m_dofs"], run["iterations"], run["converged"],
                        float(ref[11]), float(ref[12]), run["err_h1_vel_rel"],
                        run["err_l2_p_abs"], run["max_div"], run["jump_seminorm"])
        assert rec.csv_row() == run["csv_row"]


def test_stopping_row_format_and_case_check():
    from paper_2409_14222_b200 import stopping_study
    from paper_2409_14222_b200.experiments import StoppingRow
    g = _golden()
    for study in g["stopping"]:
        lines = study["csv"].strip().split("\n")[1:]
        for line, (levels, rtol, verr, perr, ok) in zip(lines, study["rows"]):
            row = StoppingRow(study["case"], study["k"], levels, rtol, verr, perr, ok)
            assert row.csv_row() == line
    with pytest.raises(ValueError, match="covers th-quad and bdm only"):
        stopping_study("th-tri", 2, 1)


def test_cli_parses_reference_flags():
    """Same subcommands / flags / defaults as the reference front end
    (cli.py:22-64)."""
    from paper_2409_14222_b200.__main__ import _parser
    p = _parser()
    a = p.parse_args("run --case rt --k 2 --out r.csv".split())
    assert (a.nu, a.levels, a.rtol, a.max_it, a.alpha, a.viscosity, a.seed, a.weighting,
            a.cheby) == (2, 1, 1e-10, 100, None, 1.0, 0, "invmult", "repeat")
    a = p.parse_args("run --case bdm --k 3 --max-it 7 --alpha 2.5 --cheby degree --out r.csv"
                     .split())
    assert (a.max_it, a.alpha, a.cheby) == (7, 2.5, "degree")
    a = p.parse_args("stopping --case th-quad --k 2 --max-levels 3 --out s.csv".split())
    assert (a.nu, a.seed, a.max_levels) == (1, 0, 3)
    for bad in ("run --case dg --k 2 --out r.csv", "run --case bdm --out r.csv",
                "stopping --case th-tri --k 2 --max-levels 1 --out s.csv", "sweep --out s.csv"):
        with pytest.raises(SystemExit):
            p.parse_args(bad.split())


def test_reference_public_names_and_manufactured_data():
    """Top-level names of the reference package (stokesmg/__init__.py:15-35)
    that the drop-in mirrors, and the manufactured solution's properties
    (reference tests/test_assembly.py:31-66)."""
    import numpy as np
    import paper_2409_14222_b200 as V
    for name in ("BlockSystem", "ProblemConfig", "assemble", "manufactured_data", "RunRecord",
                 "RunSpec", "error_norms", "run_case", "stopping_study", "sweep", "QuadratureRule",
                 "ReferenceElement", "make_quadrature", "tabulate", "EntityRef", "Mesh",
                 "MeshGeometry", "MeshTopology", "build_structured_quad", "build_structured_tri",
                 "ChebyshevParams", "MgHierarchy", "TransferPair", "build_hierarchy",
                 "build_prolongation", "chebyshev_relax", "make_preconditioner", "v_cycle",
                 "FunctionSpace", "MixedSpace", "StrongBc", "build_mixed", "build_space",
                 "interpolate", "strong_bc", "DenseFactorization", "KrylovReport",
                 "SingularMatrixError", "estimate_lambda_max", "extract_submatrix", "fgmres",
                 "lu_factor", "lu_solve", "nullspace_projector", "spmv", "triple_product", "Patch",
                 "PatchSet", "apply_additive", "build_patches_hdiv_extended",
                 "build_patches_taylor_hood", "factor_patches"):
        assert hasattr(V, name), name
    mesh = V.build_structured_tri(3)
    assert mesh.topology.num_cells == 18 and V.build_structured_quad(3).topology.num_cells == 9
    assert abs(V.make_quadrature("tri", 4).weights.sum() - 0.5) < 1e-15
    data = V.manufactured_data()
    pts = np.random.default_rng(0).random((50, 2))
    g = data.velocity_gradient(pts)
    assert np.allclose(g[:, 0, 0] + g[:, 1, 1], 0.0, atol=1e-14)          # divergence free
    assert np.allclose(0.5 * (g[:, 0, 1] + g[:, 1, 0]), 0.0, atol=1e-14)  # no shear strain
    assert np.allclose(data.velocity(np.array([[0.5, 0.0]])), [[1.0, 0.0]])
    assert np.allclose(V.manufactured_data(3.0).forcing(pts), 3 * data.forcing(pts))
    assert np.allclose(data.forcing(pts), 2 * np.pi ** 2 * data.velocity(pts))
    h = 1e-6
    for d in range(2):
        e = np.zeros(2)
        e[d] = h
        fd = (data.velocity(pts + e) - data.velocity(pts - e)) / (2 * h)
        assert np.allclose(g[:, :, d], fd, atol=1e-8)
