"""Experiment-driver layer on the device against the unmodified reference
(tests/golden/bench_golden.*, tools/make_bench_golden.py): ``error_norms`` of
the reference's own solution vectors, ``run_case`` end to end on device-built
hierarchies (reference-default Chebyshev bounds), ``sweep`` and
``stopping_study``."""

import io
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

REL_NORM = 1e-10         # error_norms of the same vector: summation order only
DIV_NOISE = 1e-9         # H(div) pairs: max |div u_h| is rounding noise (~1e-11)


@pytest.fixture(scope="module")
def golden():
    meta = json.load(open(os.path.join(GOLDEN, "bench_golden.json")))
    return meta, np.load(os.path.join(GOLDEN, "bench_golden.npz"))


def _mixed(case, k, levels):
    from paper_2409_14222_b200 import fem, mg
    shape = "quad" if case == "th-quad" else "tri"
    mesh = fem.structured_mesh(shape, mg.COARSE_CELLS_PER_SIDE * 2 ** levels)
    return fem.build_mixed(case, mesh, k)


def _check_norms(got, ref, hdiv):
    for i in (0, 1, 3):
        assert abs(got[i] - ref[i]) <= REL_NORM * abs(ref[i]) + 1e-300, (i, got, ref)
    # max |div u_h| is a cancelling sum of O(pi) gradient entries: rounding of
    # ~1e-14 absolute on top of the relative gate
    assert abs(got[2] - ref[2]) <= (DIV_NOISE if hdiv else REL_NORM * ref[2] + 1e-12)


RUNS = ["th-tri_2_1_2", "th-tri_3_1_1", "th-quad_2_1_2", "th-quad_3_2_2", "bdm_1_1_2",
        "bdm_2_1_2", "rt_1_1_2", "rt_2_2_1"]


@pytest.mark.parametrize("name", RUNS)
def test_error_norms_of_reference_solutions(name, golden, capsys):
    import torch
    import paper_2409_14222_b200 as V
    meta, arr = golden
    run = next(r for r in meta["runs"] if r["name"] == name)
    mixed = _mixed(run["case"], run["k"], run["levels"])
    hdiv = run["case"] in ("bdm", "rt")
    got = V.error_norms(arr[name + "_x"], mixed)
    _check_norms(got, arr[name + "_norms_x"], hdiv)
    # a perturbed vector, explicit quadrature degree, device input
    y = torch.from_numpy(arr[name + "_y"]).cuda()
    got_y = V.error_norms(y, mixed, 1.0, 2 * run["k"] + 1)
    _check_norms(got_y, arr[name + "_norms_y"], False)
    with capsys.disabled():
        ref = arr[name + "_norms_x"]
        print(f"\n[{name}] error norms rel diff "
              f"{[abs(g - r) / max(abs(r), 1e-300) for g, r in zip(got, ref)]}")
    with pytest.raises(ValueError):
        V.error_norms(arr[name + "_x"][:-1], mixed)


@pytest.mark.parametrize("name", RUNS)
def test_run_case_matches_reference(name, golden, capsys):
    import paper_2409_14222_b200 as V
    meta, _ = golden
    run = next(r for r in meta["runs"] if r["name"] == name)
    spec = V.RunSpec(run["case"], run["k"], nu=run["nu"], levels=run["levels"])
    rec = V.run_case(spec)
    with capsys.disabled():
        print(f"\n[{name}] {rec.csv_row()}\n{' ' * (len(name) + 3)}{run['csv_row']}")
    assert (rec.n_dofs, rec.m_dofs) == (run["n_dofs"], run["m_dofs"])
    assert rec.converged == run["converged"]
    assert abs(rec.iterations - run["iterations"]) <= 1
    for key in ("err_h1_vel_rel", "err_l2_p_abs", "jump_seminorm"):
        assert abs(getattr(rec, key) - run[key]) <= 1e-6 * abs(run[key]) + 1e-300, key
    if run["case"] in ("bdm", "rt"):
        assert rec.max_div <= 1e-9
    else:
        assert abs(rec.max_div - run["max_div"]) <= 1e-6 * run["max_div"]
    # identical leading CSV fields (case .. rtol, iterations when equal)
    assert rec.csv_row().split(",")[:9] == run["csv_row"].split(",")[:9]


def test_sweep_streams_rows_and_reuses_hierarchies():
    import paper_2409_14222_b200 as V
    out = io.StringIO()
    specs = V.expand_grid({"case": "th-quad", "k": 2, "nu": [1, 2], "levels": 1, "rtol": 1e-8})
    recs = V.sweep(specs, out)
    lines = out.getvalue().strip().split("\n")
    assert lines[0] == V.experiments.CSV_COLUMNS and len(lines) == 3
    assert recs[0].setup_s > 0.0 and recs[1].setup_s == 0.0       # one build, first use
    assert all(r.converged for r in recs)
    assert recs[1].iterations <= recs[0].iterations


@pytest.mark.parametrize("idx", [0, 1])
def test_stopping_study_matches_reference(idx, golden, capsys):
    import paper_2409_14222_b200 as V
    meta, _ = golden
    study = meta["stopping"][idx]
    out = io.StringIO()
    rows = V.stopping_study(study["case"], study["k"], study["max_levels"], out=out)
    with capsys.disabled():
        print("\n" + out.getvalue() + study["csv"])
    assert len(rows) == len(study["rows"])
    for row, (levels, rtol, verr, perr, ok) in zip(rows, study["rows"]):
        assert (row.levels, row.resolved) == (levels, ok)
        assert row.required_rtol == rtol
        assert abs(row.err_h1_vel_rel - verr) <= 1e-6 * verr
        assert abs(row.err_l2_p_abs - perr) <= 1e-6 * perr


def test_cli_run_and_sweep(tmp_path, golden, capsys):
    from paper_2409_14222_b200.__main__ import main
    import paper_2409_14222_b200 as V
    meta, _ = golden
    run = next(r for r in meta["runs"] if r["name"] == "bdm_1_1_2")
    out = tmp_path / "run.csv"
    assert main(["run", "--case", "bdm", "--k", "1", "--out", str(out)]) == 0
    header, row = out.read_text().strip().split("\n")
    assert header == V.experiments.CSV_COLUMNS
    assert row.split(",")[:11] == run["csv_row"].split(",")[:11]       # .. iterations, converged
    cfg = tmp_path / "grid.toml"
    cfg.write_text('case = "th-tri"\nk = 2\nnu = [1, 2]\nlevels = 1\nrtol = 1e-8\n')
    out2 = tmp_path / "sweep.csv"
    assert main(["sweep", "--config", str(cfg), "--out", str(out2)]) == 0
    assert len(out2.read_text().strip().split("\n")) == 3
    assert "wrote 2 rows" in capsys.readouterr().out


# ---------------------------------------------------------------------------
# the reference's own tests/test_bench.py, same conditions, on the device
# ---------------------------------------------------------------------------

def _space(case, n, k):
    from paper_2409_14222_b200 import fem
    return fem.build_mixed(case, fem.structured_mesh("quad" if case == "th-quad" else "tri", n), k)


def _interp_solution(mixed):
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.assembly import manufactured_velocity
    x = np.zeros(mixed.ndof)
    x[:mixed.offset] = V.interpolate(mixed.velocity, manufactured_velocity)
    return x


# reference tests/test_bench.py:22-50
def test_error_norm_properties():
    import paper_2409_14222_b200 as V
    errs = []
    for n in (5, 10):
        mixed = _space("th-tri", n, 2)
        verr, _, _, jump = V.error_norms(_interp_solution(mixed), mixed)
        assert verr > 0 and jump == 0.0
        errs.append(verr)
    assert errs[1] < 0.5 * errs[0]
    mixed = _space("th-quad", 3, 2)
    verr, _, _, _ = V.error_norms(np.zeros(mixed.ndof), mixed)
    assert verr == pytest.approx(1.0, abs=1e-12)
    mixed = _space("bdm", 3, 1)
    x = np.random.default_rng(0).standard_normal(mixed.ndof)
    _, p1, _, _ = V.error_norms(x, mixed)
    shifted = x.copy()
    shifted[mixed.offset:] += 7.5
    _, p2, _, _ = V.error_norms(shifted, mixed)
    assert p1 == pytest.approx(p2, rel=1e-10)


# reference tests/test_bench.py:53-66
def test_run_case_properties():
    import paper_2409_14222_b200 as V
    rec = V.run_case(V.RunSpec("th-tri", 2, nu=2, levels=1))
    assert rec.converged and rec.err_h1_vel_rel < 0.05 and rec.max_div > 1e-3
    rec = V.run_case(V.RunSpec("bdm", 2, nu=2, levels=2, rtol=1e-10))
    assert rec.converged and rec.max_div <= 1e-8
    rec = V.run_case(V.RunSpec("th-quad", 2, nu=2, levels=0, rtol=1e-10))
    assert rec.converged and rec.iterations <= 2          # single level: exact preconditioner


# reference tests/test_bench.py:79-102
def test_sweep_deterministic_without_timings():
    import paper_2409_14222_b200 as V
    grid = [V.RunSpec("th-tri", 2, nu=nu, levels=lev, rtol=1e-8) for nu in (1, 2) for lev in (0, 1)]
    outputs = []
    for _ in range(2):
        buf = io.StringIO()
        records = V.sweep(grid, buf)
        lines = buf.getvalue().strip().splitlines()
        assert lines[0] == V.experiments.CSV_COLUMNS and len(lines) == 5 and len(records) == 4
        rows = [line.split(",") for line in lines[1:]]
        for row in rows:
            row[11] = row[12] = "-"                       # wall-clock columns
        outputs.append(rows)
    assert outputs[0] == outputs[1]


# reference tests/test_bench.py:115-160
def test_stopping_plateau_and_cli(tmp_path):
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.__main__ import main
    rows = V.stopping_study("bdm", 1, 1, out=io.StringIO())
    assert len(rows) == 1 and rows[0].resolved and 1e-15 < rows[0].required_rtol <= 1e-2
    tight = V.run_case(V.RunSpec("bdm", 1, nu=1, levels=1, rtol=1e-12, max_it=200))
    assert abs(rows[0].err_h1_vel_rel - tight.err_h1_vel_rel) <= 0.01 * tight.err_h1_vel_rel
    out = tmp_path / "run.csv"
    assert main(["run", "--case", "th-tri", "--k", "2", "--nu", "2", "--levels", "0", "--rtol",
                 "1e-8", "--max-it", "50", "--out", str(out)]) == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == V.experiments.CSV_COLUMNS and lines[1].startswith("th-tri,2,2,0,")
    out = tmp_path / "stop.csv"
    assert main(["stopping", "--case", "bdm", "--k", "1", "--max-levels", "1", "--out",
                 str(out)]) == 0
    lines = out.read_text().strip().splitlines()
    assert len(lines) == 2 and lines[1].startswith("bdm,1,1,")


def _full_runs():
    p = os.path.join(GOLDEN, "bench_full_golden.json")
    return json.load(open(p))["runs"] if os.path.exists(p) else []


@pytest.mark.parametrize("run", _full_runs(), ids=lambda r: f"{r['case']}_{r['k']}_{r['levels']}")
def test_run_case_full_size_matches_reference(run, capsys):
    """run_case at a BASELINE-size configuration (coarse 16^2 refined to 128^2,
    reference-default Chebyshev bounds estimated on the device) against the
    unmodified reference's record (tools/make_bench_full_golden.py)."""
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import mg
    old = mg.COARSE_CELLS_PER_SIDE
    mg.COARSE_CELLS_PER_SIDE = 16
    try:
        rec = V.run_case(V.RunSpec(run["case"], run["k"], nu=run["nu"], levels=run["levels"],
                                   rtol=run["rtol"]))
    finally:
        mg.COARSE_CELLS_PER_SIDE = old
    with capsys.disabled():
        print(f"\n[{run['case']} k={run['k']} 128^2] device   {rec.csv_row()}\n"
              f"{'':22s}reference {run['csv_row']}")
    assert (rec.n_dofs, rec.m_dofs) == (run["n_dofs"], run["m_dofs"])
    assert rec.converged == run["converged"]
    assert abs(rec.iterations - run["iterations"]) <= 1
    for key in ("err_h1_vel_rel", "err_l2_p_abs", "jump_seminorm"):
        assert abs(getattr(rec, key) - run[key]) <= 1e-3 * abs(run[key]) + 1e-300, key
    if run["case"] in ("bdm", "rt"):
        assert rec.max_div <= 1e-8
    else:
        assert abs(rec.max_div - run["max_div"]) <= 1e-3 * run["max_div"]


def _variant_runs():
    p = os.path.join(GOLDEN, "bench_variants_golden.json")
    return json.load(open(p)) if os.path.exists(p) else []


@pytest.mark.parametrize("run", _variant_runs(), ids=lambda r: "-".join(
    f"{k}={v}" for k, v in r["spec"].items() if k not in ("levels", "nu")))
def test_run_case_non_default_fields(run, capsys):
    """cheby = degree, weighting = unit, alpha, viscosity, seed, rtol / max_it:
    every RunSpec field reaches the device path like the reference's."""
    import paper_2409_14222_b200 as V
    rec = V.run_case(V.RunSpec(**run["spec"]))
    with capsys.disabled():
        print(f"\ndevice    {rec.csv_row()}\nreference {run['csv_row']}")
    assert (rec.n_dofs, rec.m_dofs, rec.converged) == (run["n_dofs"], run["m_dofs"],
                                                       run["converged"])
    assert abs(rec.iterations - run["iterations"]) <= 1
    for key in ("err_h1_vel_rel", "err_l2_p_abs", "jump_seminorm"):
        assert abs(getattr(rec, key) - run[key]) <= 1e-5 * abs(run[key]) + 1e-300, key
    assert rec.csv_row().split(",")[:9] == run["csv_row"].split(",")[:9]
