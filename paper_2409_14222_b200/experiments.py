"""Experiment-driver layer over the device path: the callers of the hot path
in the reference's ``bench`` module (``stokesmg/bench.py``; this module is its
drop-in), with the same names, arguments, CSV output and error behaviour.

* :class:`RunSpec` / :class:`RunRecord` (``bench.py:34-92``), :func:`expand_grid`
  (``bench.py:304-327``);
* :func:`error_norms` (``bench.py:95-164``) — relative broken-H1 velocity
  error, mean-free pressure L2 error, largest pointwise divergence and the
  tangential-jump seminorm against the manufactured solution, evaluated per
  quadrature point and reduced on the device (``vk_error_cells`` /
  ``vk_error_jump`` / ``vk_error_reduce``);
* :func:`run_case` (``bench.py:174-191``): device ``build_hierarchy`` (timed
  as setup), then MG-preconditioned FGMRES on the manufactured right-hand
  side (timed as solve, device-synchronised on both sides), then the norms;
* :func:`sweep` (``bench.py:194-214``) and :func:`stopping_study`
  (``bench.py:239-301``).

Everything numerical runs in ``libvanka_b200.so``; there is no CPU path.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from . import fem
from .assembly import ProblemConfig, _dev, build_hierarchy, facet_tables
from .mg import MgHierarchy, make_preconditioner, pressure_kernel
from .sparsela import fgmres, nullspace_projector, to_device

CSV_COLUMNS = ("case,k,nu,levels,n_dofs,m_dofs,alpha,viscosity,rtol,"
               "iterations,converged,setup_s,solve_s,err_h1_vel_rel,"
               "err_l2_p_abs,max_div,jump_seminorm")
STOPPING_COLUMNS = ("case,k,levels,required_rtol,err_h1_vel_rel,"
                    "err_l2_p_abs,resolved")

HDIV_CASES = ("bdm", "rt")
# admissible orders per discretisation family (bench.py:47-55)
_FAMILIES = {"th-tri": ((2, 8), "continuous"), "th-quad": ((2, 8), "continuous"),
             "bdm": ((1, 4), "normal-continuity"), "rt": ((1, 4), "normal-continuity")}


@dataclass
class RunSpec:
    """Reference ``RunSpec`` (``bench.py:34-65``)."""
    case: str
    k: int
    nu: int = 2
    levels: int = 1
    rtol: float = 1e-10
    max_it: int = 100
    alpha: float | None = None
    viscosity: float = 1.0
    seed: int = 0
    weighting: str = "invmult"
    cheby: str = "repeat"

    def validate(self) -> None:
        family = _FAMILIES.get(self.case)
        if family is None:
            raise ValueError(f"unknown case {self.case!r}")
        (lo, hi), label = family
        checks = ((lo <= self.k <= hi, f"{label} pairs support orders {lo}..{hi}"),
                  (0 <= self.levels <= 5, "supported refinement counts are 0..5"),
                  (1 <= self.nu <= 4, "supported relaxation counts are 1..4"),
                  (self.rtol > 0 and self.max_it >= 1,
                   "need a positive tolerance and iteration cap"))
        for ok, message in checks:
            if not ok:
                raise ValueError(message)

    def config(self) -> ProblemConfig:
        return ProblemConfig(self.case, self.k, self.viscosity, self.alpha)


@dataclass
class RunRecord:
    """Reference ``RunRecord`` (``bench.py:68-92``), same CSV row."""
    spec: RunSpec
    n_dofs: int
    m_dofs: int
    iterations: int
    converged: bool
    setup_s: float
    solve_s: float
    err_h1_vel_rel: float
    err_l2_p_abs: float
    max_div: float
    jump_seminorm: float

    def csv_row(self) -> str:
        s = self.spec
        alpha = s.config().penalty if s.case in HDIV_CASES else 0.0
        fields = [s.case, s.k, s.nu, s.levels, self.n_dofs, self.m_dofs, f"{alpha:.6g}",
                  f"{s.viscosity:.6g}", f"{s.rtol:.6g}", self.iterations,
                  str(self.converged).lower(), f"{self.setup_s:.3f}", f"{self.solve_s:.3f}"]
        fields += [f"{v:.12e}" for v in (self.err_h1_vel_rel, self.err_l2_p_abs, self.max_div,
                                         self.jump_seminorm)]
        return ",".join(str(f) for f in fields)


_TABLES: dict = {}


def _error_tables(mixed: fem.Mixed, degree: int):
    """Device-resident reference tabulation and DoF maps of one space for the
    error kernels (cached per space object and quadrature degree)."""
    key = (id(mixed), degree)
    hit = _TABLES.get(key)
    if hit is not None and hit[0] is mixed:
        return hit[1]
    vel, pres = mixed.velocity, mixed.pressure
    topo, geom = vel.mesh
    rule = fem.quadrature(topo.cell_shape, degree)
    rv, rg = vel.element.tabulate(rule.points)
    pv, _ = pres.element.tabulate(rule.points)
    t = {"nq": len(rule.weights),
         "cells": [_dev(a, np.float64) for a in (rule.weights, rule.points, rv, rg, pv,
                                                 geom.vertex_coords[geom.cell_map_vertices])],
         "maps": [_dev(vel.cell_dofs, np.int32), _dev(vel.cell_dof_scale, np.float64),
                  _dev(pres.cell_dofs, np.int32), _dev(pres.cell_dof_scale, np.float64)]}
    if mixed.case in HDIV_CASES:
        info, geo, erule, tabs_v, _ = facet_tables(vel)
        t["facets"] = (len(info), len(erule.weights),
                       [_dev(erule.weights, np.float64), _dev(np.stack(tabs_v), np.float64),
                        _dev(info, np.int32), _dev(geo, np.float64)])
    _TABLES.clear()                      # one space at a time (tables are O(cells))
    _TABLES[key] = (mixed, t)
    return t


def error_norms(solution, mixed: fem.Mixed, viscosity: float = 1.0,
                quad_degree: int | None = None) -> tuple:
    """(relative H1 velocity error, absolute L2 pressure error after mean
    removal, max pointwise divergence, tangential-jump seminorm) — reference
    ``error_norms`` (``bench.py:95-164``); ``solution`` numpy or a CUDA vector."""
    import torch
    L.require_cuda()
    x, _ = to_device(solution)
    if x.numel() != mixed.ndof:
        raise ValueError("solution length does not match the space")
    vel, pres = mixed.velocity, mixed.pressure
    topo, _ = vel.mesh
    k = mixed.order
    degree = quad_degree if quad_degree is not None else min(2 * k + 4, fem.MAX_QUAD_DEGREE)
    t = _error_tables(mixed, degree)
    nc, nq = topo.num_cells, t["nq"]
    st = L.stream_ptr()
    work = torch.empty(5 * nc * nq, dtype=torch.float64, device="cuda")
    L.call("vk_error_cells", nc, nq, vel.element.ndof, pres.element.ndof,
           int(topo.cell_shape == "quad"), int(vel.element.mapping == "piola"),
           *[L.ptr(a) for a in t["cells"]], *[L.ptr(a) for a in t["maps"]], mixed.offset,
           L.ptr(x), L.ptr(work), st)
    neq, jump = 0, None
    if "facets" in t:
        ne, neq_pts, fk = t["facets"]
        neq = ne * neq_pts
        if neq:
            jump = torch.empty(neq, dtype=torch.float64, device="cuda")
            L.call("vk_error_jump", ne, neq_pts, vel.element.ndof, L.ptr(fk[0]), L.ptr(fk[1]),
                   L.ptr(fk[2]), L.ptr(fk[3]), L.ptr(t["cells"][5]), L.ptr(t["maps"][0]),
                   L.ptr(t["maps"][1]), L.ptr(x), L.ptr(jump), st)
    out = torch.empty(6, dtype=torch.float64, device="cuda")
    L.call("vk_error_reduce", nc * nq, L.ptr(work), neq, L.ptr(jump) if jump is not None else None,
           L.ptr(out), st)
    e2, b2, max_div, p2, j2, _mean = out.cpu().tolist()
    return (float(np.sqrt(e2 / b2)), float(np.sqrt(p2)), float(max_div),
            float(np.sqrt(2.0 * viscosity * j2)))


def build_solver(spec: RunSpec) -> MgHierarchy:
    """Reference ``build_solver`` (``bench.py:167-171``), built on the device."""
    spec.validate()
    return build_hierarchy(spec.case, spec.k, spec.levels, spec.config(), nu=spec.nu,
                           weighting=spec.weighting, cheb_mode=spec.cheby, seed=spec.seed)


def _sync():
    import torch
    torch.cuda.synchronize()


def run_case(spec: RunSpec, hierarchy: MgHierarchy | None = None) -> RunRecord:
    """Build (or reuse) the solver, run it, and measure errors (reference
    ``run_case``, ``bench.py:174-191``); setup and solve are wall times with
    the device synchronised at both ends."""
    spec.validate()
    _sync()
    t0 = time.perf_counter()
    hier = hierarchy if hierarchy is not None else build_solver(spec)
    _sync()
    setup_s = time.perf_counter() - t0
    system = hier.fine.system
    nsp = nullspace_projector([pressure_kernel(hier.fine.mixed)])
    t0 = time.perf_counter()
    x, report = fgmres(system.matrix, system.rhs,
                       preconditioner=make_preconditioner(hier, spec.nu, spec.cheby),
                       rtol=spec.rtol, max_it=spec.max_it, nullspace=nsp)
    _sync()
    solve_s = time.perf_counter() - t0
    verr, perr, max_div, jump = error_norms(x, hier.fine.mixed, spec.viscosity)
    return RunRecord(spec, system.num_velocity, system.num_pressure, report.iterations,
                     report.converged, setup_s, solve_s, verr, perr, max_div, jump)


def sweep(specs, out) -> list:
    """Run a grid of specs, streaming one CSV row per completed run; specs that
    differ only in nu / rtol / cheby share one hierarchy, whose build time is
    charged to the first of them (reference ``sweep``, ``bench.py:194-214``)."""
    print(CSV_COLUMNS, file=out, flush=True)
    built: dict = {}
    records = []
    for spec in specs:
        spec.validate()
        key = (spec.case, spec.k, spec.levels, spec.alpha, spec.viscosity, spec.weighting,
               spec.seed)
        first_use = key not in built
        if first_use:
            _sync()
            t0 = time.perf_counter()
            hier = build_solver(spec)
            _sync()
            built[key] = (hier, time.perf_counter() - t0)
        record = run_case(spec, built[key][0])
        record.setup_s = built[key][1] if first_use else 0.0
        records.append(record)
        print(record.csv_row(), file=out, flush=True)
    return records


@dataclass
class StoppingRow:
    case: str
    k: int
    levels: int
    required_rtol: float
    err_h1_vel_rel: float
    err_l2_p_abs: float
    resolved: bool

    def csv_row(self) -> str:
        return ",".join([self.case, str(self.k), str(self.levels), f"{self.required_rtol:.6g}",
                         f"{self.err_h1_vel_rel:.12e}", f"{self.err_l2_p_abs:.12e}",
                         str(self.resolved).lower()])


def _close(a: float, b: float, rel: float = 0.01) -> bool:
    return abs(a - b) <= rel * abs(b) + 1e-16


def _plateau(errs):
    """First tolerance index whose (velocity, pressure) errors agree within 1%
    with those two halvings (rtol / 4) and four halvings (rtol / 16) further
    down (``bench.py:279-288``); None while there is none."""
    def same(i, j):
        return all(_close(errs[i][c], errs[j][c]) for c in (0, 1))
    return next((i for i in range(len(errs) - 4) if same(i, i + 2) and same(i, i + 4)), None)


def stopping_study(case: str, k: int, max_levels: int, *, nu: int = 1, seed: int = 0, out=None,
                   min_rtol: float = 1e-15, max_it_per_leg: int = 300) -> list:
    """Loosest relative tolerance that already delivers discretisation error
    (reference ``stopping_study``, ``bench.py:239-301``): per refinement count
    the same system is solved to 1e-2, 1e-2 / 2, 1e-2 / 4, ... continuing from
    the previous iterate against the fixed baseline ||P b||, measuring the
    errors after every leg, until :func:`_plateau` accepts a tolerance or the
    ladder passes ``min_rtol`` (row reported unresolved)."""
    import torch
    if case not in ("th-quad", "bdm"):
        raise ValueError("the stopping study covers th-quad and bdm only")
    if out is not None:
        print(STOPPING_COLUMNS, file=out, flush=True)
    rows = []
    for levels in range(1, max_levels + 1):
        spec = RunSpec(case, k, nu=nu, levels=levels, seed=seed)
        hier = build_solver(spec)
        system, mixed = hier.fine.system, hier.fine.mixed
        nsp = nullspace_projector([pressure_kernel(mixed)])
        prec = make_preconditioner(hier, nu, spec.cheby)
        base = float(torch.linalg.vector_norm(nsp(system.rhs.clone())).item())
        ladder, errs, x, hit = [], [], None, None
        rtol = 1e-2
        while hit is None and rtol >= min_rtol:
            x, _ = fgmres(system.matrix, system.rhs, preconditioner=prec, rtol=rtol,
                          max_it=max_it_per_leg, nullspace=nsp, x0=x, target_norm=base)
            ladder.append(rtol)
            errs.append(error_norms(x, mixed, spec.viscosity)[:2])
            hit = _plateau(errs)
            rtol = 1e-2 * 0.5 ** len(ladder)
        at = hit if hit is not None else -1
        row = StoppingRow(case, k, levels, ladder[at] if hit is not None else min_rtol,
                          errs[at][0], errs[at][1], hit is not None)
        rows.append(row)
        if out is not None:
            print(row.csv_row(), file=out, flush=True)
    return rows


def expand_grid(table: dict) -> list:
    """RunSpecs from a flat config table: ``k``, ``nu`` and ``levels`` may be
    scalars or lists and are expanded as a product (k outermost), the other
    RunSpec fields are passed through (reference ``expand_grid``,
    ``bench.py:304-327``)."""
    import itertools
    fixed = {f: table[f] for f in ("case", "rtol", "max_it", "alpha", "viscosity", "seed",
                                   "weighting", "cheby") if f in table}
    axes = []
    for name in ("k", "nu", "levels"):
        val = table.get(name)
        if val is None:
            axes.append([()])
        else:
            axes.append([((name, v),) for v in (val if isinstance(val, (list, tuple)) else [val])])
    return [RunSpec(**fixed, **dict(sum(combo, ()))) for combo in itertools.product(*axes)]
