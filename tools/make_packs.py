#!/usr/bin/env python
"""Generate problem packs and reference golden outputs (build container only).

Imports the UNMODIFIED reference from /root/reference/pkg/src (read-only) and
runs the recipe pinned in BASELINE.md §3 / SURVEY.md §8(c):

* meshes ``build_structured_tri/quad``; spaces ``build_mixed``; operators
  ``assemble(mixed, ProblemConfig(case, k))``
* MG: ``stokesmg.mg.COARSE_CELLS_PER_SIDE = coarse``;
  ``build_hierarchy(case, k, R, nu=2, cheb_mode="repeat", est_steps=1)``;
  every non-coarse ``level.cheb`` replaced by lower=1, upper=3 (damp = 0.5)
* RHS: b_u = default_rng(0).uniform(-1, 1, n_vel); b[bc] = 0; b_p = 0
* FGMRES(30): ``fgmres(A, b, preconditioner=make_preconditioner(hier),
  rtol=1e-8, max_it=30, nullspace=P)`` warm-restarted with x0/target_norm.

Outputs
  <dir>/<name>_pack.npz    operators + topology (see paper_2409_14222_b200/pack.py)
  <dir>/<name>_golden.npz  reference outputs (patch lists, blocks sample,
                           relaxed vector, first V-cycle, FGMRES history, x)
Small cases go to tests/golden/ (committed); the full BASELINE configs go to
data/ (git-ignored, shipped to the GPU box by gpurun) with their FGMRES
histories also copied to tests/golden/<name>_history.json (committed).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"

# name: (case, k, coarse cells per side, refinements)  -- refinements None =
# single level (no MG), used for config 1.
CASES = {
    # BASELINE.json configs
    "cfg1": ("th-tri", 2, 32, None),
    "cfg2": ("th-tri", 2, 16, 4),
    "cfg3": ("th-tri", 4, 16, 3),
    "cfg4": ("th-quad", 3, 16, 3),
    "cfg5": ("bdm", 3, 16, 3),
    # small parity cases (committed)
    "s_thtri2": ("th-tri", 2, 4, 2),
    "s_thtri4": ("th-tri", 4, 4, 1),
    "s_thquad3": ("th-quad", 3, 4, 1),
    "s_bdm3": ("bdm", 3, 4, 1),
    "s_rt2": ("rt", 2, 4, 1),
    "s_thquad2": ("th-quad", 2, 3, 2),
    # tiny single-level cases mirroring the reference's own unit tests
    # (tests/test_vanka.py:23-124)
    "t_thtri2_5": ("th-tri", 2, 5, None),
    "t_thtri4_5": ("th-tri", 4, 5, None),
    "t_thquad3_5": ("th-quad", 3, 5, None),
    "t_bdm1_5": ("bdm", 1, 5, None),
    "t_rt1_5": ("rt", 1, 5, None),
    "t_thtri3_3": ("th-tri", 3, 3, None),
    "t_thquad2_3": ("th-quad", 2, 3, None),
    "t_bdm2_3": ("bdm", 2, 3, None),
    "t_rt1_3": ("rt", 1, 3, None),
    "t_thtri2_3": ("th-tri", 2, 3, None),
    "t_thquad3_2": ("th-quad", 3, 2, None),
    "t_bdm1_3": ("bdm", 1, 3, None),
    "t_thquad2_2": ("th-quad", 2, 2, None),
    "t_thtri2_2": ("th-tri", 2, 2, None),
    "t_bdm1_2": ("bdm", 1, 2, None),
}
FULL = ("cfg2", "cfg3", "cfg4", "cfg5")


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import stokesmg  # noqa: F401
    return stokesmg


def patch_arrays(ps) -> dict:
    sizes = np.array([len(p.indices) for p in ps.patches], dtype=np.int64)
    offs = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offs[1:])
    return {
        "patch_offsets": offs,
        "patch_indices": np.concatenate([p.indices for p in ps.patches]).astype(np.int32),
        "patch_nvel": np.array([p.num_velocity for p in ps.patches], dtype=np.int32),
        "patch_weights": np.concatenate([p.weights for p in ps.patches]),
        "patch_entity": np.array([(p.entity.dim, p.entity.index) for p in ps.patches],
                                 dtype=np.int32),
        "multiplicity": ps.multiplicity,
    }


def block_sample(ps, matrix, count=24) -> dict:
    from stokesmg.sparsela import extract_submatrix
    j = ps.num_patches
    pick = np.unique(np.r_[np.arange(min(8, j)), np.linspace(0, j - 1, count).astype(int),
                           np.arange(max(0, j - 8), j)])
    blocks = [extract_submatrix(matrix, ps.patches[i].indices, ps.patches[i].indices).ravel()
              for i in pick]
    return {"block_pick": pick.astype(np.int64), "block_data": np.concatenate(blocks)}


def single_level(name, case, k, n, out_dir):
    sm = _ref()
    from stokesmg.meshtopo import build_structured_quad, build_structured_tri
    from stokesmg.spaces import build_mixed
    from stokesmg.assembly import assemble, ProblemConfig
    from stokesmg.vanka import build_patches, factor_patches, apply_additive
    from paper_2409_14222_b200.pack import write_pack

    mesh = (build_structured_quad if case == "th-quad" else build_structured_tri)(n)
    mixed = build_mixed(case, mesh, k)
    system = assemble(mixed, ProblemConfig(case, k))
    t0 = time.perf_counter()
    ps = build_patches(mixed, system.bc)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    factor_patches(ps, system)
    t_factor = time.perf_counter() - t0
    nn = system.matrix.shape[0]
    r = np.random.default_rng(0).uniform(-1.0, 1.0, nn)
    best = 1e30
    for _ in range(3):
        t0 = time.perf_counter()
        out = apply_additive(ps, r)
        best = min(best, time.perf_counter() - t0)
    x = 0.5 * out
    g = {"r": r, "x_sweep": x, "Ar": system.matrix @ r}
    g.update(patch_arrays(ps))
    g.update(block_sample(ps, system.matrix))
    g["timings"] = np.array([t_build, t_factor, best])
    write_pack(os.path.join(out_dir, f"{name}_pack.npz"), case, k,
               [(mixed, system, None)], {"recipe": "single-level sweep, damping 0.5"})
    np.savez_compressed(os.path.join(out_dir, f"{name}_golden.npz"), **g)
    print(f"{name}: N={nn} nnz={system.matrix.nnz} J={ps.num_patches} "
          f"build={t_build:.2f}s factor={t_factor:.2f}s apply={best*1e3:.1f}ms", flush=True)


def multilevel(name, case, k, coarse, refinements, out_dir, hist_dir):
    sm = _ref()
    import stokesmg.mg as mg
    from stokesmg.sparsela import fgmres, nullspace_projector
    from stokesmg.vanka import apply_additive
    from paper_2409_14222_b200.pack import write_pack

    mg.COARSE_CELLS_PER_SIDE = coarse
    t0 = time.perf_counter()
    hier = mg.build_hierarchy(case, k, refinements, nu=2, cheb_mode="repeat", est_steps=1)
    t_setup = time.perf_counter() - t0
    for lvl in hier.levels[1:]:
        lvl.cheb = SimpleNamespace(lower=1.0, upper=3.0, lam=None)

    levels = []
    for i, lvl in enumerate(hier.levels):
        masked = hier.transfers[i].masked if i > 0 else None
        levels.append((lvl.mixed, lvl.system, masked))
    write_pack(os.path.join(out_dir, f"{name}_pack.npz"), case, k, levels,
               {"coarse": coarse, "refinements": refinements,
                "recipe": "BASELINE.md §3: V(2,2) repeat, damping 0.5, FGMRES(30) rtol 1e-8"})

    fine = hier.fine
    a = fine.system.matrix
    nvel = fine.system.num_velocity
    nn = a.shape[0]
    b = np.zeros(nn)
    b[:nvel] = np.random.default_rng(0).uniform(-1.0, 1.0, nvel)
    b[fine.system.bc.indices] = 0.0
    nsp = nullspace_projector([mg.pressure_kernel(fine.mixed)])
    prec = mg.make_preconditioner(hier)

    g = {"b": b}
    # single fine-level sweep on a seeded residual (config-1 style check)
    r = np.random.default_rng(1).uniform(-1.0, 1.0, nn)
    t0 = time.perf_counter()
    g["x_sweep"] = 0.5 * apply_additive(fine.patches, r)
    t_sweep = time.perf_counter() - t0
    g["r"] = r
    g["Ar"] = a @ r
    # first preconditioner application
    pb = nsp(b.copy())
    v0 = pb / np.linalg.norm(pb)
    g["v0"] = v0
    g["z0"] = prec(v0)
    # coarse solve on a seeded vector
    n0 = hier.levels[0].system.matrix.shape[0]
    rc = np.random.default_rng(2).uniform(-1.0, 1.0, n0)
    g["coarse_rhs"] = rc
    g["coarse_x"] = mg.coarse_solve(hier, rc)

    # FGMRES(30) as warm restarts with a fixed baseline
    t0 = time.perf_counter()
    x = None
    base = None
    hist = []
    its = 0
    converged = False
    for cycle in range(20):
        x, rep = fgmres(a, b, preconditioner=prec, rtol=1e-8, max_it=30,
                        nullspace=nsp, x0=x, target_norm=base)
        if base is None:
            base = float(np.linalg.norm(pb))
            hist.extend(rep.history.tolist())
        else:
            hist.extend(rep.history[1:].tolist())
        its += rep.iterations
        if rep.converged:
            converged = True
            break
    t_solve = time.perf_counter() - t0
    g["history"] = np.array(hist)
    g["iterations"] = np.array(its)
    g["converged"] = np.array(converged)
    g["x"] = x
    g["timings"] = np.array([t_setup, t_solve, t_sweep])
    g.update(patch_arrays(fine.patches))
    g.update(block_sample(fine.patches, a))
    np.savez_compressed(os.path.join(out_dir, f"{name}_golden.npz"), **g)
    info = {"name": name, "case": case, "k": k, "coarse": coarse,
            "refinements": refinements, "N": int(nn), "nnz": int(a.nnz),
            "J": int(fine.patches.num_patches), "iterations": int(its),
            "converged": bool(converged), "history": hist,
            "setup_s": t_setup, "solve_s": t_solve, "sweep_s": t_sweep,
            "x_norm": float(np.linalg.norm(x))}
    with open(os.path.join(hist_dir, f"{name}_history.json"), "w") as fh:
        json.dump(info, fh, indent=1)
    print(f"{name}: N={nn} nnz={a.nnz} its={its} conv={converged} setup={t_setup:.1f}s "
          f"solve={t_solve:.1f}s", flush=True)


def pack_only(name, case, k, coarse, refinements, out_dir):
    """Operators only (no factorisation / solve): the reference's own setup
    steps of build_hierarchy (mg.py:190-216) without the patch work."""
    _ref()
    import scipy.sparse as sp
    import stokesmg.mg as mg
    from stokesmg.meshtopo import build_structured_quad, build_structured_tri, refine_uniform
    from stokesmg.spaces import build_mixed
    from stokesmg.assembly import assemble, ProblemConfig
    from paper_2409_14222_b200.pack import write_pack

    build = build_structured_quad if case == "th-quad" else build_structured_tri
    meshes, links = [build(coarse)], []
    for _ in range(refinements or 0):
        fine, link = refine_uniform(meshes[-1])
        meshes.append(fine)
        links.append(link)
    cfg = ProblemConfig(case, k)
    lv = []
    for mesh in meshes:
        mixed = build_mixed(case, mesh, k)
        lv.append(SimpleNamespace(mixed=mixed, system=assemble(mixed, cfg)))
    levels = [(lv[0].mixed, lv[0].system, None)]
    for i in range(1, len(lv)):
        pv = mg.build_prolongation(lv[i - 1].mixed.velocity, lv[i].mixed.velocity, links[i - 1])
        pq = mg.build_prolongation(lv[i - 1].mixed.pressure, lv[i].mixed.pressure, links[i - 1])
        full = sp.block_diag((pv, pq), format="csr")
        levels.append((lv[i].mixed, lv[i].system, mg._mask_transfer(full, lv[i - 1], lv[i])))
    write_pack(os.path.join(out_dir, f"{name}_pack.npz"), case, k, levels,
               {"coarse": coarse, "refinements": refinements or 0})
    print(f"{name}: pack written", flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=None)
    ap.add_argument("--pack-only", action="store_true", help="operators only, no goldens")
    ap.add_argument("--small", action="store_true", help="cfg1 + small cases -> tests/golden")
    ap.add_argument("--full", action="store_true", help="cfg2..cfg5 -> data/")
    args = ap.parse_args(argv)
    names = list(args.names or [])
    if args.small:
        names += [n for n in CASES if n not in FULL]
    if args.full:
        names += list(FULL)
    golden = os.path.join(ROOT, "tests", "golden")
    data = os.path.join(ROOT, "data")
    os.makedirs(golden, exist_ok=True)
    os.makedirs(data, exist_ok=True)
    for name in names:
        case, k, n, refs = CASES[name]
        out_dir = data if name in FULL else golden
        if args.pack_only:
            pack_only(name, case, k, n, refs, out_dir)
        elif refs is None:
            single_level(name, case, k, n, out_dir)
        else:
            multilevel(name, case, k, n, refs, out_dir, golden)


if __name__ == "__main__":
    main()
