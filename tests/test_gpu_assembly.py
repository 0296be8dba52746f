"""Device assembly and device prolongation construction
(§8(f) 4) against the reference's own operators (the problem packs made
from the unmodified reference, tools/make_packs.py), and an MG-FGMRES solve
on a hierarchy built end to end on the device (no pack, no reference).

Gates
* DoF maps (cell_dofs of every level): identical to the reference's.
* operator A: identical sparsity pattern except entries at roundoff level
  (|a| <= 1e-12 of the row's largest entry, left by cancellation in one
  summation order and not the other); per entry |a - a_ref| <= 1e-13 of the
  row's largest entry (summation order of the duplicates differs).
* prolongation P (masked): identical pattern, values within 1e-14 (the
  blocks are the reference's own dual-functional evaluations).
* MG-FGMRES on device-built hierarchies: iterations identical to the
  reference's; history within the coarse-solve floor of the reference
  (tests/golden/reference_selfvar.json) scaled by 10 (the operators differ
  in the last bits everywhere, not only in the coarse solve).
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import FULL_MG, SMALL_MG, load_case

pytestmark = pytest.mark.gpu

CASE_SPEC = {   # tools/make_packs.py CASES: (case, k, coarse cells per side, refinements)
    "cfg1": ("th-tri", 2, 32, 0), "cfg2": ("th-tri", 2, 16, 4), "cfg3": ("th-tri", 4, 16, 3),
    "cfg4": ("th-quad", 3, 16, 3), "cfg5": ("bdm", 3, 16, 3),
    "s_thtri2": ("th-tri", 2, 4, 2), "s_thtri4": ("th-tri", 4, 4, 1),
    "s_thquad3": ("th-quad", 3, 4, 1), "s_bdm3": ("bdm", 3, 4, 1), "s_rt2": ("rt", 2, 4, 1),
    "s_thquad2": ("th-quad", 2, 3, 2),
    "t_bdm1_5": ("bdm", 1, 5, 0), "t_rt1_5": ("rt", 1, 5, 0), "t_thquad3_5": ("th-quad", 3, 5, 0),
    "t_bdm2_3": ("bdm", 2, 3, 0), "t_thtri3_3": ("th-tri", 3, 3, 0),
}


def _levels(name):
    from paper_2409_14222_b200 import fem
    case, k, n0, refs = CASE_SPEC[name]
    shape = "quad" if case == "th-quad" else "tri"
    return [(fem.build_mixed(case, fem.structured_mesh(shape, n0 * 2 ** i), k), shape, n0 * 2 ** i)
            for i in range(refs + 1)]


def compare_operator(a, ref, tol=1e-13, tiny=1e-12):
    """(max scaled entry error, #pattern-only entries); asserts the gates."""
    a, ref = sp.csr_matrix(a), sp.csr_matrix(ref)
    a.sort_indices()
    ref.sort_indices()
    rowmax = np.maximum(abs(ref).max(axis=1).toarray().ravel(), 1e-300)
    d = (a - ref).tocoo()
    err = np.abs(d.data) / rowmax[d.row] if d.nnz else np.zeros(0)
    pa = sp.csr_matrix((np.ones(a.nnz), a.indices, a.indptr), shape=a.shape)
    pr = sp.csr_matrix((np.ones(ref.nnz), ref.indices, ref.indptr), shape=ref.shape)
    only = (pa - pr).tocoo()
    only = only.row[only.data != 0], only.col[only.data != 0]
    vals_only = np.maximum(np.abs(np.asarray(a[only]).ravel()) if len(only[0]) else 0,
                           np.abs(np.asarray(ref[only]).ravel()) if len(only[0]) else 0)
    worst_only = float(np.max(vals_only / rowmax[only[0]])) if len(only[0]) else 0.0
    assert worst_only <= tiny, worst_only
    emax = float(err.max()) if err.size else 0.0
    assert emax <= tol, emax
    return emax, len(only[0])


ASSEMBLY_CASES = ["cfg1", "s_thtri2", "s_thtri4", "s_thquad3", "s_thquad2", "s_bdm3", "s_rt2",
                  "t_bdm1_5", "t_rt1_5", "t_thquad3_5", "t_bdm2_3", "t_thtri3_3"] + FULL_MG


@pytest.mark.parametrize("name", ASSEMBLY_CASES)
def test_device_assembly_matches_reference(name, capsys):
    from paper_2409_14222_b200 import assembly as A
    pack, _ = load_case(name)
    out = []
    for i, (mixed, _, n) in enumerate(_levels(name)):
        lvp = pack.levels[i]
        assert np.array_equal(mixed.velocity.cell_dofs, lvp.mixed.velocity.cell_dofs)
        system = A.assemble(mixed)
        assert np.array_equal(system.bc.indices, lvp.system.bc.indices)
        emax, nonly = compare_operator(system.matrix.to_scipy(), lvp.system.matrix)
        out.append(f"L{i} ({n}^2): nnz {system.matrix.nnz} vs {lvp.system.matrix.nnz}, "
                   f"max entry err {emax:.1e} of row max, {nonly} roundoff-only entries")
    with capsys.disabled():
        print(f"\n[{name}] " + "; ".join(out))


PROLONG_CASES = ["s_thtri2", "s_thtri4", "s_thquad3", "s_thquad2", "s_bdm3", "s_rt2"] + FULL_MG


@pytest.mark.parametrize("name", PROLONG_CASES)
def test_device_prolongation_matches_reference(name, capsys):
    from paper_2409_14222_b200 import assembly as A
    from paper_2409_14222_b200 import fem
    pack, _ = load_case(name)
    lv = _levels(name)
    msg = []
    for i in range(1, len(lv)):
        (cm, shape, nc), (fm, _, _) = lv[i - 1], lv[i]
        full, masked = A.build_prolongation(cm, fm, fem.refine_links(shape, nc),
                                            fem.strong_bc(cm.velocity), fem.strong_bc(fm.velocity))
        p, ref = masked.to_scipy(), sp.csr_matrix(pack.levels[i].prolong)
        ref.sort_indices()
        assert np.array_equal(p.indptr, ref.indptr) and np.array_equal(p.indices, ref.indices)
        err = float(np.max(np.abs(p.data - ref.data))) if p.nnz else 0.0
        same = bool(np.array_equal(p.data.view(np.uint64), ref.data.view(np.uint64)))
        assert err <= 1e-14, err
        msg.append(f"L{i}: nnz {p.nnz}, bit-identical {same}, max err {err:.1e}")
    with capsys.disabled():
        print(f"\n[{name}] P " + "; ".join(msg))


@pytest.mark.parametrize("name", ["s_thtri2", "s_thquad3", "s_bdm3", "s_rt2", "cfg2", "cfg4",
                                  "cfg5"])
def test_mg_fgmres_on_device_built_hierarchy(name, capsys):
    import time
    import torch
    from paper_2409_14222_b200 import assembly as A
    from paper_2409_14222_b200 import mg
    from paper_2409_14222_b200.solver import FgmresSolver, mg_rhs
    from test_gpu_parity import history_floor
    pack, g = load_case(name)
    case, k, n0, refs = CASE_SPEC[name]
    old = mg.COARSE_CELLS_PER_SIDE
    mg.COARSE_CELLS_PER_SIDE = n0
    try:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hier = A.build_hierarchy(case, k, refs, nu=2, damping=0.5)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
    finally:
        mg.COARSE_CELLS_PER_SIDE = old
    _, its, conv, hist = FgmresSolver(hier).solve(mg_rhs(pack))
    href = np.asarray(g["history"])
    m = min(len(hist), len(href))
    rel = float(np.max(np.abs(hist[:m] - href[:m]) / href[:m]))
    floor = history_floor(name)
    with capsys.disabled():
        print(f"\n[{name}] device-built hierarchy (setup {setup:.2f} s): iterations {its} "
              f"(ref {int(g['iterations'])}), history max rel {rel:.2e} (reference floor "
              f"{floor:.2e})")
    assert conv and its == int(g["iterations"])
    assert rel <= max(1e-9, 10 * floor)


# ---------------------------------------------------------------------------
# property tests of the reference's tests/test_assembly.py on the device
# assembly (same meshes, same conditions)
# ---------------------------------------------------------------------------

def system_for(case, k, n, apply_bc=True, **cfg):
    from paper_2409_14222_b200 import ProblemConfig, assemble, fem
    mesh = fem.structured_mesh("quad" if case == "th-quad" else "tri", n)
    mixed = fem.build_mixed(case, mesh, k)
    config = ProblemConfig(case, k, **cfg)
    return assemble(mixed, config, apply_bc=apply_bc), mixed, config


def sym_error(mat):
    diff = (mat - mat.T).tocoo()
    scale = np.max(np.abs(mat.data)) if mat.nnz else 1.0
    return (np.max(np.abs(diff.data)) / scale) if diff.nnz else 0.0


# reference tests/test_assembly.py:68-74, 131-134
@pytest.mark.parametrize("case,k,n", [("th-tri", 2, 3), ("th-quad", 3, 2), ("bdm", 1, 2),
                                      ("bdm", 2, 2), ("rt", 2, 2)])
def test_symmetry_and_zero_pressure_block(case, k, n):
    system, mixed, _ = system_for(case, k, n)
    mat = system.matrix.to_scipy()
    assert sym_error(mat) < 1e-10
    pp = mat[mixed.offset:, mixed.offset:]
    assert pp.nnz == 0 or np.max(np.abs(pp.data)) == 0.0


# reference tests/test_assembly.py:76-83
def test_constrained_rows_identity():
    system, mixed, _ = system_for("th-tri", 2, 2)
    mat = system.matrix.to_scipy().tocsr()
    rhs = system.rhs.cpu().numpy()
    for pos, idx in enumerate(system.bc.indices[:10]):
        row = mat.getrow(idx)
        assert row.nnz == 1 and row.indices[0] == idx
        assert row.data[0] == 1.0
        assert rhs[idx] == system.bc.values[pos]


# reference tests/test_assembly.py:85-91
def test_rigid_translation_in_kernel_of_raw_a():
    import paper_2409_14222_b200 as V
    system, mixed, _ = system_for("th-quad", 2, 2, apply_bc=False)
    const = np.zeros(mixed.ndof)
    const[0:mixed.offset:2] = 1.0   # unit x-translation
    out = V.spmv(system.matrix, const)
    assert np.max(np.abs(out[:mixed.offset])) < 1e-12


# reference tests/test_assembly.py:93-99, 211-224
@pytest.mark.parametrize("case,k,cfg,sign", [("th-tri", 2, {}, +1), ("bdm", 1, {}, +1),
                                             ("bdm", 1, {"alpha": 0.01}, -1)])
def test_velocity_block_definiteness(case, k, cfg, sign):
    system, mixed, _ = system_for(case, k, 2, **cfg)
    free = np.setdiff1d(np.arange(mixed.offset), system.bc.indices)
    a_free = system.matrix.to_scipy().tocsr()[free][:, free].toarray()
    lo = np.linalg.eigvalsh(a_free).min()
    assert lo > 1e-12 if sign > 0 else lo < -1e-8     # low penalty loses coercivity


# reference tests/test_assembly.py:101-107, 136-143
@pytest.mark.parametrize("case,k", [("th-tri", 2), ("th-quad", 2), ("bdm", 1), ("rt", 1)])
def test_constant_pressure_kernel(case, k):
    import paper_2409_14222_b200 as V
    system, mixed, _ = system_for(case, k, 3)
    vec = np.zeros(mixed.ndof)
    vec[mixed.offset:] = 1.0
    out = V.spmv(system.matrix, vec)
    scale = float(np.max(np.abs(system.matrix.to_scipy().data)))
    assert np.max(np.abs(out)) < 1e-12 * scale


# reference tests/test_assembly.py:109-127
def test_rhs_matches_independent_quadrature():
    from paper_2409_14222_b200 import fem
    from paper_2409_14222_b200.assembly import manufactured_velocity
    system, mixed, _ = system_for("th-tri", 2, 2, apply_bc=False)
    vel = mixed.velocity
    topo, geom = vel.mesh
    rule = fem.quadrature("tri", 6)
    tab = vel.element.tabulate(rule.points)
    expected = np.zeros(vel.ndof)
    for c in range(topo.num_cells):
        verts = geom.vertex_coords[geom.cell_map_vertices[c]]
        vals, _ = fem.push_forward(vel.element, "tri", verts, rule.points, tab)
        _, det, _ = fem.cell_jacobians("tri", verts, rule.points)
        f = 2.0 * np.pi ** 2 * manufactured_velocity(fem.map_points("tri", verts, rule.points))
        load = np.einsum("q,qv,qiv->i", rule.weights * det, f, vals)
        np.add.at(expected, vel.cell_dofs[c], vel.cell_dof_scale[c] * load)
    assert np.allclose(system.rhs.cpu().numpy()[:vel.ndof], expected, atol=1e-12)
