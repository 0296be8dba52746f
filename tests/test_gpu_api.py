"""The reference's own hot-path unit tests (reference tests/test_vanka.py,
tests/test_sparsela.py, tests/test_mg.py), restated against the device API.
Each test names the reference test it mirrors."""

import numpy as np
import pytest
import scipy.linalg
import scipy.sparse as sp

from conftest import load_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    import paper_2409_14222_b200 as V
    return V


def setup_case(V, name, weighting="invmult"):
    pack, g = load_case(name)
    lv = pack.fine
    return lv.system, lv.mixed, V.build_patches(lv.mixed, lv.system.bc, weighting)


# ---------------------------------------------------------------- vanka --
# reference tests/test_vanka.py:23-56
def test_patch_counts(V):
    assert setup_case(V, "t_thtri2_5")[2].num_patches == 36
    assert setup_case(V, "t_thtri4_5")[2].num_patches == 36 + 85 + 50
    assert setup_case(V, "t_thquad3_5")[2].num_patches == 36 + 60 + 25
    system, mixed, ps = setup_case(V, "t_bdm1_5")
    assert ps.num_patches == 50
    assert any(len(p.indices) == 19 and p.num_velocity == 18 for p in ps.patches)
    _, _, ps = setup_case(V, "t_rt1_5")
    sizes = sorted({len(p.indices) for p in ps.patches})
    assert sizes[-1] == 10
    assert all(len(p.indices) - p.num_velocity == 1 for p in ps.patches)


# reference tests/test_vanka.py:59-101
@pytest.mark.parametrize("name", ["t_thtri3_3", "t_thquad2_3", "t_bdm2_3", "t_rt1_3"])
def test_pressure_partition(V, name):
    system, mixed, ps = setup_case(V, name)
    assert np.all(ps.multiplicity[mixed.offset:] == 1.0)


@pytest.mark.parametrize("name", ["t_thtri2_3", "t_thquad3_2", "t_bdm1_3"])
def test_velocity_coverage(V, name):
    system, mixed, ps = setup_case(V, name)
    free = np.ones(mixed.ndof, dtype=bool)
    free[system.bc.indices] = False
    assert np.all(ps.multiplicity[free] >= 1.0)
    assert np.all(ps.multiplicity[system.bc.indices] == 0.0)


def test_determinism(V):
    _, _, p1 = setup_case(V, "t_thquad3_5")
    _, _, p2 = setup_case(V, "t_thquad3_5")
    e1, e2 = p1.export(), p2.export()
    for k in e1:
        assert np.array_equal(e1[k], e2[k])


def test_duplicate_free_sorted(V):
    _, _, ps = setup_case(V, "t_bdm2_3")
    for p in ps.patches:
        vel, pres = p.indices[:p.num_velocity], p.indices[p.num_velocity:]
        assert np.all(np.diff(vel) > 0) and np.all(np.diff(pres) > 0)


def test_b_row_support_inside_vertex_patch(V):
    system, mixed, ps = setup_case(V, "t_thtri2_3")
    mat = system.matrix.tocsr()
    bc = set(system.bc.indices.tolist())
    for p in ps.patches:
        prow = p.indices[p.num_velocity:][0]
        row = mat.getrow(prow)
        support = set(row.indices[np.abs(row.data) > 1e-14]) - {prow} - bc
        assert support <= set(p.indices[:p.num_velocity].tolist())


# reference tests/test_vanka.py:104-124
def test_local_blocks_symmetric(V):
    from paper_2409_14222_b200.vanka import extract_blocks
    system, _, ps = setup_case(V, "t_thquad2_2")
    for block in extract_blocks(ps, system.matrix, 0, 8):
        assert np.allclose(block, block.T, atol=1e-10 * np.abs(block).max())


def test_velocity_block_positive_definite(V):
    from paper_2409_14222_b200.vanka import extract_blocks
    system, _, ps = setup_case(V, "t_thtri2_2")
    k = int(np.argmax([p.num_velocity for p in ps.patches]))
    block = extract_blocks(ps, system.matrix, k, 1)[0]
    nv = ps.patches[k].num_velocity
    assert np.linalg.eigvalsh(block[:nv, :nv]).min() > 0


def test_singular_patch_reported(V):
    system, mixed, ps = setup_case(V, "t_bdm1_2")
    bad = sp.csr_matrix(system.matrix.shape)
    with pytest.raises(V.SingularMatrixError, match="entity"):
        V.factor_patches(ps, bad)


# reference tests/test_vanka.py:127-184
def test_zero_residual(V):
    system, _, ps = setup_case(V, "t_bdm1_2")
    V.factor_patches(ps, system)
    out = V.apply_additive(ps, np.zeros(system.matrix.shape[0]))
    assert np.all(out == 0.0)


def test_single_patch_exact_solve(V):
    rng = np.random.default_rng(0)
    m = rng.standard_normal((8, 8))
    a = sp.csr_matrix(m @ m.T + 8 * np.eye(8))
    patch = V.Patch(None, np.arange(8), 8, weights=np.ones(8))
    pset = V.PatchSet([patch], 8, np.ones(8), "unit")
    V.factor_patches(pset, a)
    r = rng.standard_normal(8)
    assert np.allclose(V.apply_additive(pset, r), np.linalg.solve(a.toarray(), r), atol=1e-12)


def test_two_patch_brute_force_oracle(V):
    rng = np.random.default_rng(1)
    m = rng.standard_normal((6, 6))
    a = m @ m.T + 6 * np.eye(6)
    idx1, idx2 = np.arange(4), np.arange(2, 6)
    mult = np.zeros(6)
    mult[idx1] += 1
    mult[idx2] += 1
    p1 = V.Patch(None, idx1, 4, weights=1.0 / mult[idx1])
    p2 = V.Patch(None, idx2, 4, weights=1.0 / mult[idx2])
    pset = V.PatchSet([p1, p2], 6, mult, "invmult")
    V.factor_patches(pset, sp.csr_matrix(a))
    r = rng.standard_normal(6)
    got = V.apply_additive(pset, r)
    expected = np.zeros(6)
    for idx in (idx1, idx2):
        rmat = np.zeros((4, 6))
        rmat[np.arange(4), idx] = 1.0
        local = np.linalg.solve(rmat @ a @ rmat.T, rmat @ r)
        expected += rmat.T @ (np.diag(1.0 / mult[idx]) @ local)
    assert np.allclose(got, expected, atol=1e-12)


def test_linearity(V):
    system, _, ps = setup_case(V, "t_thtri2_2")
    V.factor_patches(ps, system)
    rng = np.random.default_rng(2)
    r1 = rng.standard_normal(system.matrix.shape[0])
    r2 = rng.standard_normal(system.matrix.shape[0])
    c = 0.37
    lhs = V.apply_additive(ps, r1 + c * r2)
    rhs = V.apply_additive(ps, r1) + c * V.apply_additive(ps, r2)
    assert np.allclose(lhs, rhs, atol=1e-12 * max(1, np.abs(lhs).max()))


def test_unit_weighting_option(V):
    _, _, ps = setup_case(V, "t_thtri2_2", weighting="unit")
    for p in ps.patches:
        assert np.all(p.weights == 1.0)


def test_unknown_weighting_rejected(V):
    pack, _ = load_case("t_thtri2_2")
    with pytest.raises(ValueError):
        V.build_patches(pack.fine.mixed, pack.fine.system.bc, "bogus")


def test_wrong_case_rejected(V):
    pack, _ = load_case("t_bdm1_2")
    with pytest.raises(ValueError):
        V.build_patches_taylor_hood(pack.fine.mixed, pack.fine.system.bc)


# ------------------------------------------------------------- sparsela --
def random_csr(rng, n, m, density=0.3):
    dense = rng.standard_normal((n, m)) * (rng.random((n, m)) < density)
    return sp.csr_matrix(dense), dense


# reference tests/test_sparsela.py:17-55
def test_spmv_cases(V):
    x = np.arange(5.0)
    assert np.array_equal(V.spmv(sp.eye(5, format="csr"), x), x)
    a, dense = random_csr(np.random.default_rng(0), 5, 5)
    assert np.array_equal(V.spmv(a, np.zeros(5)), np.zeros(5))
    rng = np.random.default_rng(1)
    a, dense = random_csr(rng, 5, 5)
    x = rng.standard_normal(5)
    assert np.allclose(V.spmv(a, x), dense @ x, atol=1e-14)
    assert np.array_equal(V.spmv(a, x).view(np.uint64), (a @ x).view(np.uint64))


def test_spmv_long_rows_and_empty_rows(V):
    rng = np.random.default_rng(9)
    dense = np.zeros((40, 5000))
    dense[3] = rng.standard_normal(5000)            # one row > one 2048-chunk
    dense[7, ::3] = rng.standard_normal(1667)
    a = sp.csr_matrix(dense)
    x = rng.standard_normal(5000)
    assert np.array_equal(V.spmv(a, x).view(np.uint64), (a @ x).view(np.uint64))


def test_extract_cases(V):
    rng = np.random.default_rng(2)
    a, dense = random_csr(rng, 6, 6)
    assert np.array_equal(V.extract_submatrix(a, np.arange(6), np.arange(6)), dense)
    assert V.extract_submatrix(a, [], []).shape == (0, 0)
    rng = np.random.default_rng(4)
    a, dense = random_csr(rng, 30, 30)
    rows = np.sort(rng.choice(30, size=7, replace=False))
    cols = np.sort(rng.choice(30, size=11, replace=False))
    assert np.array_equal(V.extract_submatrix(a, rows, cols), dense[np.ix_(rows, cols)])
    with pytest.raises(ValueError):
        V.extract_submatrix(a, [2, 1], [0])


# reference tests/test_sparsela.py:58-98
def test_dense_lu(V):
    fact = V.lu_factor(np.eye(3))
    b = np.array([1.0, 2.0, 3.0])
    assert np.allclose(V.lu_solve(fact, b), b)
    fact = V.lu_factor(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert np.allclose(V.lu_solve(fact, np.array([2.0, 5.0])), [5.0, 2.0])
    rng = np.random.default_rng(6)
    m = rng.standard_normal((40, 40))
    a = np.block([[m @ m.T + 40 * np.eye(40), rng.standard_normal((40, 10))],
                  [rng.standard_normal((10, 40)), np.zeros((10, 10))]])
    a[40:, :40] = a[:40, 40:].T
    b = rng.standard_normal(50)
    x = V.lu_solve(V.lu_factor(a), b)
    denom = np.linalg.norm(a, np.inf) * np.linalg.norm(x) + np.linalg.norm(b)
    assert np.linalg.norm(a @ x - b) <= 1e-10 * denom
    with pytest.raises(V.SingularMatrixError):
        V.lu_factor(np.ones((3, 3)))
    with pytest.raises(V.SingularMatrixError, match="all-zero row"):
        V.lu_factor(np.array([[1.0, 2.0], [0.0, 0.0]]))


# reference tests/test_sparsela.py:116-223
def test_fgmres_identity_one_iteration(V):
    b = np.array([3.0, -1.0, 2.0])
    x, rep = V.fgmres(sp.eye(3, format="csr"), b, rtol=1e-12)
    assert rep.converged and rep.iterations == 1
    assert np.allclose(x, b)


def test_fgmres_finite_termination(V):
    a = sp.diags(np.arange(1.0, 11.0)).tocsr()
    b = np.random.default_rng(10).standard_normal(10)
    x, rep = V.fgmres(a, b, rtol=1e-12, max_it=30)
    assert rep.converged and rep.iterations <= 10
    assert np.allclose(a @ x, b, atol=1e-10)


def test_fgmres_monotone_history(V):
    rng = np.random.default_rng(11)
    a = sp.csr_matrix(rng.standard_normal((40, 40)) + 8 * np.eye(40))
    b = rng.standard_normal(40)
    _, rep = V.fgmres(a, b, rtol=1e-12, max_it=40)
    assert np.all(np.diff(rep.history) <= 1e-14)
    assert len(rep.history) == rep.iterations + 1
    assert rep.history[-1] <= 1e-12


def test_fgmres_host_ssor_preconditioner(V):
    rng = np.random.default_rng(12)
    m = rng.standard_normal((100, 100))
    a = m @ m.T + 100 * np.eye(100)
    b = rng.standard_normal(100)
    lower, diag = np.tril(a), np.diag(a)

    def ssor(r):
        y = scipy.linalg.solve_triangular(lower, r, lower=True)
        return scipy.linalg.solve_triangular(lower.T, diag * y, lower=False)

    x, rep = V.fgmres(sp.csr_matrix(a), b, preconditioner=ssor, rtol=1e-12, max_it=100)
    exact = np.linalg.solve(a, b)
    assert rep.converged
    assert np.linalg.norm(x - exact) <= 1e-8 * np.linalg.norm(exact)


def test_fgmres_nullspace(V):
    rng = np.random.default_rng(14)
    q = np.ones(20) / np.sqrt(20)
    m = rng.standard_normal((20, 20))
    a = m @ m.T + 20 * np.eye(20)
    proj = np.eye(20) - np.outer(q, q)
    a = proj @ a @ proj
    b = rng.standard_normal(20)
    nsp = V.nullspace_projector([q])
    x, rep = V.fgmres(sp.csr_matrix(a), b, rtol=1e-12, max_it=40, nullspace=nsp)
    assert rep.converged
    assert abs(q @ x) < 1e-12
    assert np.linalg.norm(a @ x - proj @ b) < 1e-9 * np.linalg.norm(b)


def test_fgmres_breakdown(V):
    a = sp.diags([1.0, 2.0, 3.0]).tocsr()
    b = np.array([2.0, 0.0, 0.0])
    x, rep = V.fgmres(a, b, rtol=1e-16, max_it=10)
    assert rep.breakdown and rep.converged
    assert np.allclose(x, [2.0, 0.0, 0.0], atol=1e-14)


def test_fgmres_warm_restart(V):
    rng = np.random.default_rng(15)
    a = sp.csr_matrix(rng.standard_normal((30, 30)) + 6 * np.eye(30))
    b = rng.standard_normal(30)
    base = np.linalg.norm(b)
    x1, _ = V.fgmres(a, b, rtol=1e-4, max_it=50, target_norm=base)
    x2, rep2 = V.fgmres(a, b, rtol=1e-10, max_it=50, x0=x1, target_norm=base)
    assert rep2.converged
    assert np.linalg.norm(b - a @ x2) <= 1e-10 * base * (1 + 1e-9)


def test_fgmres_matches_oracle_exactly_on_small_case(V):
    # same MGS / Givens arithmetic as the reference (sparsela.py:155-189)
    from oracle import vanka_oracle as O
    rng = np.random.default_rng(13)
    n = 50
    a = sp.csr_matrix(rng.standard_normal((n, n)) + 10 * np.eye(n))
    b = rng.standard_normal(n)
    _, rep = V.fgmres(a, b, rtol=1e-12, max_it=40)
    _, rep_o = O.fgmres(a, b, rtol=1e-12, max_it=40)
    assert rep.iterations == rep_o.iterations
    assert np.allclose(rep.history, rep_o.history, rtol=1e-8, atol=0)


# reference tests/test_sparsela.py:226-252
def test_lambda_max(V):
    a = sp.diags([1.0, 2.0, 4.0]).tocsr()
    assert V.estimate_lambda_max(a, m=3, seed=0) == pytest.approx(4.0, abs=1e-10)
    rng = np.random.default_rng(16)
    m = rng.standard_normal((60, 60))
    a = m @ m.T + np.eye(60)
    true = np.max(np.linalg.eigvalsh(a))
    lam = V.estimate_lambda_max(sp.csr_matrix(a), m=10, seed=1)
    assert 0.8 * true <= lam <= true * (1 + 1e-6)
    a = sp.diags([1.0, 2.0, 8.0]).tocsr()
    minv = lambda r: r / np.array([1.0, 2.0, 8.0])  # noqa: E731
    assert V.estimate_lambda_max(a, m=3, seed=0, preconditioner=minv) == pytest.approx(1.0, abs=1e-10)


def test_nullspace_projector(V):
    proj = V.nullspace_projector([np.array([1.0, 1.0, 1.0, 1.0])])
    assert np.allclose(proj(np.ones(4)), 0.0, atol=1e-14)
    proj = V.nullspace_projector([np.array([1.0, 0.0, 0.0])])
    v = np.array([0.0, 2.0, -3.0])
    assert np.allclose(proj(v), v)
    with pytest.raises(ValueError):
        V.nullspace_projector([np.array([1.0, 2.0, 3.0]), np.array([2.0, 4.0, 6.0])])


# ------------------------------------------------------------------- mg --
@pytest.fixture(scope="module")
def hier_thtri2():
    import paper_2409_14222_b200 as V
    pack, _ = load_case("s_thtri2")
    return pack, V.hierarchy_from_pack(pack)


# reference tests/test_mg.py:112-164
def test_chebyshev_zero_residual_noop(V, hier_thtri2):
    pack, hier = hier_thtri2
    level = hier.fine
    x = np.random.default_rng(2).standard_normal(level.n)
    b = level.system.matrix @ x
    for mode in ("degree", "repeat"):
        out = V.chebyshev_relax(level, b, x.copy(), 3, mode)
        assert np.allclose(out, x, atol=1e-10 * np.abs(x).max())


def test_chebyshev_degree_one_is_damped_step(V, hier_thtri2):
    pack, hier = hier_thtri2
    level = hier.fine
    b = np.random.default_rng(3).standard_normal(level.n)
    got = V.chebyshev_relax(level, b, np.zeros_like(b), 1)
    damp = 2.0 / (level.cheb.lower + level.cheb.upper)
    expected = damp * V.apply_additive(level.patches, b)
    assert np.allclose(got, expected, atol=1e-13 * max(1, np.abs(b).max()))


def test_repeat_mode_is_iterated_damping(V, hier_thtri2):
    pack, hier = hier_thtri2
    level = hier.fine
    b = np.random.default_rng(5).standard_normal(level.n)
    damp = 2.0 / (level.cheb.lower + level.cheb.upper)
    x = np.zeros_like(b)
    for _ in range(3):
        x = x + damp * V.apply_additive(level.patches, b - level.system.matrix @ x)
    got = V.chebyshev_relax(level, b, np.zeros_like(b), 3, "repeat")
    assert np.allclose(got, x, atol=1e-12 * max(1, np.abs(x).max()))


def test_minimax_bound_on_model_spectrum(V):
    import torch
    lam = np.linspace(25.0, 110.0, 200)
    rng = np.random.default_rng(4)
    xstar, e0 = rng.standard_normal(200), rng.standard_normal(200)
    ld = torch.from_numpy(lam).cuda()
    op = lambda v: ld * v  # noqa: E731
    op._device = True
    ident = lambda r: r  # noqa: E731
    ident._device = True
    for nu in (1, 2, 3, 4):
        x = V.chebyshev_iteration(op, ident, 25.0, 110.0, torch.from_numpy(lam * xstar).cuda(),
                                  torch.from_numpy(xstar - e0).cuda(), nu).cpu().numpy()
        theta = 0.5 * (110.0 + 25.0) / (0.5 * (110.0 - 25.0))
        bound = 1.0 / np.cosh(nu * np.arccosh(theta))
        assert np.max(np.abs((xstar - x) / e0)) <= bound * 1.05


# reference tests/test_mg.py:167-217
def test_vcycle_linearity(V):
    pack, _ = load_case("s_bdm3")
    hier = V.hierarchy_from_pack(pack)
    n = hier.fine.n
    rng = np.random.default_rng(7)
    r1, r2 = rng.standard_normal(n), rng.standard_normal(n)
    c = -1.3
    lhs = V.v_cycle(hier, r1 + c * r2)
    rhs = V.v_cycle(hier, r1) + c * V.v_cycle(hier, r2)
    assert np.allclose(lhs, rhs, atol=1e-12 * max(1, np.abs(lhs).max()))


def test_vcycle_graph_matches_eager(V, hier_thtri2):
    pack, hier = hier_thtri2
    b = np.random.default_rng(8).standard_normal(hier.fine.n)
    import torch
    bd = torch.from_numpy(b).cuda()
    g = hier.vcycle_device(bd, graph=True).clone()
    e = hier.vcycle_device(bd, graph=False).clone()
    assert torch.equal(g, e)


def test_restriction_is_transpose(V, hier_thtri2):
    pack, hier = hier_thtri2
    t = hier.transfers[-1]
    rng = np.random.default_rng(8)
    xf = rng.standard_normal(t.masked.shape[0])
    xc = rng.standard_normal(t.masked.shape[1])
    assert np.allclose(xf @ t.prolong(xc), t.restrict(xf) @ xc, atol=1e-12)
    # bit-identical with scipy's csr / csc matvec
    assert np.array_equal(t.prolong(xc).view(np.uint64), (t.masked @ xc).view(np.uint64))
    assert np.array_equal(t.restrict(xf).view(np.uint64), (t.masked.T @ xf).view(np.uint64))


def test_single_level_is_direct_solve(V):
    pack, _ = load_case("t_thtri2_5")
    hier = V.hierarchy_from_pack(pack)
    q = V.pressure_kernel(pack.fine.mixed)
    b = np.random.default_rng(6).standard_normal(len(q))
    b -= q * (q @ b)
    x = V.v_cycle(hier, b)
    assert np.allclose(x, V.coarse_solve(hier, b))
    assert abs(q @ x) < 1e-12 * np.linalg.norm(x)
    assert np.linalg.norm(pack.fine.system.matrix @ x - b) < 1e-9 * np.linalg.norm(b)


def test_fgmres_step_graphs_match_eager(V):
    # one CUDA graph per Arnoldi step (FgmresWorkspace) == kernel-by-kernel
    pack, _ = load_case("s_bdm3")
    hier = V.hierarchy_from_pack(pack)
    from paper_2409_14222_b200.solver import mg_rhs
    b = mg_rhs(pack)
    nsp = V.nullspace_projector([V.pressure_kernel(pack.fine.mixed)])
    prec = V.make_preconditioner(hier)
    A = pack.fine.system.matrix
    x1, r1 = V.fgmres(A, b, preconditioner=prec, rtol=1e-8, max_it=30, nullspace=nsp)
    ws = V.FgmresWorkspace(len(b), 30)
    x2, r2 = V.fgmres(A, b, preconditioner=prec, rtol=1e-8, max_it=30, nullspace=nsp,
                      workspace=ws)
    x3, r3 = V.fgmres(A, b, preconditioner=prec, rtol=1e-8, max_it=30, nullspace=nsp,
                      workspace=ws)                     # replays the captured graphs
    assert len(ws.graphs) == r2.iterations
    for r in (r2, r3):
        assert r.iterations == r1.iterations
        assert np.array_equal(r.history, r1.history)
    assert np.array_equal(x1, x2) and np.array_equal(x1, x3)


def test_preconditioned_solver_converges(V):
    pack, _ = load_case("s_thquad2")
    hier = V.hierarchy_from_pack(pack)
    from paper_2409_14222_b200.solver import mg_rhs
    nsp = V.nullspace_projector([V.pressure_kernel(pack.fine.mixed)])
    x, rep = V.fgmres(pack.fine.system.matrix, mg_rhs(pack),
                      preconditioner=V.make_preconditioner(hier), rtol=1e-10, max_it=40,
                      nullspace=nsp)
    assert rep.converged and rep.iterations <= 40
