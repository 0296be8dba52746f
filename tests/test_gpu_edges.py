"""Edge cases of the device path (empty / ragged / maximum sizes, singular
blocks), each checked against the oracle or the reference semantics."""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    import paper_2409_14222_b200 as V
    return V


def _ref_like_mixed(cell_dofs, nvel, npres):
    """Minimal duck-typed MixedSpace for direct builder calls."""
    from paper_2409_14222_b200.pack import (LiteMesh, LiteMixed, LiteSpace, LiteTopology)
    nc = cell_dofs.shape[0]
    topo = LiteTopology("tri", 1, 0, 0, nc, np.zeros((nc, 3), np.int32),
                        np.zeros(1, np.int32), np.zeros(0, np.int32),
                        np.zeros(1, np.int32), np.zeros(0, np.int32))
    mesh = LiteMesh(topo)
    vel = LiteSpace(mesh, nvel, {}, cell_dofs)
    pres = LiteSpace(mesh, npres, {})
    return LiteMixed(vel, pres, "th-tri", 2)


def test_empty_candidates_dropped_like_reference(V):
    # reference vanka._finish drops patches with no dofs (vanka.py:64-65)
    from paper_2409_14222_b200.vanka import _launch_build, _Entities
    cd = np.array([[0, 1, 2], [2, 3, 4]], dtype=np.int64)
    mixed = _ref_like_mixed(cd, 5, 2)
    bc = type("B", (), {"indices": np.array([0, 1, 2])})()
    # candidate 0: cell 0 only, all constrained, no pressure -> empty -> dropped
    # candidate 1: no cells, pressure dof 5
    # candidate 2: cell 1 + pressure 6
    e2c_ptr = np.array([0, 1, 1, 2], np.int32)
    e2c = np.array([0, 1], np.int32)
    pptr = np.array([0, 0, 1, 2], np.int32)
    pdofs = np.array([5, 6], np.int32)
    ps = _launch_build(mixed, bc, "invmult", e2c_ptr, e2c, pptr, pdofs,
                       _Entities([(0, 3)]))
    ex = ps.export()
    assert ps.num_patches == 2
    assert ex["candidate"].tolist() == [1, 2]
    assert ex["indices"].tolist() == [5, 3, 4, 6]
    assert ex["num_velocity"].tolist() == [0, 2]
    assert ex["multiplicity"].tolist() == [0, 0, 0, 1, 1, 1, 1]
    assert ps.entity_of(0).index == 1


def test_size_one_patches_and_zero_row(V):
    a = sp.csr_matrix(np.diag([2.0, 4.0, 8.0]))
    ps = V.PatchSet([V.Patch(None, np.array([i]), 1, np.ones(1)) for i in range(3)], 3,
                    np.ones(3), "unit")
    V.factor_patches(ps, a)
    out = V.apply_additive(ps, np.array([1.0, 1.0, 1.0]))
    assert np.array_equal(out, [0.5, 0.25, 0.125])
    bad = sp.csr_matrix(np.diag([2.0, 0.0, 8.0]))
    ps2 = V.PatchSet([V.Patch(("e", i), np.array([i]), 1, np.ones(1)) for i in range(3)], 3,
                     np.ones(3), "unit")
    with pytest.raises(V.SingularMatrixError, match="entity"):
        V.factor_patches(ps2, bad)


def test_small_pivot_guard_matches_oracle(V):
    from oracle import vanka_oracle as O
    # pivot exactly at / below the 1e-12 row-scale threshold (sparsela.py:82-83)
    for eps, singular in [(1e-13, True), (1e-11, False)]:
        m = np.array([[1.0, 1.0], [1.0, 1.0 + eps]])
        ok_o = True
        try:
            O.lu_factor(m)
        except O.SingularMatrixError:
            ok_o = False
        ok_g = True
        try:
            V.lu_factor(m)
        except V.SingularMatrixError:
            ok_g = False
        assert ok_o == ok_g == (not singular)


def test_oversize_patch_rejected(V):
    n = 200
    a = sp.identity(n, format="csr")
    ps = V.PatchSet([V.Patch(None, np.arange(n), n, np.ones(n))], n, np.ones(n), "unit")
    with pytest.raises(NotImplementedError):
        V.factor_patches(ps, a)


def test_largest_supported_patch(V):
    rng = np.random.default_rng(3)
    n = 164
    m = rng.standard_normal((n, n)) + n * np.eye(n)
    ps = V.PatchSet([V.Patch(None, np.arange(n), n, np.ones(n))], n, np.ones(n), "unit")
    V.factor_patches(ps, sp.csr_matrix(m))
    r = rng.standard_normal(n)
    assert np.allclose(V.apply_additive(ps, r), np.linalg.solve(m, r), rtol=1e-12, atol=1e-14)


def test_unsorted_patch_lists_rejected(V):
    ps = V.PatchSet([V.Patch(None, np.array([2, 1]), 2, np.ones(2))], 3, np.ones(3), "unit")
    with pytest.raises(ValueError):
        V.factor_patches(ps, sp.identity(3, format="csr"))


def test_empty_and_zero_matrices(V):
    z = sp.csr_matrix((7, 5))
    assert np.array_equal(V.spmv(z, np.ones(5)), np.zeros(7))
    e = sp.csr_matrix((0, 4))
    assert V.spmv(e, np.ones(4)).shape == (0,)
    # rows of all-zero entries in a block of 600 empty rows (masked BC rows)
    rng = np.random.default_rng(4)
    d = np.zeros((1500, 300))
    d[::3] = rng.standard_normal((500, 300)) * (rng.random((500, 300)) < 0.05)
    a = sp.csr_matrix(d)
    x = rng.standard_normal(300)
    assert np.array_equal(V.spmv(a, x).view(np.uint64), (a @ x).view(np.uint64))


def test_residual_bit_identical_to_scipy(V):
    import torch
    from conftest import load_case
    pack, _ = load_case("s_bdm3")
    a = pack.fine.system.matrix
    rng = np.random.default_rng(5)
    b, x = rng.standard_normal(a.shape[0]), rng.standard_normal(a.shape[0])
    d = V.device_csr(a)
    r = torch.empty(a.shape[0], dtype=torch.float64, device="cuda")
    d.residual(torch.from_numpy(b).cuda(), torch.from_numpy(x).cuda(), r)
    assert np.array_equal(r.cpu().numpy().view(np.uint64), (b - a @ x).view(np.uint64))


def test_apply_accumulation_order_matches_reference(V):
    # the DoF-major accumulation reproduces out[idx] += w*local in patch order
    # exactly: feeding the oracle's local solves through the same order gives
    # the same bits when the local solves agree (here: 1x1 patches)
    rng = np.random.default_rng(6)
    n = 50
    diag = rng.uniform(1, 2, n)
    a = sp.csr_matrix(np.diag(diag))
    patches = []
    mult = np.zeros(n)
    for _ in range(200):
        i = int(rng.integers(n))
        patches.append(V.Patch(None, np.array([i]), 1, None))
        mult[i] += 1
    for p in patches:
        p.weights = 1.0 / mult[p.indices]
    ps = V.PatchSet(patches, n, mult, "invmult")
    V.factor_patches(ps, a)
    r = rng.standard_normal(n)
    got = V.apply_additive(ps, r)
    inv = 1.0 / diag          # device inverse of a 1x1 block is 1/a exactly
    ref = np.zeros(n)
    for p in patches:
        ref[p.indices] += p.weights * (inv[p.indices] * r[p.indices])
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("n", [0, 1, 257, 75_776, 592_387])
def test_fused_mgs_step_bit_identical(V, n):
    """vk_axpy_dot == vk_axpy_dev then vk_dot / vk_nrm2, bit for bit."""
    import torch
    from paper_2409_14222_b200 import _lib as L
    rng = np.random.default_rng(n)
    x = torch.from_numpy(rng.standard_normal(n)).cuda()
    x2 = torch.from_numpy(rng.standard_normal(n)).cuda()
    w0 = torch.from_numpy(rng.standard_normal(n)).cuda()
    a = torch.tensor([0.37], dtype=torch.float64, device="cuda")
    st = L.stream_ptr()
    red = L.reduce_scratch()[0]
    for sqrt_out in (0, 1):
        w1, w2 = w0.clone(), w0.clone()
        o1 = torch.zeros(1, dtype=torch.float64, device="cuda")
        o2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        L.call("vk_axpy_dev", n, L.ptr(a), L.ptr(x), L.ptr(w1), st)
        if sqrt_out:
            L.call("vk_nrm2", n, L.ptr(w1), L.ptr(o1), L.ptr(red), st)
            L.call("vk_axpy_dot", n, L.ptr(a), L.ptr(x), L.ptr(w2), L.ptr(w2), L.ptr(o2), 1,
                   L.ptr(red), st)
        else:
            L.call("vk_dot", n, L.ptr(x2), L.ptr(w1), L.ptr(o1), L.ptr(red), st)
            L.call("vk_axpy_dot", n, L.ptr(a), L.ptr(x), L.ptr(w2), L.ptr(x2), L.ptr(o2), 0,
                   L.ptr(red), st)
        torch.cuda.synchronize()
        assert torch.equal(w1, w2)
        assert o1.cpu().numpy().view(np.uint64)[0] == o2.cpu().numpy().view(np.uint64)[0]


@pytest.mark.parametrize("name", ["s_thtri2", "s_thtri4", "s_bdm3"])
def test_refactor_reuses_schedule_and_tracks_values(V, name):
    """Re-factorising a patch set (schedule and operator storage cached in
    the handle, size classes on two streams) reproduces the first
    factorisation bit for bit, and follows new matrix values: Gauss-Jordan
    is exactly equivariant under a power-of-two scaling, so inv(2A) = inv(A)/2
    to the last bit."""
    import scipy.sparse as sp
    from conftest import load_case
    from paper_2409_14222_b200.vanka import patch_inverses
    pack, _ = load_case(name)
    lv = pack.fine
    ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), lv.system)
    n = ps.num_patches
    pick = sorted({0, n // 3, n // 2, n - 1})
    first = [patch_inverses(ps, p, 1)[0] for p in pick]
    V.factor_patches(ps, lv.system)                       # same values again
    again = [patch_inverses(ps, p, 1)[0] for p in pick]
    for a, b in zip(first, again):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    a2 = sp.csr_matrix(lv.system.matrix * 2.0)
    V.factor_patches(ps, a2)
    halved = [patch_inverses(ps, p, 1)[0] for p in pick]
    for a, h in zip(first, halved):
        assert np.array_equal((a * 0.5).view(np.uint64), h.view(np.uint64))


@pytest.mark.parametrize("name", ["s_thtri4", "s_bdm3"])
def test_refactor_rebuilds_extraction_map_on_new_pattern(V, name):
    """The extraction map cached by the first factorisation (CSR entry ->
    patch-local column) is keyed by the matrix's sparsity pattern: factoring
    against the same values stored with extra explicit zeros (every row
    offset shifted) must reproduce the first inverses bit for bit, and so
    must going back to the original matrix; the inverses agree with numpy's
    inverse of the extracted block."""
    import scipy.sparse as sp
    from conftest import load_case
    from paper_2409_14222_b200.vanka import patch_inverses
    pack, _ = load_case(name)
    lv = pack.fine
    a = sp.csr_matrix(lv.system.matrix)
    ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), a)
    n = ps.num_patches
    pick = sorted({0, n // 5, n // 2, n - 1})
    first = [patch_inverses(ps, p, 1)[0] for p in pick]
    rng = np.random.default_rng(7)
    coo = a.tocoo()
    m = a.shape[0]
    extra_r = rng.integers(0, m, 4 * m)
    extra_c = rng.integers(0, m, 4 * m)
    keep = a[extra_r, extra_c].A1 == 0          # only positions not yet stored
    padded = sp.csr_matrix((np.concatenate([coo.data, np.zeros(int(keep.sum()))]),
                            (np.concatenate([coo.row, extra_r[keep]]),
                             np.concatenate([coo.col, extra_c[keep]]))), shape=a.shape)
    padded.sum_duplicates()
    padded.sort_indices()
    assert padded.nnz > a.nnz
    V.factor_patches(ps, padded)
    second = [patch_inverses(ps, p, 1)[0] for p in pick]
    V.factor_patches(ps, a)
    third = [patch_inverses(ps, p, 1)[0] for p in pick]
    exp = ps.export()
    ad = a.tocsr()
    for k, p in enumerate(pick):
        assert np.array_equal(first[k].view(np.uint64), second[k].view(np.uint64))
        assert np.array_equal(first[k].view(np.uint64), third[k].view(np.uint64))
        ii = exp["indices"][exp["offsets"][p]:exp["offsets"][p + 1]]
        blk = ad[ii][:, ii].toarray()
        ref = np.linalg.inv(blk)
        err = np.abs(first[k] - ref).max() / np.abs(ref).max()
        assert err <= 1e2 * np.finfo(float).eps * np.linalg.cond(blk)


def _uniform_patch_system(npatch, s, seed):
    """Diagonally dominant sparse matrix + `npatch` random sorted patches of
    exactly `s` DoFs (every block is nonsingular)."""
    rng = np.random.default_rng(seed)
    n = 4 * npatch + s
    a = sp.random(n, n, density=8.0 / n, random_state=seed, format="csr")
    a = (a + a.T + sp.diags(np.full(n, 40.0))).tocsr()
    a.sort_indices()
    idx = [np.sort(rng.choice(n, size=s, replace=False)) for _ in range(npatch)]
    return a, idx


def _dense_sweep(a, idx, r, weights):
    out = np.zeros(a.shape[0])
    ad = a.toarray()
    for ii, w in zip(idx, weights):
        if ii.size == 0:
            continue
        out[ii] += w * np.linalg.solve(ad[np.ix_(ii, ii)], r[ii])
    return out


@pytest.mark.parametrize("s", [16, 29])
def test_bulk_kernel_uniform_small_patches(V, s):
    """>= 4,736 uniform patches of s <= 30 take the TMA bulk-copy sweep with
    one row slot per lane (R = 1); lanes past s must not read past their
    shared-memory stage: the result matches a dense solve."""
    npatch = 5000
    a, idx = _uniform_patch_system(npatch, s, seed=s)
    ps = V.PatchSet([V.Patch(None, ii, s, np.ones(s)) for ii in idx], a.shape[0],
                    None, "unit")
    V.factor_patches(ps, a)
    r = np.random.default_rng(1).uniform(-1, 1, a.shape[0])
    got = V.apply_additive(ps, r)
    ref = _dense_sweep(a, idx, r, [np.ones(s)] * npatch)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_zero_size_patches_are_dropped(V):
    """Hand-built patch lists may hold size-0 patches (the reference's
    apply_additive skips them, lu_solve of s=0 is empty); the device handle
    drops them and keeps the input position for entity lookup."""
    a, idx = _uniform_patch_system(40, 7, seed=3)
    pats, ents = [], []
    for k, ii in enumerate(idx):
        if k % 5 == 0:
            pats.append(V.Patch(("empty", k), np.zeros(0, np.int64), 0, np.ones(0)))
        pats.append(V.Patch(("p", k), ii, 7, np.ones(7)))
    ps = V.PatchSet(pats, a.shape[0], None, "unit")
    V.factor_patches(ps, a)
    ex = ps.export()
    assert len(ex["offsets"]) - 1 == 40
    assert all(ps.entity_of(p)[0] == "p" for p in range(40))
    assert [ps.entity_of(p)[1] for p in range(40)] == list(range(40))
    r = np.random.default_rng(2).uniform(-1, 1, a.shape[0])
    got = V.apply_additive(ps, r)
    ref = _dense_sweep(a, idx, r, [np.ones(7)] * 40)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_device_csr_cache_follows_in_place_changes(V):
    """The reference reads the live scipy matrix on every call; the device
    copy cache must notice ``A.data *= 2``."""
    a = sp.random(500, 500, density=0.02, random_state=4, format="csr") + sp.eye(500)
    a = a.tocsr()
    x = np.random.default_rng(0).standard_normal(500)
    y1 = V.spmv(a, x)
    a.data *= 2.0
    y2 = V.spmv(a, x)
    assert np.array_equal(y2, 2.0 * y1)
    assert np.array_equal(y2, a @ x)
