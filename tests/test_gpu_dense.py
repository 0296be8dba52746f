"""Coarse dense operator and its device inverse (vk_coarse_operator,
vk_dense_inverse) against numpy / the reference semantics
(mg.py:228-232, sparsela.lu_factor guard sparsela.py:76-83)."""

import ctypes as C

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


def _inv(m):
    import torch
    from paper_2409_14222_b200 import _lib as L
    n = m.shape[0]
    md = torch.from_numpy(np.ascontiguousarray(m)).cuda()
    out = torch.empty_like(md)
    work = torch.empty(max(int(L.lib().vk_dense_inverse_workspace(n)), 1), dtype=torch.uint8,
                       device="cuda")
    reason, col = C.c_int32(0), C.c_int32(-1)
    rc = L.lib().vk_dense_inverse(n, L.ptr(md), L.ptr(out), L.ptr(work), C.byref(reason),
                                  C.byref(col), L.stream_ptr())
    return rc, reason.value, col.value, out.cpu().numpy()


@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 64, 100, 517, 1030])
def test_dense_inverse_random(n):
    from paper_2409_14222_b200 import _lib as L
    rng = np.random.default_rng(n)
    m = rng.standard_normal((n, n))
    rc, reason, _, inv = _inv(m)
    assert rc == L.VK_OK and reason == 0
    ref = np.linalg.inv(m)
    cond = np.linalg.cond(m)
    assert np.linalg.norm(inv - ref) <= 1e-14 * cond * np.linalg.norm(ref)
    assert np.linalg.norm(inv @ m - np.eye(n)) <= 1e-13 * cond * np.sqrt(n)


def test_dense_inverse_needs_pivoting():
    # zero leading entries: only partial pivoting gets through
    from paper_2409_14222_b200 import _lib as L
    n = 70
    rng = np.random.default_rng(1)
    m = rng.standard_normal((n, n))
    m[np.arange(n), np.arange(n)] = 0.0
    m[0, :5] = 0.0
    rc, _, _, inv = _inv(m)
    assert rc == L.VK_OK
    assert np.abs(inv @ m - np.eye(n)).max() <= 1e-10


def test_dense_inverse_deterministic():
    rng = np.random.default_rng(5)
    m = rng.standard_normal((300, 300))
    a = _inv(m)[3]
    b = _inv(m)[3]
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_dense_inverse_singular_verdicts():
    from paper_2409_14222_b200 import _lib as L
    rng = np.random.default_rng(2)
    m = rng.standard_normal((40, 40))
    z = m.copy()
    z[17] = 0.0
    rc, reason, col, _ = _inv(z)
    assert rc == L.VK_SINGULAR and reason == L.VK_PATCH_ZERO_ROW and col == 17
    d = m.copy()
    d[30] = d[3]                      # exactly rank deficient
    rc, reason, _, _ = _inv(d)
    assert rc == L.VK_SINGULAR and reason == L.VK_PATCH_SMALL_PIVOT


def test_coarse_operator_bit_identical_to_numpy():
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    from conftest import load_case
    pack, _ = load_case("s_bdm3")
    c = pack.levels[0]
    q = V.pressure_kernel(c.mixed)
    a0 = c.system.matrix
    shift = np.max(np.abs(a0.data))
    ref = a0.toarray() + shift * np.outer(q, q)            # reference mg.py:229-232
    d = V.device_csr(a0)
    out = torch.empty(ref.shape, dtype=torch.float64, device="cuda")
    L.call("vk_coarse_operator", d.handle, L.ptr(torch.from_numpy(q).cuda()), float(shift),
           L.ptr(out), L.stream_ptr())
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("name", ["s_thtri2", "s_bdm3", "cfg3"])
def test_coarse_inverse_accuracy(name):
    """The device coarse inverse vs the reference's LAPACK solve: the
    difference is at the level of two valid factorizations (cond * eps)."""
    import paper_2409_14222_b200 as V
    from conftest import load_case
    pack, g = load_case(name)
    hier = V.hierarchy_from_pack(pack)
    n0 = pack.levels[0].system.matrix.shape[0]
    rc = np.random.default_rng(2).uniform(-1.0, 1.0, n0)
    x = V.coarse_solve(hier, rc)
    rel = np.linalg.norm(x - g["coarse_x"]) / np.linalg.norm(g["coarse_x"])
    print(f"\n[{name}] device coarse solve vs reference rel {rel:.3e}")
    assert rel <= 1e-6


def _lu(m):
    import torch
    from paper_2409_14222_b200 import _lib as L
    n = m.shape[0]
    md = torch.from_numpy(np.ascontiguousarray(m)).cuda()
    lu = torch.empty_like(md)
    work = torch.empty(max(int(L.lib().vk_dense_inverse_workspace(n)), 1), dtype=torch.uint8,
                       device="cuda")
    piv = np.zeros(n, dtype=np.int32)
    reason, col = C.c_int32(0), C.c_int32(-1)
    rc = L.lib().vk_dense_lu(n, L.ptr(md), L.ptr(lu), L.ptr(piv), L.ptr(work), C.byref(reason),
                             C.byref(col), L.stream_ptr())
    return rc, lu.cpu().numpy(), piv


@pytest.mark.parametrize("name", ["s_thtri2", "s_bdm3", "s_thtri4", "cfg3", "cfg5"])
def test_dense_lu_matches_lapack_pivots(name, capsys):
    """The device getrf of the coarse operator takes LAPACK's pivots (same
    swap sequence as scipy.linalg.lu_factor) and agrees with its factors to
    rounding; solving with it is as accurate as with LAPACK's."""
    import scipy.linalg as sl
    from threadpoolctl import threadpool_limits
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    from conftest import load_case
    pack, g = load_case(name)
    c = pack.levels[0]
    q = V.pressure_kernel(c.mixed)
    a0 = c.system.matrix
    m = a0.toarray() + np.max(np.abs(a0.data)) * np.outer(q, q)
    rc, lu, piv = _lu(m)
    assert rc == L.VK_OK
    with threadpool_limits(1):
        lu_ref, piv_ref = sl.lu_factor(m)
    n0 = m.shape[0]
    b = np.random.default_rng(2).uniform(-1.0, 1.0, n0)
    b = b - q * (q @ b)
    x = sl.lu_solve((lu, piv), b)
    x = x - q * (q @ x)
    ref = g["coarse_x"]
    rel_x = np.linalg.norm(x - ref) / np.linalg.norm(ref)
    rel_lu = np.linalg.norm(lu - lu_ref) / np.linalg.norm(lu_ref)
    # another valid LAPACK-type factorization (getri inverse) as the yardstick
    xi = np.linalg.inv(m) @ b
    xi = xi - q * (q @ xi)
    rel_i = np.linalg.norm(xi - ref) / np.linalg.norm(ref)
    same = float(np.mean(piv == piv_ref))
    with capsys.disabled():
        print(f"\n[{name}] pivots equal to LAPACK's: {same:.4f}; |LU - LU_lapack| rel "
              f"{rel_lu:.2e}; solve with device LU vs reference {rel_x:.2e} (LAPACK getri "
              f"inverse: {rel_i:.2e})")
    # near-ties may flip a pivot under different rounding, nothing more
    assert same >= 0.99
    assert rel_x <= max(3.0 * rel_i, 1e-12)


def test_lu_factor_beyond_the_patch_kernels():
    """sparsela.lu_factor / lu_solve of a matrix larger than the batched patch
    kernels take (s > 128) goes through the dense blocked LU: LAPACK-accurate
    solves and the reference's guard verdicts (sparsela.py:76-83)."""
    import scipy.linalg as sl
    import paper_2409_14222_b200 as V
    rng = np.random.default_rng(11)
    for n in (129, 300, 777):
        a = rng.standard_normal((n, n)) + n * np.eye(n)
        b = rng.standard_normal(n)
        fact = V.lu_factor(a)
        assert fact.shape == (n, n)
        x = V.lu_solve(fact, b)
        ref = sl.lu_solve(sl.lu_factor(a), b)
        assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
    a = rng.standard_normal((200, 200))
    a[57] = 0.0
    with pytest.raises(V.SingularMatrixError, match="all-zero row"):
        V.lu_factor(a)
    a = rng.standard_normal((200, 200))
    a[:, 120] = a[:, 3]                      # exactly dependent columns
    with pytest.raises(V.SingularMatrixError, match="pivot below 1e-12"):
        V.lu_factor(a)
