"""K5/K6 kernel selection: the thread-per-row kernel (short rows, e.g.
prolongations) and the block stream kernel must both reproduce scipy's
csr_matvec bit for bit (reference sparsela.py:45-47, mg.py:41-45, 270, 294),
for y = A x, the prolong-add y += P x, and the fused residual b - A x."""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    import paper_2409_14222_b200 as V
    return V


def _csr_with_row_lengths(rng, lens, ncols):
    """Random CSR with the given stored entries per row (sorted, distinct
    columns, no explicit zeros)."""
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    cols = np.concatenate([np.sort(rng.choice(ncols, size=l, replace=False)) for l in lens]
                          ).astype(np.int32) if len(lens) else np.zeros(0, np.int32)
    vals = rng.standard_normal(int(indptr[-1]))
    vals[vals == 0.0] = 1.0
    return sp.csr_matrix((vals, cols, indptr), shape=(len(lens), ncols))


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


CASES = {
    # mean over 32-row groups of the longest row <= 11 -> csr_row_kernel
    "short": lambda rng: rng.integers(0, 9, 7000),
    # prolongation-like: 1-5 entries, some empty rows (masked BC rows)
    "prolong": lambda rng: np.where(rng.random(9000) < 0.1, 0, rng.integers(1, 6, 9000)),
    # stream kernel: 12-60 entries
    "medium": lambda rng: rng.integers(12, 61, 3000),
    # mixed: short head, long tail (the selector sees the mean)
    "mixed": lambda rng: np.concatenate([rng.integers(0, 4, 4000), rng.integers(20, 80, 800)]),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_spmv_and_prolong_add_bit_identical(V, case):
    import torch
    from paper_2409_14222_b200 import _lib as L
    rng = np.random.default_rng(sum(map(ord, case)))
    lens = CASES[case](rng)
    ncols = 2500
    a = _csr_with_row_lengths(rng, lens, ncols)
    x = rng.standard_normal(ncols)
    x[::17] = -0.0
    d = V.device_csr(a)
    xd = torch.from_numpy(x).cuda()
    # y = A x
    assert np.array_equal(_bits(V.spmv(a, x)), _bits(a @ x))
    # y += P x (prolong-add, mg.py:294-296): y + (P @ x) in one rounding
    y0 = rng.standard_normal(a.shape[0])
    yd = torch.from_numpy(y0.copy()).cuda()
    L.call("vk_spmv", d.handle, L.ptr(xd), L.ptr(yd), 1.0, 1.0, L.stream_ptr())
    assert np.array_equal(_bits(yd.cpu().numpy()), _bits(y0 + a @ x))
    # y = 0.5 * A x + 2 * y
    yd = torch.from_numpy(y0.copy()).cuda()
    L.call("vk_spmv", d.handle, L.ptr(xd), L.ptr(yd), 0.5, 2.0, L.stream_ptr())
    assert np.array_equal(_bits(yd.cpu().numpy()), _bits(2.0 * y0 + 0.5 * (a @ x)))


@pytest.mark.parametrize("case", sorted(CASES))
def test_residual_bit_identical(V, case):
    import torch
    rng = np.random.default_rng(7 + len(case))
    lens = CASES[case](rng)
    n = len(lens)
    a = _csr_with_row_lengths(rng, lens, n)
    b, x = rng.standard_normal(n), rng.standard_normal(n)
    d = V.device_csr(a)
    r = torch.empty(n, dtype=torch.float64, device="cuda")
    d.residual(torch.from_numpy(b).cuda(), torch.from_numpy(x).cuda(), r)
    assert np.array_equal(_bits(r.cpu().numpy()), _bits(b - a @ x))


def test_transpose_restriction_order(V):
    """Restriction through the explicit transpose: entries of each row in
    ascending source-row order = scipy's csc_matvec on masked.T."""
    import torch
    rng = np.random.default_rng(11)
    p = _csr_with_row_lengths(rng, CASES["prolong"](rng), 1800)
    v = rng.standard_normal(p.shape[0])
    d = V.device_csr(p)
    out = d.T.matvec(torch.from_numpy(v).cuda())
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(p.T @ v))
