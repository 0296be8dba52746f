"""Fused V-cycle units and device Chebyshev (degree mode), bit for bit
against their unfused definitions.

* vk_residual_restrict == vk_residual then vk_spmv(P^T)      (mg.py:294-295)
* vk_prolong_residual  == vk_spmv(P, beta=1) then vk_residual (mg.py:296-297)
* the captured V-cycle is bit-identical with and without the fused units,
  in both Chebyshev modes;
* degree-mode relaxation (fused Chebyshev epilogue, vk_patches_apply_cheb)
  equals the reference recurrence mg.py:237-255 written out with separate
  device operations (apply_additive, residual, elementwise torch ops in the
  reference's order).
"""

import numpy as np
import pytest

from conftest import FULL_MG, SMALL_MG, load_case

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("name", SMALL_MG + FULL_MG)
def test_fused_transfer_units_bit_identical(name):
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    pack, _ = load_case(name)
    fine = pack.fine
    A = V.device_csr(fine.system.matrix)
    P = V.device_csr(fine.prolong)
    PT = P.T
    n, nc = P.shape
    rng = np.random.default_rng(4)
    b = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    x = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    xc = torch.from_numpy(rng.uniform(-1, 1, nc)).cuda()
    st = L.stream_ptr()
    r1, rc1 = torch.empty_like(b), torch.empty_like(xc)
    L.call("vk_residual", A.handle, L.ptr(b), L.ptr(x), L.ptr(r1), st)
    L.call("vk_spmv", PT.handle, L.ptr(r1), L.ptr(rc1), 1.0, 0.0, st)
    r2, rc2 = torch.empty_like(b), torch.empty_like(xc)
    L.call("vk_residual_restrict", A.handle, L.ptr(b), L.ptr(x), L.ptr(r2), PT.handle,
           L.ptr(rc2), st)
    assert np.array_equal(_bits(r1), _bits(r2)) and np.array_equal(_bits(rc1), _bits(rc2))
    x1, x2 = x.clone(), x.clone()
    L.call("vk_spmv", P.handle, L.ptr(xc), L.ptr(x1), 1.0, 1.0, st)
    L.call("vk_residual", A.handle, L.ptr(b), L.ptr(x1), L.ptr(r1), st)
    L.call("vk_prolong_residual", P.handle, L.ptr(xc), L.ptr(x2), A.handle, L.ptr(b),
           L.ptr(r2), st)
    assert np.array_equal(_bits(x1), _bits(x2)) and np.array_equal(_bits(r1), _bits(r2))
    # and against scipy (the reference's csr_matvec / csc_matvec order)
    bh, xh, xch = b.cpu().numpy(), x.cpu().numpy(), xc.cpu().numpy()
    a, p = fine.system.matrix, fine.prolong
    assert np.array_equal(x2.cpu().numpy(), xh + p @ xch)
    assert np.array_equal(r2.cpu().numpy(), bh - a @ (xh + p @ xch))
    assert np.array_equal(rc1.cpu().numpy(), p.T @ (bh - a @ xh))


@pytest.mark.parametrize("name", ["s_thtri2", "s_thquad3", "s_bdm3", "cfg2", "cfg5"])
@pytest.mark.parametrize("mode", ["repeat", "degree"])
def test_vcycle_fused_equals_unfused(name, mode):
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import mg
    pack, _ = load_case(name)
    n = pack.fine.system.matrix.shape[0]
    v = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, n)).cuda()
    out = {}
    for fused in (True, False):
        mg.FUSED_TRANSFERS = fused
        try:
            hier = V.hierarchy_from_pack(pack, cheb_mode=mode)
            out[fused] = (hier.vcycle_device(v).clone(), hier.vcycle_device(v, graph=False).clone())
        finally:
            mg.FUSED_TRANSFERS = False
    for a in out[True] + out[False]:
        assert np.array_equal(_bits(a), _bits(out[True][0]))


def _degree_reference(level, b, x, nu):
    """mg.py:237-255 with separate device ops (test-side definition)."""
    import torch
    import paper_2409_14222_b200 as V
    A = level.A
    lower, upper = level.cheb.lower, level.cheb.upper
    theta = 0.5 * (upper + lower)
    delta = 0.5 * (upper - lower)
    sigma = theta / delta
    rho = 1.0 / sigma

    def prec(r):
        return V.apply_additive(level.patches, r)
    r = b - A.matvec(x)
    d = prec(r) / theta
    for step in range(nu):
        x = x + d
        if step == nu - 1:
            break
        r = b - A.matvec(x)
        rho_next = 1.0 / (2.0 * sigma - rho)
        d = rho_next * rho * d + (2.0 * rho_next / delta) * prec(r)
        rho = rho_next
    return x


@pytest.mark.parametrize("name", ["s_thtri2", "s_bdm3", "s_rt2"])
@pytest.mark.parametrize("nu", [1, 2, 3])
def test_degree_relaxation_matches_reference_recurrence(name, nu):
    import torch
    import paper_2409_14222_b200 as V
    pack, _ = load_case(name)
    hier = V.hierarchy_from_pack(pack, cheb_mode="degree")
    lv = hier.fine
    n = lv.n
    rng = np.random.default_rng(6)
    b = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    x0 = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    ref = _degree_reference(lv, b, x0.clone(), nu)
    got = V.chebyshev_relax(lv, b, x0, nu, "degree")
    assert np.array_equal(_bits(got), _bits(ref))
    # generic operator / preconditioner form (chebyshev_iteration)
    prec = lambda r: V.apply_additive(lv.patches, r)  # noqa: E731
    prec._device = True
    it = V.chebyshev_iteration(lv.A, prec, lv.cheb.lower, lv.cheb.upper, b, x0, nu)
    assert np.array_equal(_bits(it), _bits(ref))
    # from a zero guess (the V-cycle's pre-smoothing)
    z = torch.zeros_like(b)
    refz = _degree_reference(lv, b, z.clone(), nu)
    gotz = V.chebyshev_relax(lv, b, z, nu, "degree")
    assert np.allclose(gotz.cpu().numpy(), refz.cpu().numpy(), rtol=0, atol=0)
