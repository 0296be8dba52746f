"""Where does the FGMRES history difference come from?

The device MG-FGMRES is run twice on the same case:

* as shipped: every kernel on the device, coarse solve = the device
  LU-based explicit inverse (``vk_dense_inverse``) applied by a GEMV;
* with ONE change: the coarse solve (reference ``mg.py:274-279``) replaced
  by the reference's own LAPACK ``getrf``/``getrs`` path — the oracle's
  ``coarse_solve``, bit-identical to the reference when its BLAS runs on one
  thread — called from the device V-cycle through a host round trip
  (test-only instrumentation; the V-cycle is not graph-captured here).

If the second run meets the strict 1e-10 per-entry history gate while the
first does not, the whole remaining difference is the coarse solve — and
there, two valid factorizations of A0 + shift q q^T already differ by about
cond(A0) * eps, which moves the reference's own history by the recorded
floor (tools/reference_selfvar.py, tests/golden/reference_selfvar.json).
"""

import numpy as np
import pytest

from conftest import FULL_MG, SMALL_MG, load_case

pytestmark = pytest.mark.gpu


def _history_rel(h, href):
    m = min(len(h), len(href))
    return float(np.max(np.abs(h[:m] - href[:m]) / href[:m]))


def _solve(hier, pack, workspace):
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.solver import mg_rhs
    b = mg_rhs(pack)
    nsp = V.nullspace_projector([V.pressure_kernel(pack.fine.mixed)])
    if workspace:
        from paper_2409_14222_b200.solver import FgmresSolver
        _, its, conv, hist = FgmresSolver(hier).solve(b)
        return its, hist

    def prec(v):          # device V-cycle, kernel by kernel (no graph capture)
        return hier.vcycle_device(v, graph=False)
    prec._device = True
    x, base, hist, its = None, None, [], 0
    for _ in range(20):
        x, rep = V.fgmres(hier.fine.A, b, preconditioner=prec, rtol=1e-8, max_it=30,
                          nullspace=nsp, x0=x, target_norm=base)
        if base is None:
            base = float(np.linalg.norm(nsp(b.copy())))
            hist.extend(rep.history.tolist())
        else:
            hist.extend(rep.history[1:].tolist())
        its += rep.iterations
        if rep.converged:
            break
    return its, np.array(hist)


def _swap_in_reference_coarse_solve(hier, pack):
    """hier's coarse solve -> the oracle's LAPACK path (one BLAS thread)."""
    import torch
    from threadpoolctl import threadpool_limits
    from oracle import vanka_oracle as O
    c = pack.levels[0]
    q = O.pressure_kernel(c.mixed)
    a0 = c.system.matrix
    with threadpool_limits(1):
        fac = O.lu_factor(a0.toarray() + np.max(np.abs(a0.data)) * np.outer(q, q))
    oh = type("H", (), {"coarse_kernel": q, "coarse_factor": fac})()

    def coarse_into(rhs, x):
        with threadpool_limits(1):
            xs = O.coarse_solve(oh, rhs.cpu().numpy())
        x.copy_(torch.from_numpy(xs))
    hier._coarse_into = coarse_into
    return oh


@pytest.mark.parametrize("name", ["s_bdm3", "s_rt2", "s_thtri4", "cfg3", "cfg5"])
def test_history_gap_is_the_coarse_solve(name, capsys):
    import paper_2409_14222_b200 as V
    from threadpoolctl import threadpool_limits
    from oracle import vanka_oracle as O
    pack, g = load_case(name)
    href = np.asarray(g["history"])
    its_dev, h_dev = _solve(V.hierarchy_from_pack(pack), pack, workspace=True)
    hier = V.hierarchy_from_pack(pack)
    oh = _swap_in_reference_coarse_solve(hier, pack)
    # is this host's LAPACK the reference's?  (the goldens were made elsewhere)
    n0 = pack.levels[0].system.matrix.shape[0]
    rc = np.random.default_rng(2).uniform(-1.0, 1.0, n0)
    with threadpool_limits(1):
        host_same = np.array_equal(O.coarse_solve(oh, rc), g["coarse_x"])
    its_ref, h_ref = _solve(hier, pack, workspace=False)
    rel_dev = _history_rel(h_dev, href)
    rel_ref = _history_rel(h_ref, href)
    with capsys.disabled():
        print(f"\n[{name}] history max rel: device coarse solve {rel_dev:.3e} "
              f"(its {its_dev}); reference coarse solve swapped in {rel_ref:.3e} "
              f"(its {its_ref}); host LAPACK reproduces the golden coarse solve: {host_same}")
    assert its_ref == int(g["iterations"])
    if host_same:
        # with the reference's own coarse solve swapped in, the device path is
        # inside the strict gate (or, on the hypersensitive P4 16^2 case, at
        # least 100x below the reference's own coarse-solve floor): everything
        # else (sweeps, SpMVs, transfers, MGS) agrees with the reference
        from test_gpu_parity import history_floor
        assert rel_ref <= max(1e-10, 0.01 * history_floor(name)), rel_ref
