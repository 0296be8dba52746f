"""MG-preconditioned FGMRES(restart) driver (the timed TTS window).

Mirrors how the reference drives a solve (``bench.run_case``,
``bench.py:174-191``; warm restarts as in ``bench.stopping_study``,
``bench.py:261-274``): ``fgmres(A, b, preconditioner=make_preconditioner(hier),
nullspace=P, rtol, max_it=restart, x0, target_norm)`` repeated until
converged, everything device resident.
"""

from __future__ import annotations

import numpy as np

from . import _lib as L
from .mg import MgHierarchy, make_preconditioner, pressure_kernel
from .sparsela import FgmresWorkspace, fgmres, nullspace_projector, to_device


def mg_rhs(pack) -> np.ndarray:
    """BASELINE.md §3 forcing: b_u ~ U[-1,1] (seed 0) on the velocity block,
    zero on constrained rows and on the pressure block."""
    fine = pack.fine
    n = fine.system.matrix.shape[0]
    nvel = fine.mixed.velocity.ndof
    b = np.zeros(n)
    b[:nvel] = np.random.default_rng(0).uniform(-1.0, 1.0, nvel)
    b[np.asarray(fine.system.bc.indices)] = 0.0
    return b


class FgmresSolver:
    """Reusable solver state (device operator, preconditioner, projector)."""

    def __init__(self, hier: MgHierarchy, *, rtol=1e-8, restart=30, max_cycles=20):
        import torch
        self.hier = hier
        self.rtol = rtol
        self.restart = restart
        self.max_cycles = max_cycles
        self.prec = make_preconditioner(hier)
        self.nsp = nullspace_projector([pressure_kernel(hier.fine.mixed)])
        self.A = hier.fine.A
        self.workspace = FgmresWorkspace(hier.fine.n, restart)
        self._red = L.reduce_scratch()[0]
        self._norm = torch.zeros(1, dtype=torch.float64, device="cuda")

    def solve(self, b):
        """Returns (x, iterations, converged, history) with x on the device
        when b is a CUDA tensor, else numpy."""
        import torch
        bd, host = to_device(b)
        x = None
        base = None
        hist = []
        its = 0
        conv = False
        for _ in range(self.max_cycles):
            x, rep = fgmres(self.A, bd, preconditioner=self.prec, rtol=self.rtol,
                            max_it=self.restart, nullspace=self.nsp, x0=x, target_norm=base,
                            workspace=self.workspace)
            if base is None:
                pb = self.nsp(bd.clone())
                if rep.iterations:
                    L.call("vk_nrm2", pb.numel(), L.ptr(pb), L.ptr(self._norm),
                           L.ptr(self._red), L.stream_ptr())
                    base = float(self._norm.item())
                else:
                    base = None
                hist.extend(rep.history.tolist())
                if base is None:
                    conv = rep.converged
                    break
            else:
                hist.extend(rep.history[1:].tolist())
            its += rep.iterations
            if rep.converged:
                conv = True
                break
        return (x.cpu().numpy() if host else x), its, conv, np.array(hist)
