"""Device multigrid V-cycle behind the reference ``mg`` API.

Mirrors ``stokesmg.mg`` (reference ``mg.py``): ``TransferPair``,
``ChebyshevParams``, ``Level``, ``MgHierarchy``, ``chebyshev_relax``,
``chebyshev_iteration``, ``coarse_solve``, ``v_cycle``,
``make_preconditioner``, ``pressure_kernel``.

Hierarchy setup (meshes, assembly, prolongation construction) is out of scope
(SURVEY.md §2): :func:`hierarchy_from_pack` takes the assembled operators from
a problem pack, :func:`hierarchy_from_reference` wraps a hierarchy built by
the reference itself.  Everything per level then lives on the device:
operator CSR, masked prolongation and its explicit transpose, factored
patches, work vectors.  The coarse operator A0 + max|A0| q q^T is densified
and inverted once on the device by the library's blocked Gauss-Jordan kernels
(:func:`coarse_inverse`) and applied as a dense GEMV.

One V(nu,nu) cycle in ``repeat`` mode is ~15 kernel launches per level; it is
captured once into a CUDA graph and replayed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .sparsela import (DeviceCSR, device_csr, estimate_lambda_max, to_device, to_host,
                       _device_operator)
from .vanka import apply_additive, build_patches, factor_patches

COARSE_CELLS_PER_SIDE = 5          # reference mg.py:28 (setup is not rebuilt here)
LAMBDA_LOWER_FRACTION = 0.25       # reference mg.py:29
LAMBDA_UPPER_FACTOR = 1.1          # reference mg.py:30
CHEB_MODES = ("degree", "repeat")  # reference mg.py:31


@dataclass
class ChebyshevParams:
    """Reference ``mg.ChebyshevParams`` (``mg.py:48-60``)."""
    lam: float
    steps: int
    seed: int

    @property
    def lower(self) -> float:
        return LAMBDA_LOWER_FRACTION * self.lam

    @property
    def upper(self) -> float:
        return LAMBDA_UPPER_FACTOR * self.lam


@dataclass
class FixedDamping:
    """Pinned spectrum bounds (lower=1, upper=3 -> damp 0.5)."""
    lower: float = 1.0
    upper: float = 3.0
    lam: float | None = None


class TransferPair:
    """Reference ``mg.TransferPair`` (``mg.py:34-45``) on the device:
    prolong = masked @ v, restrict = masked.T @ v (explicit transpose CSR)."""

    def __init__(self, full, masked):
        self.full = full
        self.masked = masked
        self.P = device_csr(masked)
        self.PT = self.P.T

    def prolong(self, coarse_vec):
        return self.P.matvec(coarse_vec)

    def restrict(self, fine_vec):
        return self.PT.matvec(fine_vec)


class Level:
    """Reference ``mg.Level`` (``mg.py:63-69``) plus device state."""

    def __init__(self, mixed, system, patches, cheb):
        import torch
        self.mixed = mixed
        self.system = system
        self.patches = patches
        self.cheb = cheb
        self.A = device_csr(system.matrix)
        n = system.matrix.shape[0]
        self.n = n
        bc = system.bc.indices if system.bc is not None else np.zeros(0, np.int64)
        self.bc = torch.from_numpy(np.ascontiguousarray(bc, dtype=np.int32)).cuda()
        self.x = torch.zeros(n, dtype=torch.float64, device="cuda")
        self.r = torch.zeros(n, dtype=torch.float64, device="cuda")
        self.rhs = torch.zeros(n, dtype=torch.float64, device="cuda")

    @property
    def damp(self) -> float:
        return 2.0 / (self.cheb.lower + self.cheb.upper)   # mg.py:268


def pressure_kernel(mixed) -> np.ndarray:
    """Reference ``mg.pressure_kernel`` (``mg.py:170-174``)."""
    vec = np.zeros(mixed.ndof)
    vec[mixed.offset:] = 1.0
    return vec / np.linalg.norm(vec)


def coarse_inverse(a0, q, shift: float):
    """Explicit inverse of the coarse operator A0 + shift q q^T (reference
    ``mg.build_hierarchy``, ``mg.py:228-232``, which LU-factors it), formed
    and inverted on the device by the library's own kernels
    (``vk_coarse_operator``: bit-identical to numpy's ``a0.toarray() +
    shift * np.outer(q, q)``; ``vk_dense_inverse``: blocked Gauss-Jordan
    with partial pivoting and the ``lu_factor`` guard).  Raises
    ``SingularMatrixError`` like the reference."""
    import ctypes as C
    import torch
    from .sparsela import SingularMatrixError
    n = a0.shape[0]
    st = L.stream_ptr()
    m = torch.empty((n, n), dtype=torch.float64, device="cuda")
    L.call("vk_coarse_operator", a0.handle, L.ptr(q), float(shift), L.ptr(m), st)
    work = torch.empty(max(int(L.lib().vk_dense_inverse_workspace(n)), 1), dtype=torch.uint8,
                       device="cuda")
    inv = torch.empty((n, n), dtype=torch.float64, device="cuda")
    reason, col = C.c_int32(0), C.c_int32(-1)
    rc = L.call("vk_dense_inverse", n, L.ptr(m), L.ptr(inv), L.ptr(work), C.byref(reason),
                C.byref(col), st)
    if rc == L.VK_SINGULAR:
        raise SingularMatrixError("matrix has an all-zero row" if reason.value == L.VK_PATCH_ZERO_ROW
                                  else "pivot below 1e-12 of its row magnitude")
    return inv


class MgHierarchy:
    """Reference ``mg.MgHierarchy`` (``mg.py:72-88``), device resident."""

    def __init__(self, levels, transfers, coarse_kernel, config=None, nu=2, cheb_mode="repeat"):
        import torch
        self.levels = levels
        self.transfers = transfers
        self.coarse_kernel = coarse_kernel
        self.config = config
        self.nu = nu
        self.cheb_mode = cheb_mode
        c = levels[0]
        q = torch.from_numpy(np.ascontiguousarray(coarse_kernel)).cuda()
        shift = float(np.max(np.abs(c.system.matrix.data)))            # mg.py:231
        self.coarse_inverse = coarse_inverse(c.A, q, shift)             # mg.py:232
        self.coarse_factor = self.coarse_inverse
        self.q = q
        self._scratch = L.reduce_scratch()[0]     # this hierarchy's reductions
        self._graphs = {}
        self._in = torch.zeros(levels[-1].n, dtype=torch.float64, device="cuda")

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    @property
    def fine(self) -> Level:
        return self.levels[-1]

    # ------------------------------------------------------------ kernels --
    def _coarse_into(self, rhs, x):
        """x = coarse_solve(rhs) (mg.py:274-279) into preallocated x."""
        st = L.stream_ptr()
        n = rhs.numel()
        c = self.levels[0]
        c.r.copy_(rhs)
        L.call("vk_project", n, L.ptr(self.q), L.ptr(c.r), L.ptr(self._scratch), st)
        L.call("vk_gemv", n, n, L.ptr(self.coarse_inverse), L.ptr(c.r), L.ptr(x), st)
        L.call("vk_project", n, L.ptr(self.q), L.ptr(x), L.ptr(self._scratch), st)

    def _relax_repeat(self, lv: Level, rhs, x, nu, x_is_zero):
        """nu x { x += damp * apply(rhs - A x) } (mg.py:268-271), fused
        epilogues; the first sweep from x = 0 uses r = rhs exactly."""
        st = L.stream_ptr()
        h = lv.patches.handle
        damp = lv.damp
        for it in range(nu):
            if it == 0 and x_is_zero:
                L.call("vk_patches_apply", h, L.ptr(rhs), L.ptr(x), damp, L.VK_APPLY_XSET, None,
                       st)
            else:
                L.call("vk_residual", lv.A.handle, L.ptr(rhs), L.ptr(x), L.ptr(lv.r), st)
                L.call("vk_patches_apply", h, L.ptr(lv.r), L.ptr(x), damp, L.VK_APPLY_XADD, None,
                       st)

    def _cycle(self, idx, rhs, x, nu, mode):
        if idx == 0:
            self._coarse_into(rhs, x)
            return
        st = L.stream_ptr()
        lv = self.levels[idx]
        coarse = self.levels[idx - 1]
        if mode == "repeat":
            if nu > 0:
                self._relax_repeat(lv, rhs, x, nu, True)
            else:
                x.zero_()
        else:
            x.zero_()
            x.copy_(chebyshev_relax(lv, rhs, x, nu, mode))
        L.call("vk_residual", lv.A.handle, L.ptr(rhs), L.ptr(x), L.ptr(lv.r), st)
        t = self.transfers[idx]
        L.call("vk_spmv", t.PT.handle, L.ptr(lv.r), L.ptr(coarse.rhs), 1.0, 0.0, st)
        self._cycle(idx - 1, coarse.rhs, coarse.x, nu, mode)
        L.call("vk_spmv", t.P.handle, L.ptr(coarse.x), L.ptr(x), 1.0, 1.0, st)
        if mode == "repeat":
            self._relax_repeat(lv, rhs, x, nu, False)
        else:
            x.copy_(chebyshev_relax(lv, rhs, x, nu, mode))
        if lv.bc.numel():
            L.call("vk_copy_index", lv.bc.numel(), L.ptr(lv.bc), L.ptr(rhs), L.ptr(x), st)

    def vcycle_device(self, b, nu=None, mode=None, graph=True):
        """One V(nu,nu) cycle of a CUDA vector; returns the level-L x buffer
        (overwritten by the next call)."""
        import torch
        nu = self.nu if nu is None else nu
        mode = self.cheb_mode if mode is None else mode
        top = len(self.levels) - 1
        lv = self.levels[top]
        if top == 0:
            self._in.copy_(b)
            self._coarse_into(self._in, lv.x)
            return lv.x
        if not graph or mode != "repeat":
            self._in.copy_(b)
            self._cycle(top, self._in, lv.x, nu, mode)
            return lv.x
        key = (nu, mode)
        g = self._graphs.get(key)
        if g is None:
            # warm up once eagerly (lazy module loads), then capture
            self._in.copy_(b)
            self._cycle(top, self._in, lv.x, nu, mode)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self._cycle(top, self._in, lv.x, nu, mode)
            torch.cuda.current_stream().wait_stream(s)
            self._graphs[key] = g
        self._in.copy_(b)
        g.replay()
        return lv.x


def chebyshev_iteration(operator, preconditioner, lower, upper, b, x, nu):
    """Degree-nu Chebyshev iteration (reference ``mg.py:237-255``) on device
    vectors (operator / preconditioner: matrices or device callables)."""
    op = _device_operator(operator)
    prec = _device_operator(preconditioner)
    theta = 0.5 * (upper + lower)
    delta = 0.5 * (upper - lower)
    sigma = theta / delta
    rho = 1.0 / sigma
    r = b - op(x)
    d = prec(r) / theta
    for step in range(nu):
        x = x + d
        if step == nu - 1:
            break
        r = b - op(x)
        rho_next = 1.0 / (2.0 * sigma - rho)
        d = rho_next * rho * d + (2.0 * rho_next / delta) * prec(r)
        rho = rho_next
    return x


def _level_precond(level):
    def precond(r):
        return _apply_out(level, r)
    precond._device = True
    return precond


def _apply_out(level, r):
    import torch
    out = torch.empty_like(r)
    L.call("vk_patches_apply", level.patches.handle, L.ptr(r), L.ptr(out), 1.0,
           L.VK_APPLY_OUT, None, L.stream_ptr())
    return out


def chebyshev_relax(level, b, x, nu, mode: str = "degree"):
    """Patch-preconditioned Chebyshev relaxation on one level (reference
    ``mg.chebyshev_relax``, ``mg.py:258-271``); numpy or device vectors."""
    import torch
    bd, host = to_device(b)
    xd = to_device(x)[0].clone()
    lower, upper = level.cheb.lower, level.cheb.upper
    if mode == "degree":
        out = chebyshev_iteration(level.A if hasattr(level, "A") else level.system.matrix,
                                  _level_precond(level), lower, upper, bd, xd, nu)
        return to_host(out, host)
    if mode != "repeat":
        raise ValueError(f"unknown chebyshev mode {mode!r}")
    damp = 2.0 / (lower + upper)
    A = level.A if hasattr(level, "A") else device_csr(level.system.matrix)
    r = torch.empty_like(bd)
    st = L.stream_ptr()
    for _ in range(nu):
        L.call("vk_residual", A.handle, L.ptr(bd), L.ptr(xd), L.ptr(r), st)
        L.call("vk_patches_apply", level.patches.handle, L.ptr(r), L.ptr(xd), damp,
               L.VK_APPLY_XADD, None, st)
    return to_host(xd, host)


def coarse_solve(hier: MgHierarchy, b):
    """Direct coarse solve with the constant-pressure component projected out
    (reference ``mg.coarse_solve``, ``mg.py:274-279``)."""
    import torch
    bd, host = to_device(b)
    x = torch.empty_like(bd)
    rhs = bd.clone()
    hier._coarse_into(rhs, x)
    return to_host(x, host)


def v_cycle(hier: MgHierarchy, b, nu=None, mode=None):
    """One V(nu, nu) cycle from a zero initial guess (reference ``mg.v_cycle``,
    ``mg.py:282-303``)."""
    bd, host = to_device(b)
    out = hier.vcycle_device(bd, nu, mode).clone()
    return to_host(out, host)


def make_preconditioner(hier: MgHierarchy, nu=None, mode=None):
    """Reference ``mg.make_preconditioner`` (``mg.py:306-308``); the returned
    callable is device-aware (CUDA vector in -> CUDA vector out) and also
    accepts numpy."""
    def prec(r):
        import torch
        if isinstance(r, torch.Tensor) and r.is_cuda:
            return hier.vcycle_device(r, nu, mode)
        return v_cycle(hier, r, nu, mode)
    prec._device = True
    # eager (kernel-by-kernel) form, recorded into FGMRES step graphs
    prec._eager = lambda r: hier.vcycle_device(r, nu, mode, graph=False)
    return prec


# ----------------------------------------------------------------------------
# hierarchy construction from prebuilt operators
# ----------------------------------------------------------------------------

def _build(levels_in, nu, weighting, cheb_mode, damping_for, config=None):
    levels = []
    transfers = [None]
    for i, (mixed, system, masked, full) in enumerate(levels_in):
        patches = None
        if i > 0:
            patches = factor_patches(build_patches(mixed, system.bc, weighting), system)
        levels.append(Level(mixed, system, patches, damping_for(i)))
        if i > 0:
            transfers.append(TransferPair(full, masked))
    q = pressure_kernel(levels_in[0][0])
    return MgHierarchy(levels, transfers, q, config, nu=nu, cheb_mode=cheb_mode)


def estimate_spectra(hier: MgHierarchy, *, est_steps: int = 10, seed: int = 0) -> MgHierarchy:
    """Chebyshev bounds of every relaxed level from the patch-preconditioned
    operator, on the device (reference ``mg.build_hierarchy``, ``mg.py:
    214-221``): lam_i = estimate_lambda_max(v -> A_i apply_additive(v),
    m=est_steps, seed=seed + 31 i); ``level.cheb = ChebyshevParams(lam_i,
    est_steps, seed + 31 i)``.  Cached V-cycle graphs are dropped (the
    damping is baked into them)."""
    import torch
    for i, level in enumerate(hier.levels):
        if level.patches is None:
            continue
        tmp = torch.empty(level.n, dtype=torch.float64, device="cuda")

        def op(v, lv=level, t=tmp):
            apply_additive(lv.patches, v, t)
            return lv.A.matvec(t)
        op._device = True
        lam = estimate_lambda_max(op, m=est_steps, seed=seed + 31 * i, n=level.n)
        level.cheb = ChebyshevParams(lam, est_steps, seed + 31 * i)
    hier._graphs = {}
    return hier


def hierarchy_from_pack(pack, *, nu=2, weighting="invmult", cheb_mode="repeat",
                        damping=0.5, est_steps=10, seed=0) -> MgHierarchy:
    """Device hierarchy from a problem pack (assembled operators of every
    level, coarsest first).  ``damping`` pins damp = 2/(lower+upper) like the
    BASELINE recipe (lower=1, upper=2/damping-1); ``damping=None`` keeps the
    reference's own bounds instead, estimated on the device
    (:func:`estimate_spectra`, ``est_steps``/``seed`` as in
    ``mg.build_hierarchy``)."""
    if cheb_mode not in CHEB_MODES:
        raise ValueError(f"unknown chebyshev mode {cheb_mode!r}")
    lv = [(pl.mixed, pl.system, pl.prolong, None) for pl in pack.levels]
    if damping is None:
        hier = _build(lv, nu, weighting, cheb_mode, lambda i: None)
        return estimate_spectra(hier, est_steps=est_steps, seed=seed)
    upper = 2.0 / damping - 1.0
    return _build(lv, nu, weighting, cheb_mode,
                  lambda i: FixedDamping(1.0, upper) if i > 0 else None)


def hierarchy_from_reference(ref_hier, *, weighting="invmult") -> MgHierarchy:
    """Device copy of a hierarchy built by the reference package
    (``stokesmg.mg.build_hierarchy``): same operators, transfers and Chebyshev
    bounds; patches rebuilt and factored on the device."""
    lv = []
    for i, level in enumerate(ref_hier.levels):
        t = ref_hier.transfers[i] if i > 0 else None
        lv.append((level.mixed, level.system, t.masked if t else None, t.full if t else None))
    return _build(lv, ref_hier.nu, weighting, ref_hier.cheb_mode,
                  lambda i: ref_hier.levels[i].cheb, ref_hier.config)
