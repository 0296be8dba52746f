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

One V(nu,nu) cycle (``repeat`` or ``degree`` Chebyshev) is ~15 kernel
launches per level; it is captured once into a CUDA graph and replayed.
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
        self.d = torch.zeros(n, dtype=torch.float64, device="cuda")   # Chebyshev direction

    @property
    def damp(self) -> float:
        return 2.0 / (self.cheb.lower + self.cheb.upper)   # mg.py:268


def pressure_kernel(mixed) -> np.ndarray:
    """Reference ``mg.pressure_kernel`` (``mg.py:170-174``)."""
    vec = np.zeros(mixed.ndof)
    vec[mixed.offset:] = 1.0
    return vec / np.linalg.norm(vec)


def _max_abs(matrix) -> float:
    """max |a_ij| of a host (scipy) or device CSR."""
    import ctypes as C
    if isinstance(matrix, DeviceCSR):
        out = C.c_double()
        L.call("vk_csr_max_abs", matrix.handle, C.byref(out))
        return float(out.value)
    return float(np.max(np.abs(matrix.data)))


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
        shift = _max_abs(c.system.matrix)                               # mg.py:231
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

    def _cycle(self, idx, rhs, x, nu, mode):
        if idx == 0:
            self._coarse_into(rhs, x)
            return
        st = L.stream_ptr()
        lv = self.levels[idx]
        coarse = self.levels[idx - 1]
        if nu > 0:
            _relax_device(lv, rhs, x, nu, mode, x_is_zero=True)
        else:
            x.zero_()
        t = self.transfers[idx]
        if FUSED_TRANSFERS:
            # r = rhs - A x and rc = P^T r in one launch (mg.py:294-295)
            L.call("vk_residual_restrict", lv.A.handle, L.ptr(rhs), L.ptr(x), L.ptr(lv.r),
                   t.PT.handle, L.ptr(coarse.rhs), st)
        else:
            L.call("vk_residual", lv.A.handle, L.ptr(rhs), L.ptr(x), L.ptr(lv.r), st)
            L.call("vk_spmv", t.PT.handle, L.ptr(lv.r), L.ptr(coarse.rhs), 1.0, 0.0, st)
        self._cycle(idx - 1, coarse.rhs, coarse.x, nu, mode)
        if FUSED_TRANSFERS and nu > 0:
            # x += P xc and the first post-smoothing residual in one launch
            L.call("vk_prolong_residual", t.P.handle, L.ptr(coarse.x), L.ptr(x), lv.A.handle,
                   L.ptr(rhs), L.ptr(lv.r), st)
            _relax_device(lv, rhs, x, nu, mode, x_is_zero=False, r_ready=True)
        else:
            L.call("vk_spmv", t.P.handle, L.ptr(coarse.x), L.ptr(x), 1.0, 1.0, st)
            if nu > 0:
                _relax_device(lv, rhs, x, nu, mode, x_is_zero=False)
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
        if mode not in CHEB_MODES:
            raise ValueError(f"unknown chebyshev mode {mode!r}")
        if not graph:
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


# True: the V-cycle's residual + restriction and prolongation + residual
# pairs run as single cooperative launches (vk_residual_restrict /
# vk_prolong_residual, bit-identical to the separate kernels).  Measured on
# the B200 (tools/fused_probe.py) the captured V-cycle is
# 0.5-2% SLOWER fused (cfg2 1.287 vs 1.277 ms, cfg5 2.163 vs 2.117 ms): the
# persistent grid-barrier form of the residual loses more than the launch
# boundary it removes, so the separate launches are the default.
FUSED_TRANSFERS = False


def _relax_device(lv, rhs, x, nu, mode, x_is_zero, r_ready=False):
    """nu relaxation sweeps on one level, all on the device, x updated in place
    (reference ``mg.chebyshev_relax``, ``mg.py:258-271``).

    ``repeat``: nu x {x += damp * apply(rhs - A x)}, damp = 2/(lower+upper),
    the damped update fused into the sweep's epilogue.  ``degree``: the
    preconditioned Chebyshev recurrence of ``chebyshev_iteration``
    (``mg.py:237-255``) — residual kernel, then one fused sweep whose epilogue
    forms d (= z/theta, then rho_next*rho*d + (2 rho_next/delta) z) and
    x + d in the reference's elementwise order; the scalars are the
    reference's Python-float arithmetic.  From x = 0 the first residual is
    rhs itself (b - A 0 = b); ``r_ready``: lv.r already holds rhs - A x."""
    st = L.stream_ptr()
    h = lv.patches.handle
    lower, upper = lv.cheb.lower, lv.cheb.upper
    if mode == "repeat":
        damp = 2.0 / (lower + upper)                                    # mg.py:268
        for it in range(nu):
            if it == 0 and x_is_zero:
                L.call("vk_patches_apply", h, L.ptr(rhs), L.ptr(x), damp, L.VK_APPLY_XSET, None,
                       st)
            else:
                if not (it == 0 and r_ready):
                    L.call("vk_residual", lv.A.handle, L.ptr(rhs), L.ptr(x), L.ptr(lv.r), st)
                L.call("vk_patches_apply", h, L.ptr(lv.r), L.ptr(x), damp, L.VK_APPLY_XADD, None,
                       st)
        return
    if mode != "degree":
        raise ValueError(f"unknown chebyshev mode {mode!r}")
    theta = 0.5 * (upper + lower)                                       # mg.py:241-244
    delta = 0.5 * (upper - lower)
    sigma = theta / delta
    rho = 1.0 / sigma
    if x_is_zero:
        r0 = rhs
    else:
        if not r_ready:
            L.call("vk_residual", lv.A.handle, L.ptr(rhs), L.ptr(x), L.ptr(lv.r), st)
        r0 = lv.r
    L.call("vk_patches_apply_cheb", h, L.ptr(r0), L.ptr(x), L.ptr(lv.d), 0.0, theta,
           2 if x_is_zero else 1, None, st)
    for _ in range(1, nu):
        L.call("vk_residual", lv.A.handle, L.ptr(rhs), L.ptr(x), L.ptr(lv.r), st)
        rho_next = 1.0 / (2.0 * sigma - rho)                            # mg.py:252-254
        L.call("vk_patches_apply_cheb", h, L.ptr(lv.r), L.ptr(x), L.ptr(lv.d), rho_next * rho,
               2.0 * rho_next / delta, 0, None, st)
        rho = rho_next


def chebyshev_iteration(operator, preconditioner, lower, upper, b, x, nu):
    """Degree-nu preconditioned Chebyshev iteration (reference ``mg.py:
    237-255``) for a generic operator / preconditioner (matrices or device
    callables) on device vectors: the residual b - op(x) and the d / x
    recurrence run in the library's kernels (``vk_axpy``, ``vk_cheb_update``,
    elementwise in the reference's order)."""
    import torch
    op = _device_operator(operator)
    prec = _device_operator(preconditioner)
    st = L.stream_ptr()
    theta = 0.5 * (upper + lower)
    delta = 0.5 * (upper - lower)
    sigma = theta / delta
    rho = 1.0 / sigma
    b, host = to_device(b)
    x = to_device(x)[0].clone()
    n = x.numel()
    r = torch.empty_like(x)
    d = torch.empty_like(x)

    def residual():                       # r = b - op(x)
        y = op(x)
        r.copy_(b)
        L.call("vk_axpy", n, -1.0, L.ptr(y), L.ptr(r), st)

    residual()
    L.call("vk_cheb_update", n, L.ptr(prec(r)), L.ptr(d), L.ptr(x), 0.0, theta, 1, st)
    for _ in range(1, nu):
        residual()
        rho_next = 1.0 / (2.0 * sigma - rho)
        L.call("vk_cheb_update", n, L.ptr(prec(r)), L.ptr(d), L.ptr(x), rho_next * rho,
               2.0 * rho_next / delta, 0, st)
        rho = rho_next
    return to_host(x, host)


def chebyshev_relax(level, b, x, nu, mode: str = "degree"):
    """Patch-preconditioned Chebyshev relaxation on one level (reference
    ``mg.chebyshev_relax``, ``mg.py:258-271``); numpy or device vectors."""
    import torch
    if mode not in CHEB_MODES:
        raise ValueError(f"unknown chebyshev mode {mode!r}")
    bd, host = to_device(b)
    xd = to_device(x)[0].clone()
    if not hasattr(level, "A"):
        level = _LevelView(level, bd.numel())
    if nu > 0:
        _relax_device(level, bd, xd, nu, mode, x_is_zero=False)
    return to_host(xd, host)


class _LevelView:
    """Device work vectors for a reference-shaped level object passed to
    :func:`chebyshev_relax` (``system``, ``patches``, ``cheb``)."""

    def __init__(self, level, n):
        import torch
        self.patches = level.patches
        self.cheb = level.cheb
        self.A = device_csr(level.system.matrix)
        self.r = torch.empty(n, dtype=torch.float64, device="cuda")
        self.d = torch.empty(n, dtype=torch.float64, device="cuda")


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
