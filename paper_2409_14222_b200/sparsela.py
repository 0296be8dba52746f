"""Device sparse/dense linear algebra behind the reference ``sparsela`` API.

Mirrors ``stokesmg.sparsela`` (reference ``sparsela.py``) name for name:
``spmv``, ``extract_submatrix``, ``lu_factor``, ``lu_solve``, ``fgmres``,
``estimate_lambda_max``, ``nullspace_projector``, ``SingularMatrixError``,
``DenseFactorization``, ``KrylovReport``.  Every numeric operation runs in the
sm_100a library ``libvanka_b200.so``; inputs may be numpy arrays / scipy
matrices (results come back as numpy) or CUDA ``torch.float64`` tensors /
:class:`DeviceCSR` (results stay on the device).
"""

from __future__ import annotations

import ctypes as C
import time
import weakref
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from . import _lib as L


class SingularMatrixError(Exception):
    """A dense factorization hit a pivot that is numerically zero
    (reference ``sparsela.py:19-20``)."""


@dataclass
class DenseFactorization:
    """Reference ``sparsela.py:23-27``.  The device factorization keeps the
    explicit inverse (``inverse``: CUDA s x s row-major) of the partially
    pivoted LU; ``lu``/``piv`` are not materialised (None)."""
    lu: object
    piv: object
    shape: tuple
    inverse: object = None


@dataclass
class KrylovReport:
    """Reference ``sparsela.py:30-36``."""
    iterations: int
    relative_residual: float
    converged: bool
    history: np.ndarray
    breakdown: bool = False


# ----------------------------------------------------------------------------
# device vectors
# ----------------------------------------------------------------------------

def _torch():
    return L.require_cuda()


def to_device(x):
    """(CUDA float64 tensor, came_from_host)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            t = x if x.dtype == torch.float64 else x.double()
            return t.contiguous(), False
        return x.to(device="cuda", dtype=torch.float64, non_blocking=x.is_pinned()), True
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to("cuda"), True


def to_host(t, host: bool):
    return t.cpu().numpy() if host else t


def _stream():
    return L.stream_ptr()


# ----------------------------------------------------------------------------
# matrices
# ----------------------------------------------------------------------------

class DeviceCSR:
    """scipy-compatible CSR resident on the device (owns a ``vk_csr_t``)."""

    def __init__(self, a=None, *, _handle=None, _shape=None, _nnz=None):
        L.require_cuda()
        if _handle is not None:
            self._h = C.c_void_p(_handle)
            self.shape = _shape
            self.nnz = _nnz
        else:
            a = sp.csr_matrix(a)
            if not a.has_sorted_indices:
                a = a.sorted_indices()
            indptr = np.ascontiguousarray(a.indptr, dtype=np.int32)
            indices = np.ascontiguousarray(a.indices, dtype=np.int32)
            data = np.ascontiguousarray(a.data, dtype=np.float64)
            h = C.c_void_p()
            L.call("vk_csr_create", L.ptr(indptr), L.ptr(indices), L.ptr(data),
                   a.shape[0], a.shape[1], a.nnz, C.byref(h))
            self._h = h
            self.shape = tuple(a.shape)
            self.nnz = int(a.nnz)
        self._finalizer = weakref.finalize(self, _destroy_csr, self._h.value)
        self._t = None

    @property
    def handle(self):
        return self._h

    @property
    def T(self) -> "DeviceCSR":
        """Explicit transpose (restriction = masked.T, reference mg.py:44-45)."""
        if self._t is None:
            h = C.c_void_p()
            L.call("vk_csr_transpose", self._h, C.byref(h))
            self._t = DeviceCSR(_handle=h.value, _shape=(self.shape[1], self.shape[0]),
                                _nnz=self.nnz)
        return self._t

    def matvec(self, x, out=None, alpha=1.0, beta=0.0):
        torch = _torch()
        xd, host = to_device(x)
        if xd.numel() != self.shape[1]:
            raise ValueError(f"dimension mismatch: {self.shape} @ {xd.numel()}")
        y = out if out is not None else torch.empty(self.shape[0], dtype=torch.float64,
                                                    device="cuda")
        L.call("vk_spmv", self._h, L.ptr(xd), L.ptr(y), alpha, beta, _stream())
        return to_host(y, host)

    def residual(self, b, x, out):
        L.call("vk_residual", self._h, L.ptr(b), L.ptr(x), L.ptr(out), _stream())
        return out

    def __matmul__(self, x):
        return self.matvec(x)

    def to_scipy(self):
        """Host scipy copy (bit-exact)."""
        indptr = np.zeros(self.shape[0] + 1, dtype=np.int32)
        indices = np.zeros(self.nnz, dtype=np.int32)
        data = np.zeros(self.nnz, dtype=np.float64)
        L.call("vk_csr_export", self._h, L.ptr(indptr), L.ptr(indices), L.ptr(data))
        return sp.csr_matrix((data, indices, indptr), shape=self.shape)

    def todense_device(self):
        torch = _torch()
        d = torch.empty(self.shape, dtype=torch.float64, device="cuda")
        L.call("vk_csr_to_dense", self._h, L.ptr(d), _stream())
        return d


def _destroy_csr(h):
    try:
        L.lib().vk_csr_destroy(C.c_void_p(h))
    except Exception:  # interpreter teardown
        pass


_CSR_CACHE: dict = {}


def _fingerprint(a):
    """Cheap identity of a host CSR's contents: array addresses, sizes and a
    strided sample of the values/indices (<= 4,096 of each), so an in-place
    change such as ``A.data *= 2`` or a reassigned ``A.data`` is seen."""
    try:
        data, ind, ptr = a.data, a.indices, a.indptr
    except AttributeError:
        return None
    step = max(1, data.size // 4096)
    return (a.shape, data.size, data.ctypes.data, ind.ctypes.data, ptr.ctypes.data,
            hash(data[::step].tobytes()), hash(ind[::step].tobytes()),
            hash(ptr[::max(1, ptr.size // 4096)].tobytes()))


def device_csr(a) -> DeviceCSR:
    """Device copy of a host CSR, cached per host object (the reference
    passes the same scipy matrix to every call) and revalidated by a cheap
    content fingerprint on every lookup: the reference always reads the live
    scipy matrix, so a matrix changed in place gets a fresh device copy."""
    if isinstance(a, DeviceCSR):
        return a
    key = id(a)
    fp = _fingerprint(a)
    hit = _CSR_CACHE.get(key)
    if hit is not None and hit[0]() is a and hit[2] == fp:
        return hit[1]
    d = DeviceCSR(a)
    try:
        ref = weakref.ref(a, lambda _r, k=key: _CSR_CACHE.pop(k, None))
    except TypeError:
        return d
    _CSR_CACHE[key] = (ref, d, fp)
    return d


def spmv(a, x):
    """y = A x (reference ``sparsela.spmv``, ``sparsela.py:45-47``)."""
    return device_csr(a).matvec(x)


def _index_list(v, name):
    arr = np.asarray(v, dtype=np.int64).ravel()
    return arr


def extract_submatrix(a, rows, cols):
    """Dense A[rows, cols] with absent entries zero (reference
    ``sparsela.extract_submatrix``, ``sparsela.py:50-60``): stored values are
    copied bit-exactly by the device gather kernel."""
    rows = _index_list(rows, "rows")
    cols = _index_list(cols, "cols")
    if rows.size == 0 or cols.size == 0:
        return np.zeros((rows.size, cols.size))
    if np.any(rows[:-1] >= rows[1:]) or np.any(cols[:-1] >= cols[1:]):
        raise ValueError("index lists must be sorted and duplicate-free")
    if rows[-1] >= a.shape[0] or cols[-1] >= a.shape[1] or rows[0] < 0 or cols[0] < 0:
        raise ValueError("index out of range")
    torch = _torch()
    d = device_csr(a)
    r = torch.from_numpy(rows.astype(np.int32)).cuda()
    c = torch.from_numpy(cols.astype(np.int32)).cuda()
    out = torch.empty((rows.size, cols.size), dtype=torch.float64, device="cuda")
    L.call("vk_extract", d.handle, L.ptr(r), rows.size, L.ptr(c), cols.size, L.ptr(out),
           _stream())
    return out.cpu().numpy()


# largest block the batched patch kernels take; above it lu_factor uses the
# dense coarse-operator path (same LAPACK pivot order, same guard)
_PATCH_KERNEL_MAX = 128


def _dense_inverse(a: np.ndarray):
    """(explicit inverse on the device, guard status) of a large dense matrix
    by the hand-written blocked LU (``vk_dense_inverse``)."""
    import ctypes as C
    torch = _torch()
    n = a.shape[0]
    m = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    work = torch.empty(max(int(L.lib().vk_dense_inverse_workspace(n)), 1), dtype=torch.uint8,
                       device="cuda")
    inv = torch.empty((n, n), dtype=torch.float64, device="cuda")
    reason, col = C.c_int32(0), C.c_int32(-1)
    rc = L.call("vk_dense_inverse", n, L.ptr(m), L.ptr(inv), L.ptr(work), C.byref(reason),
                C.byref(col), _stream())
    if rc == L.VK_SINGULAR:
        return None, int(reason.value)
    return inv, 0


def lu_factor(a) -> DenseFactorization:
    """Dense factorization with partial pivoting and the reference guard
    (``sparsela.py:63-84``), on the device: one-patch Gauss-Jordan with the
    same pivot order and singularity verdicts; keeps the explicit inverse."""
    from .vanka import _single_block_inverse
    a = np.asarray(a, dtype=float)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("need a square matrix")
    if a.shape[0] == 0:
        return DenseFactorization(None, None, (0, 0), None)
    if a.shape[0] > _PATCH_KERNEL_MAX:
        inv, status = _dense_inverse(a)      # blocked LU + inverse (vk_dense_inverse)
    else:
        inv, status = _single_block_inverse(a)
    if status == L.VK_PATCH_ZERO_ROW:
        raise SingularMatrixError("matrix has an all-zero row")
    if status == L.VK_PATCH_SMALL_PIVOT:
        raise SingularMatrixError("pivot below 1e-12 of its row magnitude")
    return DenseFactorization(None, None, a.shape, inv)


def lu_solve(fact: DenseFactorization, b):
    """Reference ``sparsela.lu_solve`` (``sparsela.py:87-90``)."""
    torch = _torch()
    if fact.shape[0] == 0:
        return np.zeros_like(b) if not isinstance(b, torch.Tensor) else torch.zeros_like(b)
    bd, host = to_device(b)
    y = torch.empty_like(bd)
    L.call("vk_gemv", fact.shape[0], fact.shape[1], L.ptr(fact.inverse), L.ptr(bd), L.ptr(y),
           _stream())
    return to_host(y, host)


def triple_product(p, a, p_right=None):
    """Reference ``sparsela.triple_product`` (``sparsela.py:93-96``) — a
    setup/test helper outside the hot path, kept as the scipy expression."""
    q = p if p_right is None else p_right
    return (p.T @ (a @ q)).tocsr()


# ----------------------------------------------------------------------------
# nullspace projection (reference sparsela.py:99-114)
# ----------------------------------------------------------------------------

class NullspaceProjector:
    """x - Q (Q^T x) with Q from the same numpy QR as the reference."""

    def __init__(self, basis):
        mat = np.column_stack([np.asarray(v, dtype=float) for v in basis])
        q, r = np.linalg.qr(mat)
        if np.min(np.abs(np.diag(r))) < 1e-12 * max(1.0, np.max(np.abs(r))):
            raise ValueError("nullspace basis is linearly dependent")
        self.q = q
        torch = _torch()
        self._qd = [torch.from_numpy(np.ascontiguousarray(q[:, c])).cuda()
                    for c in range(q.shape[1])]
        self._scratch = L.reduce_scratch()[0]

    def apply_(self, xd, scratch=None):
        """In-place projection of a CUDA vector.  ``scratch`` (a
        ``VK_REDUCE_SCRATCH`` device buffer) must be the caller's own when
        projections may run concurrently on several streams."""
        sc = self._scratch if scratch is None else scratch
        for qc in self._qd:
            L.call("vk_project", xd.numel(), L.ptr(qc), L.ptr(xd), L.ptr(sc), _stream())
        return xd

    def __call__(self, x):
        xd, host = to_device(x)
        xd = xd.clone()
        return to_host(self.apply_(xd), host)


def nullspace_projector(basis) -> NullspaceProjector:
    return NullspaceProjector(basis)


# ----------------------------------------------------------------------------
# flexible GMRES (reference sparsela.py:117-191), device vectors
# ----------------------------------------------------------------------------

def _device_operator(a):
    """Operator on CUDA vectors: DeviceCSR / host CSR -> device SpMV; a
    callable is used as is when it is device-aware (``_device``), else it is
    fed numpy (host callables such as hand-written preconditioners)."""
    torch = _torch()
    if a is None:
        return None
    if callable(a) and not isinstance(a, (DeviceCSR, sp.spmatrix)) and not sp.issparse(a):
        if getattr(a, "_device", False):
            return a

        def host_op(v, f=a):
            out = f(v.cpu().numpy())
            return torch.as_tensor(np.asarray(out, dtype=np.float64), device="cuda")
        host_op._host = True
        return host_op
    d = device_csr(a)

    def op(v, out=None):
        y = out if out is not None else torch.empty(d.shape[0], dtype=torch.float64,
                                                    device="cuda")
        L.call("vk_spmv", d.handle, L.ptr(v), L.ptr(y), 1.0, 0.0, _stream())
        return y
    return op


class FgmresWorkspace:
    """Persistent Krylov buffers + one captured CUDA graph per Arnoldi step.

    With a workspace, step j of :func:`fgmres` — preconditioner (V-cycle
    kernels recorded eagerly into the graph), SpMV, nullspace projection,
    the j+1 MGS dot/axpy pairs, the norm and the normalisation — is captured
    once and replayed as a single graph launch; the host still performs the
    Givens update in the reference's scalar arithmetic after one D2H read."""

    def __init__(self, n: int, max_it: int):
        torch = _torch()
        self.n, self.max_it = n, max_it
        self.vmat = torch.zeros((max_it + 1, n), dtype=torch.float64, device="cuda")
        self.zmat = torch.zeros((max_it, n), dtype=torch.float64, device="cuda")
        self.w = torch.empty(n, dtype=torch.float64, device="cuda")
        self.scal = torch.zeros(max_it + 3, dtype=torch.float64, device="cuda")
        self.red = L.reduce_scratch()[0]      # this workspace's reduction scratch
        self.graphs = {}
        self._key = None

    def fits(self, n, max_it):
        return n == self.n and max_it == self.max_it

    @staticmethod
    def capturable(op, prec, proj):
        return (prec is None or hasattr(prec, "_eager")) and not hasattr(op, "_host") and \
            getattr(proj, "_device", True)

    def replay(self, j, step, prec):
        torch = _torch()
        key = (id(prec),)
        if key != self._key:             # a different preconditioner: recapture
            self.graphs.clear()
            self._key = key
        g = self.graphs.get(j)
        if g is None:
            eager = prec._eager if prec is not None else None
            step(j, eager)               # warm-up run (also this step's result)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):   # records only; step j already ran
                    step(j, eager)
            torch.cuda.current_stream().wait_stream(s)
            self.graphs[j] = g
            return
        g.replay()


# tools/fgmres_profile.py sets this to a dict to collect per-iteration host
# timings (graph launch call, wait for the Hessenberg column, Givens update)
FGMRES_PROFILE = None


def fgmres(a, b, *, preconditioner=None, rtol: float = 1e-10, max_it: int = 100,
           nullspace=None, x0=None, target_norm=None, workspace: FgmresWorkspace | None = None):
    """Unrestarted flexible GMRES (reference ``sparsela.fgmres``,
    ``sparsela.py:117-191``).  Krylov/direction vectors, SpMVs, dot products,
    MGS updates and the final combination run on the device; only the
    Hessenberg column (j+2 scalars) crosses to the host once per iteration for
    the Givens update, in exactly the reference's scalar arithmetic.  With a
    :class:`FgmresWorkspace` each Arnoldi step is one CUDA-graph replay."""
    torch = _torch()
    op = _device_operator(a)
    prec = _device_operator(preconditioner) if preconditioner is not None else None
    ws = workspace
    # reduction scratch owned by this solve (or its workspace): solves running
    # concurrently on different streams never share reduction state
    red = ws.red if ws is not None else L.reduce_scratch()[0]
    if nullspace is not None and not isinstance(nullspace, NullspaceProjector):
        proj_host = nullspace

        def proj(v):
            v.copy_(torch.as_tensor(proj_host(v.cpu().numpy()), device="cuda"))
            return v
        proj._device = False
    elif nullspace is not None:
        def proj(v, _ns=nullspace):
            return _ns.apply_(v, red)
    else:
        def proj(v):
            return v
    bd, host = to_device(b)
    n = bd.numel()
    st = _stream()
    b_ = proj(bd.clone())
    x = torch.zeros(n, dtype=torch.float64, device="cuda") if x0 is None \
        else to_device(x0)[0].clone()
    scal = torch.zeros(max_it + 3, dtype=torch.float64, device="cuda")
    if x0 is not None:
        r = b_ - op(x)
        proj(r)
    else:
        r = b_.clone()
    L.call("vk_nrm2", n, L.ptr(r), L.ptr(scal[max_it + 2:]), L.ptr(red), st)
    beta = float(scal[max_it + 2].item())
    base = float(target_norm) if target_norm is not None else beta
    if base == 0.0:
        return to_host(x, host), KrylovReport(0, 0.0, True, np.zeros(1))
    history = [beta / base]
    if beta <= rtol * base:
        return to_host(x, host), KrylovReport(0, history[0], True, np.array(history))

    ws = workspace if (workspace is not None and workspace.fits(n, max_it)) else None
    if ws is None and workspace is not None:
        red = red.clone()            # a mismatched workspace keeps nothing shared
    if ws is not None:
        vmat, zmat, w = ws.vmat, ws.zmat, ws.w
        ws.scal[max_it + 2:max_it + 3].copy_(scal[max_it + 2:max_it + 3])
        scal = ws.scal
    else:
        vmat = torch.zeros((max_it + 1, n), dtype=torch.float64, device="cuda")
        zmat = torch.zeros((max_it, n), dtype=torch.float64, device="cuda")
        w = torch.empty(n, dtype=torch.float64, device="cuda")
    hess = np.zeros((max_it + 1, max_it))
    cs = np.zeros(max_it)
    sn = np.zeros(max_it)
    g = np.zeros(max_it + 1)
    g[0] = beta
    L.call("vk_div_dev", n, L.ptr(r), L.ptr(scal[max_it + 2:]), L.ptr(vmat[0]), st)

    def arnoldi_step(j, eager_prec):
        s_ = _stream()
        if prec is not None:
            z = eager_prec(vmat[j])
            zmat[j].copy_(z)
        else:
            zmat[j].copy_(vmat[j])
        wz = op(zmat[j])
        w.copy_(wz)
        proj(w)
        L.call("vk_nrm2", n, L.ptr(w), L.ptr(scal[max_it + 1:]), L.ptr(red), s_)  # wnorm0
        # MGS (sparsela.py:160-163): h_0 = v_0.w, then for each i the update
        # w -= h_i v_i fused with the next dot (v_{i+1}.w, or ||w|| after the
        # last one) -- bit-identical to separate dot / axpy / nrm2 kernels
        L.call("vk_dot", n, L.ptr(vmat[0]), L.ptr(w), L.ptr(scal[0:]), L.ptr(red), s_)
        for i in range(j + 1):
            if i < j:
                L.call("vk_axpy_dot", n, L.ptr(scal[i:]), L.ptr(vmat[i]), L.ptr(w),
                       L.ptr(vmat[i + 1]), L.ptr(scal[i + 1:]), 0, L.ptr(red), s_)
            else:
                L.call("vk_axpy_dot", n, L.ptr(scal[i:]), L.ptr(vmat[i]), L.ptr(w),
                       L.ptr(w), L.ptr(scal[j + 1:]), 1, L.ptr(red), s_)
        L.call("vk_div_dev", n, L.ptr(w), L.ptr(scal[j + 1:]), L.ptr(vmat[j + 1]), s_)

    converged = False
    breakdown = False
    j = 0
    prof = FGMRES_PROFILE
    for j in range(max_it):
        if prof is not None:
            t0 = time.perf_counter()
        if ws is not None and ws.capturable(op, prec, proj):
            ws.replay(j, arnoldi_step, prec)       # one CUDA graph per Arnoldi step
        else:
            arnoldi_step(j, prec)
        if prof is not None:
            t1 = time.perf_counter()
        hs = scal.cpu().numpy()                                           # 1 sync
        if prof is not None:
            t2 = time.perf_counter()
        hess[:j + 2, j] = hs[:j + 2]
        wnorm0 = hs[max_it + 1]
        if hess[j + 1, j] <= 1e-14 * max(1.0, wnorm0):
            breakdown = True
        for i in range(j):
            t = cs[i] * hess[i, j] + sn[i] * hess[i + 1, j]
            hess[i + 1, j] = -sn[i] * hess[i, j] + cs[i] * hess[i + 1, j]
            hess[i, j] = t
        denom = np.hypot(hess[j, j], hess[j + 1, j])
        cs[j] = hess[j, j] / denom
        sn[j] = hess[j + 1, j] / denom
        hess[j, j] = denom
        hess[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        res = abs(g[j + 1])
        history.append(res / base)
        if prof is not None:
            t3 = time.perf_counter()
            prof.setdefault("launch_s", []).append(t1 - t0)
            prof.setdefault("sync_s", []).append(t2 - t1)
            prof.setdefault("host_s", []).append(t3 - t2)
        if breakdown or res <= rtol * base:
            converged = True
            break

    its = j + 1
    y = scipy.linalg.solve_triangular(hess[:its, :its], g[:its], check_finite=False)
    yd = torch.from_numpy(np.ascontiguousarray(y)).cuda()
    L.call("vk_combine", n, its, L.ptr(zmat), L.ptr(yd), L.ptr(x), st)
    proj(x)
    return to_host(x, host), KrylovReport(its, history[-1], converged, np.array(history),
                                          breakdown)


def estimate_lambda_max(a, *, m: int = 10, seed: int = 0, preconditioner=None,
                        n: int | None = None) -> float:
    """Largest |Ritz value| of the right-preconditioned operator (reference
    ``sparsela.estimate_lambda_max``, ``sparsela.py:194-226``): Arnoldi on
    the device, eigenvalues of the m x m Hessenberg on the host."""
    torch = _torch()
    if m < 1:
        raise ValueError("need at least one Arnoldi step")
    op = _device_operator(a)
    prec = _device_operator(preconditioner) if preconditioner is not None else None
    if n is None:
        n = a.shape[0]
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    st = _stream()
    vmat = torch.zeros((m + 1, n), dtype=torch.float64, device="cuda")
    vmat[0].copy_(torch.from_numpy(v))
    scal = torch.zeros(m + 2, dtype=torch.float64, device="cuda")
    red = L.reduce_scratch()[0]
    hess = np.zeros((m + 1, m))
    used = 0
    for j in range(m):
        z = prec(vmat[j]) if prec is not None else vmat[j]
        w = op(z).clone()
        for i in range(j + 1):
            L.call("vk_dot", n, L.ptr(vmat[i]), L.ptr(w), L.ptr(scal[i:]), L.ptr(red), st)
            L.call("vk_axpy_dev", n, L.ptr(scal[i:]), L.ptr(vmat[i]), L.ptr(w), st)
        L.call("vk_nrm2", n, L.ptr(w), L.ptr(scal[j + 1:]), L.ptr(red), st)
        hs = scal.cpu().numpy()
        hess[:j + 2, j] = hs[:j + 2]
        used = j + 1
        if hess[j + 1, j] <= 1e-14:
            break
        L.call("vk_div_dev", n, L.ptr(w), L.ptr(scal[j + 1:]), L.ptr(vmat[j + 1]), st)
    eigs = np.linalg.eigvals(hess[:used, :used])
    return float(np.max(np.abs(eigs)))
