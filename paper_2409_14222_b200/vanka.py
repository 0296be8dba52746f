"""Device Vanka patches behind the reference ``vanka`` API.

Mirrors ``stokesmg.vanka`` (reference ``vanka.py``): ``Patch``, ``PatchSet``,
``build_patches_taylor_hood``, ``build_patches_hdiv_extended``,
``build_patches``, ``factor_patches``, ``apply_additive``.

* patch DoF lists, multiplicities and weights are built on the device (K1)
  from the cell-to-DoF map and the topology's entity->cell incidence; the
  host only flattens the incidence lists into CSR form;
* ``factor_patches`` extracts every patch block from the device CSR and
  inverts it in one batched launch per size class (K2+K3);
* ``apply_additive`` is the fused gather / dense solve / weighted
  partition-of-unity accumulation (K4), deterministic and atomic-free.

Inputs are duck-typed: the reference's own ``MixedSpace``/``StrongBc``/
``BlockSystem`` objects, or the light pack objects of ``pack.py``.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .sparsela import SingularMatrixError, device_csr, to_device, to_host, DeviceCSR

WEIGHTINGS = ("invmult", "unit")


@dataclass(frozen=True, order=True)
class EntityRef:
    """Reference ``meshtopo.EntityRef`` (``meshtopo.py:27-32``)."""
    dim: int
    index: int


@dataclass
class Patch:
    """Reference ``vanka.Patch`` (``vanka.py:28-34``)."""
    entity: object
    indices: np.ndarray
    num_velocity: int
    weights: np.ndarray | None = None
    factor: object = None


class PatchSet:
    """Reference ``vanka.PatchSet`` (``vanka.py:37-46``), device resident.

    Built by :func:`build_patches` (device K1) or, like the reference, from a
    list of :class:`Patch` objects; ``patches`` and ``multiplicity`` are
    exported from the device lazily."""

    def __init__(self, patches=None, size=None, multiplicity=None, weighting="invmult", *,
                 _handle=None, _entities=None):
        self.size = int(size)
        self.weighting = weighting
        self._patches = patches
        self._mult = None if multiplicity is None else np.asarray(multiplicity, dtype=float)
        self._entities = _entities
        self._h = None
        self._fin = None
        self.factored = False
        if _handle is not None:
            self._set_handle(_handle)

    # -- handle management --------------------------------------------------
    def _set_handle(self, h):
        self._h = C.c_void_p(h)
        self._fin = weakref.finalize(self, _destroy_patches, h)
        npatch, total, smax = C.c_int32(), C.c_int64(), C.c_int32()
        L.call("vk_patches_info", self._h, C.byref(npatch), C.byref(total), C.byref(smax))
        self._npatch, self._total, self.max_size = npatch.value, total.value, smax.value

    @property
    def handle(self):
        if self._h is None:
            self._upload_lists()
        return self._h

    def _upload_lists(self):
        """Device copy of hand-built patches (reference tests build PatchSet
        from Patch objects, tests/test_vanka.py:134-168)."""
        L.require_cuda()
        ps = self._patches
        offs = np.zeros(len(ps) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(p.indices) for p in ps])
        idx = np.ascontiguousarray(np.concatenate([np.asarray(p.indices) for p in ps])
                                   if ps else np.zeros(0), dtype=np.int32)
        nv = np.array([p.num_velocity for p in ps], dtype=np.int32)
        w = np.ascontiguousarray(np.concatenate(
            [np.ones(len(p.indices)) if p.weights is None else np.asarray(p.weights, float)
             for p in ps]) if ps else np.zeros(0), dtype=np.float64)
        h = C.c_void_p()
        L.call("vk_patches_from_lists", L.ptr(offs), L.ptr(idx), L.ptr(nv), L.ptr(w),
               len(ps), self.size, C.byref(h))
        self._set_handle(h.value)

    # -- reference attributes -------------------------------------------------
    @property
    def zbuf_size(self) -> int:
        """Entries of a caller-owned correction buffer for :func:`apply_additive`."""
        self.handle
        return max(int(self._total), 1)

    def new_zbuf(self):
        import torch
        return torch.empty(self.zbuf_size, dtype=torch.float64, device="cuda")

    @property
    def num_patches(self) -> int:
        if self._patches is not None:
            return len(self._patches)
        return self._npatch

    def export(self) -> dict:
        """Bit-exact host copy of the device patch arrays."""
        h = self.handle
        n, t = self._npatch, self._total
        offs = np.zeros(n + 1, dtype=np.int64)
        idx = np.zeros(t, dtype=np.int32)
        nv = np.zeros(n, dtype=np.int32)
        w = np.zeros(t, dtype=np.float64)
        mult = np.zeros(self.size, dtype=np.float64)
        cand = np.zeros(n, dtype=np.int32)
        L.call("vk_patches_export", h, L.ptr(offs), L.ptr(idx), L.ptr(nv), L.ptr(w),
               L.ptr(mult), L.ptr(cand))
        return {"offsets": offs, "indices": idx, "num_velocity": nv, "weights": w,
                "multiplicity": mult, "candidate": cand}

    @property
    def multiplicity(self) -> np.ndarray:
        if self._mult is None:
            self._mult = self.export()["multiplicity"]
        return self._mult

    @property
    def patches(self) -> list:
        if self._patches is None:
            ex = self.export()
            ents = self._entities
            out = []
            for p in range(self._npatch):
                a, b = ex["offsets"][p], ex["offsets"][p + 1]
                ent = ents[ex["candidate"][p]] if ents is not None else None
                out.append(Patch(ent, ex["indices"][a:b].astype(np.int64),
                                 int(ex["num_velocity"][p]), ex["weights"][a:b]))
            self._patches = out
        return self._patches

    def entity_of(self, p: int):
        """Entity of kept patch ``p`` (device patch index; size-0 input
        patches are dropped on the device, ``candidate`` maps back)."""
        cand = self.export()["candidate"]
        if self._entities is None:
            return self.patches[int(cand[p])].entity
        return self._entities[cand[p]]


def _destroy_patches(h):
    try:
        L.lib().vk_patches_destroy(C.c_void_p(h))
    except Exception:
        pass


# ----------------------------------------------------------------------------
# construction (reference vanka.py:49-126)
# ----------------------------------------------------------------------------

def _ragged_csr(lists):
    if hasattr(lists, "ptr") and hasattr(lists, "idx"):
        return np.asarray(lists.ptr, np.int32), np.asarray(lists.idx, np.int32)
    lens = np.fromiter((len(x) for x in lists), dtype=np.int64, count=len(lists))
    ptr = np.zeros(len(lists) + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    idx = np.fromiter((v for x in lists for v in x), dtype=np.int64, count=int(ptr[-1]))
    return ptr.astype(np.int32), idx.astype(np.int32)


def _topology_csr(topo, name):
    ptr_name, idx_name = f"{name}_ptr", f"{name}_idx"
    if hasattr(topo, ptr_name):
        return np.asarray(getattr(topo, ptr_name), np.int32), \
            np.asarray(getattr(topo, idx_name), np.int32)
    cache = topo.__dict__.setdefault("_vk_csr_cache", {}) if hasattr(topo, "__dict__") else {}
    if name not in cache:
        cache[name] = _ragged_csr(getattr(topo, name))
    return cache[name]


def _constrained_mask(ndof, bc):
    mask = np.zeros(ndof, dtype=np.uint8)
    if bc is not None:
        mask[np.asarray(bc.indices, dtype=np.int64)] = 1
    return mask


def _launch_build(mixed, bc, weighting, e2c_ptr, e2c, pptr, pdofs, entities):
    if weighting not in WEIGHTINGS:
        raise ValueError(f"unknown weighting {weighting!r}")
    L.require_cuda()
    vel = mixed.velocity
    cd = np.ascontiguousarray(vel.cell_dofs, dtype=np.int32)
    ndof = int(mixed.ndof)
    h = C.c_void_p()
    con = _constrained_mask(ndof, bc)
    L.call("vk_patches_build", L.ptr(cd), cd.shape[0], cd.shape[1],
           L.ptr(np.ascontiguousarray(e2c_ptr, np.int32)), L.ptr(np.ascontiguousarray(e2c, np.int32)),
           len(e2c_ptr) - 1, L.ptr(np.ascontiguousarray(pptr, np.int32)),
           L.ptr(np.ascontiguousarray(pdofs, np.int32)), L.ptr(con), ndof,
           L.VK_WEIGHT_INVMULT if weighting == "invmult" else L.VK_WEIGHT_UNIT, C.byref(h))
    return PatchSet(None, ndof, None, weighting, _handle=h.value, _entities=entities)


class _Entities:
    """Lazy (dim, index) list for candidate patches."""

    def __init__(self, blocks):
        self.blocks = blocks          # list of (dim, count)
        self.starts = np.cumsum([0] + [c for _, c in blocks])

    def __getitem__(self, k):
        k = int(k)
        b = int(np.searchsorted(self.starts, k, side="right") - 1)
        return EntityRef(self.blocks[b][0], k - int(self.starts[b]))

    def __len__(self):
        return int(self.starts[-1])


def taylor_hood_candidates(mixed):
    """Host flattening for :func:`build_patches_taylor_hood`: candidate patch
    p = entity (dim, index) in reference order (``vanka.py:87-95``); its cells
    are star(entity)'s cells (vertex_cells / edge_cells / the cell), its
    pressure DoFs ``pres.entity_dofs[dim][ent] + offset``.  Pure numpy."""
    vel, pres = mixed.velocity, mixed.pressure
    topo = vel.mesh.topology
    off = int(mixed.offset)
    ptrs, idxs, pptrs, pds, blocks = [], [], [], [], []
    base_c, base_p = 0, 0
    for dim in range(3):
        ed = np.asarray(pres.entity_dofs[dim])
        if ed.shape[1] == 0:
            continue
        count = topo.entity_count(dim)
        if dim == 0:
            p, i = _topology_csr(topo, "vertex_cells")
        elif dim == 1:
            p, i = _topology_csr(topo, "edge_cells")
        else:
            p, i = np.arange(count + 1, dtype=np.int32), np.arange(count, dtype=np.int32)
        ptrs.append(p[:-1].astype(np.int64) + base_c)
        idxs.append(i)
        base_c += int(p[-1])
        pptrs.append(np.arange(count, dtype=np.int64) * ed.shape[1] + base_p)
        pds.append((ed + off).ravel())
        base_p += ed.size
        blocks.append((dim, count))
    e2c_ptr = np.concatenate(ptrs + [[base_c]]).astype(np.int32)
    pptr = np.concatenate(pptrs + [[base_p]]).astype(np.int32)
    e2c = np.concatenate(idxs).astype(np.int32) if idxs else np.zeros(0, np.int32)
    pdofs = np.concatenate(pds).astype(np.int32) if pds else np.zeros(0, np.int32)
    return e2c_ptr, e2c, pptr, pdofs, _Entities(blocks)


def build_patches_taylor_hood(mixed, bc=None, weighting: str = "invmult") -> PatchSet:
    """One patch per pressure-carrying entity (reference ``vanka.py:77-96``):
    velocity = DoFs of the cells in star(entity) minus constrained, pressure =
    the entity's pressure DoFs, entities in (dim, index) order."""
    if mixed.case not in ("th-tri", "th-quad"):
        raise ValueError("entity patches are for the continuous pairs")
    return _launch_build(mixed, bc, weighting, *taylor_hood_candidates(mixed))


def hdiv_candidates(mixed):
    """Host flattening for :func:`build_patches_hdiv_extended`: one candidate
    per cell with cells = {c} U edge neighbours (``vanka.py:111-118``),
    pressure = the cell's DoFs + offset.  Pure numpy."""
    vel, pres = mixed.velocity, mixed.pressure
    topo = vel.mesh.topology
    nc = topo.num_cells
    ep, ei = _topology_csr(topo, "edge_cells")
    ce = np.asarray(topo.cell_edges, dtype=np.int64)
    lens = np.diff(ep)
    ec2 = np.full((len(lens), 2), -1, dtype=np.int64)
    has1 = lens > 0
    ec2[has1, 0] = ei[ep[:-1][has1]]
    has2 = lens > 1
    ec2[has2, 1] = ei[ep[:-1][has2] + 1]
    cand = np.concatenate([np.arange(nc)[:, None], ec2[ce].reshape(nc, -1)], axis=1)
    cand.sort(axis=1)
    keep = np.ones_like(cand, dtype=bool)
    keep[:, 1:] = cand[:, 1:] != cand[:, :-1]
    keep &= cand >= 0
    e2c_ptr = np.zeros(nc + 1, dtype=np.int64)
    np.cumsum(keep.sum(axis=1), out=e2c_ptr[1:])
    e2c = cand[keep]
    ed = np.asarray(pres.entity_dofs[2])
    pptr = np.arange(nc + 1, dtype=np.int64) * ed.shape[1]
    pdofs = (ed + int(mixed.offset)).ravel()
    return (e2c_ptr.astype(np.int32), e2c.astype(np.int32), pptr.astype(np.int32),
            pdofs.astype(np.int32), _Entities([(2, nc)]))


def build_patches_hdiv_extended(mixed, bc=None, weighting: str = "invmult") -> PatchSet:
    """One patch per cell extended over its edge neighbours (reference
    ``vanka.py:99-119``)."""
    if mixed.case not in ("bdm", "rt"):
        raise ValueError("extended cell patches are for the normal-continuity pairs")
    return _launch_build(mixed, bc, weighting, *hdiv_candidates(mixed))


def build_patches(mixed, bc=None, weighting: str = "invmult") -> PatchSet:
    """Reference ``vanka.build_patches`` (``vanka.py:122-126``)."""
    if mixed.case in ("th-tri", "th-quad"):
        return build_patches_taylor_hood(mixed, bc, weighting)
    return build_patches_hdiv_extended(mixed, bc, weighting)


# ----------------------------------------------------------------------------
# factor / apply (reference vanka.py:129-148)
# ----------------------------------------------------------------------------

def factor_patches(patchset: PatchSet, system) -> PatchSet:
    """Extract and invert every patch block (reference ``vanka.factor_patches``,
    ``vanka.py:129-139``); a singular block raises ``SingularMatrixError``
    naming the patch entity, like the reference."""
    matrix = system.matrix if hasattr(system, "matrix") else system
    d = device_csr(matrix)
    n = patchset.num_patches
    status = np.zeros(max(n, 1), dtype=np.int32)
    bad = C.c_int32(-1)
    st = L.call("vk_patches_factor", patchset.handle, d.handle, L.ptr(status), C.byref(bad))
    if st == L.VK_SINGULAR:
        p = bad.value
        why = ("matrix has an all-zero row" if status[p] == L.VK_PATCH_ZERO_ROW
               else "pivot below 1e-12 of its row magnitude")
        raise SingularMatrixError(
            f"singular patch block at entity {patchset.entity_of(p)}") from SingularMatrixError(why)
    patchset.factored = True
    patchset._matrix = d
    return patchset


def apply_additive(patchset: PatchSet, residual, out=None, *, scale: float = 1.0,
                   mode: int = L.VK_APPLY_OUT, zbuf=None):
    """Weighted sum of exact local solves, sum_i R_i^T W_i A_i^{-1} R_i r
    (reference ``vanka.apply_additive``, ``vanka.py:142-148``).

    numpy in -> numpy out (host copies inside); CUDA tensor in -> CUDA tensor
    out.  ``mode``/``scale`` expose the fused damped-update epilogues used by
    the smoother (``x = scale*out`` / ``x += scale*out``).  ``zbuf`` (a CUDA
    float64 tensor of :meth:`PatchSet.zbuf_size` entries) holds the per-patch
    corrections; sweeps of one patch set that may run concurrently on
    different streams each need their own (default: the set's buffer)."""
    import torch
    if not patchset.factored:
        raise ValueError("patches must be factored before apply_additive")
    rd, host = to_device(residual)
    if rd.numel() != patchset.size:
        raise ValueError(f"residual has {rd.numel()} entries, patch set needs {patchset.size}")
    if out is None:
        out = torch.empty_like(rd)
    if zbuf is not None and (zbuf.numel() < patchset.zbuf_size or zbuf.dtype != torch.float64
                             or not zbuf.is_cuda):
        raise ValueError(f"zbuf needs {patchset.zbuf_size} CUDA float64 entries")
    L.call("vk_patches_apply", patchset.handle, L.ptr(rd), L.ptr(out), scale, mode,
           L.ptr(zbuf), L.stream_ptr())
    return to_host(out, host)


class SweepStream:
    """Pipelined host-to-host additive sweeps (the batched form of
    :func:`apply_additive` for many right-hand sides held in host memory).

    Three CUDA streams: the host->device copy of residual k+1 and the
    device->host copy of result k-1 overlap the sweep of residual k; device
    buffers rotate through ``depth`` slots guarded by events.  Every residual
    still crosses PCIe in and every result out."""

    def __init__(self, patchset: PatchSet, *, scale: float = 1.0, mode: int = L.VK_APPLY_OUT,
                 depth: int = 3):
        import torch
        if not patchset.factored:
            raise ValueError("patches must be factored")
        self.ps = patchset
        self.scale = scale
        self.mode = mode
        self.depth = depth
        n = patchset.size
        self.r_dev = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(depth)]
        self.o_dev = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(depth)]
        self.s_in, self.s_comp, self.s_out = (torch.cuda.Stream() for _ in range(3))
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_comp = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self._used = [False] * depth

    def run(self, residuals, outputs):
        """residuals / outputs: sequences of (preferably pinned) host float64
        tensors of length ``size``; results are in ``outputs`` once
        :meth:`wait` (or a device synchronize) returns."""
        import torch
        h = self.ps.handle
        start = torch.cuda.current_stream()
        for s in (self.s_in, self.s_comp, self.s_out):
            s.wait_stream(start)
        for k, (rh, oh) in enumerate(zip(residuals, outputs)):
            q = k % self.depth
            with torch.cuda.stream(self.s_in):
                if self._used[q]:
                    self.s_in.wait_event(self.ev_comp[q])      # slot's residual consumed
                self.r_dev[q].copy_(rh, non_blocking=True)
                self.ev_in[q].record(self.s_in)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(self.ev_in[q])
                if self._used[q]:
                    self.s_comp.wait_event(self.ev_out[q])     # slot's result drained
                L.call("vk_patches_apply", h, L.ptr(self.r_dev[q]), L.ptr(self.o_dev[q]),
                       self.scale, self.mode, None, self.s_comp.cuda_stream)
                self.ev_comp[q].record(self.s_comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_comp[q])
                oh.copy_(self.o_dev[q], non_blocking=True)
                self.ev_out[q].record(self.s_out)
            self._used[q] = True
        start.wait_stream(self.s_out)
        return outputs

    def wait(self):
        self.s_out.synchronize()


def patch_inverses(patchset: PatchSet, first: int = 0, count: int | None = None) -> list:
    """Host copies of the explicit patch inverses (row-major), for tests."""
    n = patchset.num_patches
    count = n - first if count is None else count
    ex = patchset.export()
    sizes = np.diff(ex["offsets"])[first:first + count]
    buf = np.zeros(int(np.sum(sizes.astype(np.int64) ** 2)))
    L.call("vk_patches_export_inverse", patchset.handle, first, count, L.ptr(buf))
    out, o = [], 0
    for s in sizes:
        out.append(buf[o:o + s * s].reshape(s, s))
        o += s * s
    return out


def extract_blocks(patchset: PatchSet, matrix, first: int = 0, count: int | None = None) -> list:
    """Device-extracted dense patch blocks A[idx, idx] (bit-exact), for tests."""
    d = device_csr(matrix)
    n = patchset.num_patches
    count = n - first if count is None else count
    ex = patchset.export()
    sizes = np.diff(ex["offsets"])[first:first + count]
    buf = np.zeros(int(np.sum(sizes.astype(np.int64) ** 2)))
    L.call("vk_patches_extract", patchset.handle, d.handle, first, count, L.ptr(buf))
    out, o = [], 0
    for s in sizes:
        out.append(buf[o:o + s * s].reshape(s, s))
        o += s * s
    return out


def _single_block_inverse(a: np.ndarray):
    """Explicit inverse + guard status of one dense block on the device (used
    by ``sparsela.lu_factor``): a one-patch set over a CSR copy of ``a``."""
    import scipy.sparse as sp
    import torch
    s = a.shape[0]
    csr = DeviceCSR(sp.csr_matrix(a))
    ps = PatchSet([Patch(None, np.arange(s), s)], s, np.ones(s), "unit")
    status = np.zeros(1, dtype=np.int32)
    bad = C.c_int32(-1)
    L.call("vk_patches_factor", ps.handle, csr.handle, L.ptr(status), C.byref(bad))
    if status[0] != L.VK_PATCH_OK:
        return None, int(status[0])
    inv = patch_inverses(ps)[0]
    return torch.from_numpy(np.ascontiguousarray(inv)).cuda(), 0
