"""Device assembly of the global saddle-point operator and of the
natural-embedding prolongation — the setup
that produces what the hot path consumes, without the reference and
without problem packs.

* :func:`assemble` — reference ``assembly.assemble`` (``assembly.py:
  288-332``) for the operator: cell terms 2 nu (eps u, eps v) - (div v, p)
  (``assembly.py:136-172``), for H(div) pairs the interior-facet terms with
  the alpha / h_e tangential-jump penalty (``assembly.py:230-270``), COO ->
  CSR with duplicates summed (``assembly.py:93-129``) and the symmetric
  strong-BC elimination with identity rows (``assembly.py:273-285``).  The
  element matrices are computed per cell / per facet on the device from the
  reference-cell tabulation (``vk_assemble_cells`` / ``vk_assemble_facets``).
* :func:`build_prolongation` — reference ``mg.build_prolongation`` /
  ``_mask_transfer`` (``mg.py:127-167``): the dual functionals of the fine
  element applied to the coarse basis for each parent/child configuration of
  the uniform refinement (host, a handful of small blocks, cached like the
  reference's), scattered on the device with the first-occurrence dedup and
  the |v| > 1e-12 filter (``vk_prolong_entries``, ``vk_coo_to_csr``).
* :func:`build_hierarchy` — reference ``mg.build_hierarchy`` (``mg.py:
  177-234``) end to end on the device.

The right-hand side of the manufactured problem (``assembly.py:136-172``
load with the forcing of ``assembly.py:62-87``, the Dirichlet lift and
boundary values of ``assembly.py:273-285`` / ``spaces.py:170-220``) is
assembled too (``System.rhs``, a device vector): the per-cell loads on the
device (``vk_assemble_load``), reduced in the reference's ``np.add.at``
order by the same deterministic COO reduction, the lift ``rhs - A @ lift``
with the unconstrained operator by the bit-exact residual kernel, and the
Taylor-Hood boundary values by the elements' dual functionals on the host
(boundary cells only).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from . import fem
from .sparsela import DeviceCSR


@dataclass
class ProblemConfig:
    """Reference ``assembly.ProblemConfig`` (``assembly.py:24-35``)."""
    case: str
    order: int
    viscosity: float = 1.0
    alpha: float | None = None

    @property
    def penalty(self) -> float:
        return self.alpha if self.alpha is not None else 10.0 * self.order ** 2


@dataclass
class System:
    """Reference ``BlockSystem`` (``assembly.py:38-51``): device matrix."""
    matrix: DeviceCSR
    rhs: object
    mixed: fem.Mixed
    bc: fem.StrongBc | None

    @property
    def num_velocity(self) -> int:
        return self.mixed.velocity.ndof

    @property
    def num_pressure(self) -> int:
        return self.mixed.pressure.ndof


def _dev(a, dtype=None):
    import torch
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return torch.from_numpy(arr).cuda()


def _mask(n, idx):
    m = np.zeros(max(n, 1), dtype=np.uint8)
    m[np.asarray(idx, dtype=np.int64)] = 1
    return _dev(m)


def _interior_edges(mesh):
    """Interior edges with their two cells (ascending), the local edge slot
    and orientation flag in each, tangent, normal and length."""
    topo, geom = mesh
    ptr, idx = topo.edge_cells_ptr, topo.edge_cells_idx
    inner = np.flatnonzero(np.diff(ptr) == 2)
    c1, c2 = idx[ptr[inner]], idx[ptr[inner] + 1]
    info = np.empty((len(inner), 6), dtype=np.int32)
    info[:, 0], info[:, 1] = c1, c2
    for col, cells in ((2, c1), (4, c2)):
        slots = np.argmax(geom.cell_edge_ids[cells] == inner[:, None], axis=1)
        info[:, col] = slots
        info[:, col + 1] = geom.cell_edge_aligned[cells, slots]
    geo = np.column_stack([geom.edge_tangent[inner], geom.edge_normal[inner],
                           geom.edge_length[inner]])
    return info, geo


def facet_tables(vel: fem.Space):
    """Interior-edge data of an H(div) velocity space: (info, geo) of
    :func:`_interior_edges`, the edge quadrature of degree 2 deg + 2
    (``assembly.py:194``) and the element's reference tabulation on each
    (local edge slot, orientation) — six tables, points matched by arc length
    along the global edge direction like ``jump_average_tables``
    (``assembly.py:188-226``)."""
    info, geo = _interior_edges(vel.mesh)
    erule = fem.quadrature("interval", 2 * vel.element.degree + 2)
    s = erule.points[:, 0]
    tabs_v, tabs_g = [], []
    for la, lb in fem.TRI_SLOTS:
        for aligned in (0, 1):
            a, b = (fem.TRI_REF[la], fem.TRI_REF[lb]) if aligned else \
                (fem.TRI_REF[lb], fem.TRI_REF[la])
            tv, tg = vel.element.tabulate(a + s[:, None] * (b - a))
            tabs_v.append(tv)
            tabs_g.append(tg)
    return info, geo, erule, tabs_v, tabs_g


class ManufacturedSolution:
    """Closed-form enclosed-flow solution with zero pressure (reference
    ``assembly.ManufacturedSolution``, ``assembly.py:54-87``): u = (sin pi x
    cos pi y, -cos pi x sin pi y), divergence-free with zero normal component
    on the unit-square boundary; forcing 2 pi^2 nu u.  Host evaluation for
    callers; the device kernels evaluate the same formulas per quadrature
    point (``vk_assemble_load``, ``vk_error_cells``)."""

    def __init__(self, viscosity: float = 1.0):
        self.viscosity = viscosity

    @staticmethod
    def velocity(pts):
        return manufactured_velocity(np.asarray(pts, dtype=float))

    @staticmethod
    def velocity_gradient(pts):
        pts = np.asarray(pts, dtype=float)
        sx, cx = np.sin(np.pi * pts[:, 0]), np.cos(np.pi * pts[:, 0])
        sy, cy = np.sin(np.pi * pts[:, 1]), np.cos(np.pi * pts[:, 1])
        g = np.empty((len(pts), 2, 2))
        g[:, 0, 0], g[:, 0, 1] = np.pi * cx * cy, -np.pi * sx * sy
        g[:, 1, 0], g[:, 1, 1] = np.pi * sx * sy, -np.pi * cx * cy
        return g

    @staticmethod
    def pressure(pts):
        return np.zeros(len(pts))

    def forcing(self, pts):
        return 2.0 * np.pi ** 2 * self.viscosity * self.velocity(pts)


def manufactured_data(viscosity: float = 1.0) -> ManufacturedSolution:
    """Reference ``assembly.manufactured_data`` (``assembly.py:90-91``)."""
    return ManufacturedSolution(viscosity)


def manufactured_velocity(pts):
    """Reference ``ManufacturedSolution.velocity`` (``assembly.py:65-69``)."""
    x, y = pts[:, 0], pts[:, 1]
    return np.column_stack([np.sin(np.pi * x) * np.cos(np.pi * y),
                            -np.cos(np.pi * x) * np.sin(np.pi * y)])


def interpolate(space: fem.Space, fn, *, boundary_only: bool = False) -> np.ndarray:
    """Reference ``spaces.interpolate`` (``spaces.py:170-200``): every dual
    functional applied to ``fn`` on the mapped cell, the last cell in cell
    order winning for shared DoFs, like the reference's loop.
    ``boundary_only``: just the cells that touch a boundary DoF (the only
    values ``strong_bc`` keeps)."""
    el = space.element
    topo, geom = space.mesh
    pts = np.vstack(el.dof_points)
    bounds = np.cumsum([0] + [len(p) for p in el.dof_points])
    coeffs = np.zeros(space.ndof)
    cells = np.flatnonzero(space.boundary_dof[space.cell_dofs].any(axis=1)) if boundary_only \
        else np.arange(topo.num_cells)
    # point-evaluation elements (Lagrange: one point per functional): the
    # per-DoF np.sum over one (scalar) or two (vector) products is a + (0. + b)
    # — numpy copies the first term and adds the rest onto a zero-started
    # partial sum, which matters only for the sign of zero — done for all the
    # cell's DoFs at once
    pointwise = el.mapping != "piola" and all(len(p) == 1 for p in el.dof_points)
    if pointwise:
        wmat = np.stack([np.asarray(w, dtype=float).reshape(-1) for w in el.dof_weights])
    for c in cells:
        verts = geom.vertex_coords[geom.cell_map_vertices[c]]
        fv = np.asarray(fn(fem.map_points(topo.cell_shape, verts, pts)), dtype=float)
        if pointwise:
            prod = wmat * fv.reshape(el.ndof, -1)
            val = prod[:, 0] if prod.shape[1] == 1 else prod[:, 0] + (0.0 + prod[:, 1])
            coeffs[space.cell_dofs[c]] = val / space.cell_dof_scale[c]
            continue
        if el.mapping == "piola":
            _, det, inv = fem.cell_jacobians(topo.cell_shape, verts, pts)
            fv = det[:, None] * np.einsum("qab,qb->qa", inv, fv)
        for i in range(el.ndof):
            val = np.sum(el.dof_weights[i] * fv[bounds[i]:bounds[i + 1]])
            coeffs[space.cell_dofs[c, i]] = val / space.cell_dof_scale[c, i]
    return coeffs


def interpolate_boundary(space: fem.Space, fn) -> np.ndarray:
    return interpolate(space, fn, boundary_only=True)


def assemble(mixed: fem.Mixed, config: ProblemConfig | None = None, *,
             apply_bc: bool = True, rhs: bool = True) -> System:
    """Assembled saddle-point operator on the device (velocity block first,
    then pressure), strong BCs eliminated with identity rows, and (``rhs``)
    the manufactured right-hand side with the Dirichlet lift."""
    import torch
    L.require_cuda()
    if config is None:
        config = ProblemConfig(mixed.case, mixed.order)
    vel, pres = mixed.velocity, mixed.pressure
    topo, geom = vel.mesh
    shape = topo.cell_shape
    rule = fem.quadrature(shape, 2 * config.order + 2)                 # assembly.py:143
    rv, rg = vel.element.tabulate(rule.points)
    pv, _ = pres.element.tabulate(rule.points)
    nv, npl = vel.element.ndof, pres.element.ndof
    nc = topo.num_cells
    n = mixed.ndof
    cell_xy = geom.vertex_coords[geom.cell_map_vertices]
    piola = int(vel.element.mapping == "piola")
    per_cell = nv * nv + 2 * npl * nv
    facets = mixed.case in ("bdm", "rt")
    if facets:
        info, geo, erule, tabs_v, tabs_g = facet_tables(vel)
        nfe = len(info)
    else:
        nfe = 0
    total = nc * per_cell + nfe * (2 * nv) ** 2
    keys = torch.empty(total + n, dtype=torch.int64, device="cuda")
    vals = torch.empty(total + n, dtype=torch.float64, device="cuda")
    keep = [_dev(rule.weights, np.float64), _dev(rule.points, np.float64), _dev(rv, np.float64),
            _dev(rg, np.float64), _dev(pv, np.float64), _dev(cell_xy, np.float64),
            _dev(vel.cell_dofs, np.int32), _dev(vel.cell_dof_scale, np.float64),
            _dev(pres.cell_dofs, np.int32), _dev(pres.cell_dof_scale, np.float64)]
    st = L.stream_ptr()
    L.call("vk_assemble_cells", nc, len(rule.weights), nv, npl, int(shape == "quad"), piola,
           *[L.ptr(t) for t in keep[:9]], L.ptr(keep[9]), vel.ndof, config.viscosity, n,
           L.ptr(keys), L.ptr(vals), st)
    if facets and nfe:
        fk = [_dev(erule.weights, np.float64), _dev(np.stack(tabs_v), np.float64),
              _dev(np.stack(tabs_g), np.float64), _dev(info, np.int32), _dev(geo, np.float64)]
        L.call("vk_assemble_facets", nfe, len(erule.weights), nv, *[L.ptr(t) for t in fk],
               L.ptr(keep[5]), L.ptr(keep[6]), L.ptr(keep[7]), config.viscosity,
               config.penalty, n, L.ptr(keys[nc * per_cell:]), L.ptr(vals[nc * per_cell:]), st)
    bc = fem.strong_bc(vel) if apply_bc else None
    b = None
    if rhs:
        # load: (dof, s_i load_i) per cell, reduced like the operator's COO
        # (an n x 1 matrix: duplicates summed in cell order = np.add.at)
        lk = torch.empty(nc * nv, dtype=torch.int64, device="cuda")
        lv = torch.empty(nc * nv, dtype=torch.float64, device="cuda")
        L.call("vk_assemble_load", nc, len(rule.weights), nv, int(shape == "quad"), piola,
               L.ptr(keep[0]), L.ptr(keep[1]), L.ptr(keep[2]), L.ptr(keep[5]), L.ptr(keep[6]),
               L.ptr(keep[7]), config.viscosity, L.ptr(lk), L.ptr(lv), st)
        hl = C.c_void_p()
        L.call("vk_coo_to_csr", nc * nv, L.ptr(lk), L.ptr(lv), n, 1, 0, 0.0, None, None, None,
               C.byref(hl))
        b = DeviceCSR(_handle=hl.value, _shape=(n, 1), _nnz=_nnz(hl)).matvec(
            torch.ones(1, dtype=torch.float64, device="cuda"))
        if bc is not None:
            if mixed.case in ("th-tri", "th-quad"):          # assembly.py:300 (Dirichlet data)
                values = interpolate_boundary(vel, manufactured_velocity)[bc.indices]
                bc = fem.StrongBc(bc.indices, values)
                lift = torch.zeros(n, dtype=torch.float64, device="cuda")
                lift[_dev(bc.indices, np.int64)] = _dev(values, np.float64)
                hf = C.c_void_p()                            # unconstrained operator
                L.call("vk_coo_to_csr", total, L.ptr(keys), L.ptr(vals), n, n, 0, 0.0, None,
                       None, None, C.byref(hf))
                full = DeviceCSR(_handle=hf.value, _shape=(n, n), _nnz=_nnz(hf))
                lifted = torch.empty_like(b)
                full.residual(b, lift, lifted)               # rhs - matrix @ lift
                b = lifted
                del full
            b[_dev(bc.indices, np.int64)] = _dev(bc.values, np.float64)   # assembly.py:280
    mask = _mask(n, bc.indices) if bc is not None else None
    h = C.c_void_p()
    mp = L.ptr(mask) if mask is not None else None
    L.call("vk_coo_to_csr", total, L.ptr(keys), L.ptr(vals), n, n, 0, 0.0, mp, mp, mp,
           C.byref(h))
    matrix = DeviceCSR(_handle=h.value, _shape=(n, n), _nnz=_nnz(h))
    return System(matrix, b, mixed, bc)


def _nnz(h):
    nr, ncol, nnz = C.c_int32(), C.c_int32(), C.c_int64()
    L.call("vk_csr_info", h, C.byref(nr), C.byref(ncol), C.byref(nnz))
    return int(nnz.value)


# ----------------------------------------------------------------------------
# prolongation (reference mg.py:91-167)
# ----------------------------------------------------------------------------

def _unique_rows(rows: np.ndarray):
    """(index of the first occurrence of every distinct row, group id of every
    row) like ``np.unique(rows, axis=0, return_index=True,
    return_inverse=True)``, with the groups in ascending order of a 64-bit row
    hash instead of lexicographic order (the callers only use first
    occurrences).  The lexicographic sort of 5e5 ten-column rows was the
    largest single item of the P2 256^2 setup (0.74 of 1.4 s); hashing the
    rows and sorting one integer column is ~20x cheaper.  Every row is then
    compared with its group's representative, so a hash collision cannot go
    unnoticed (it falls back to the lexicographic path)."""
    rows = np.ascontiguousarray(rows, dtype=np.float64) + 0.0        # -0.0 -> +0.0
    mult = (np.arange(1, rows.shape[1] + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) \
        | np.uint64(1)
    h = (rows.view(np.uint64) * mult).sum(axis=1, dtype=np.uint64)
    h ^= h >> np.uint64(29)
    _, first, inv = np.unique(h, return_index=True, return_inverse=True)
    inv = inv.ravel()
    if not np.array_equal(rows, rows[first][inv]):
        _, first, inv = np.unique(rows, axis=0, return_index=True, return_inverse=True)
        inv = inv.ravel()
    return first, inv


def _configurations(coarse: fem.Space, fine: fem.Space, children):
    """Configuration id of every (parent, child) pair: the reference's cache
    key (coarse Jacobian, fine Jacobian, child origin in the parent's
    reference coordinates rounded to 12 digits, ``mg.py:95-98``); ids in
    order of first occurrence, with that first pair."""
    cg, fg = coarse.mesh.geometry, fine.mesh.geometry
    cxy = cg.vertex_coords[cg.cell_map_vertices]
    fxy = fg.vertex_coords[fg.cell_map_vertices]
    par = np.repeat(np.arange(len(children)), 4)
    chi = children.ravel()
    cj = np.stack([cxy[:, 1] - cxy[:, 0], cxy[:, 2] - cxy[:, 0]], -1)      # columns
    fj = np.stack([fxy[:, 1] - fxy[:, 0], fxy[:, 2] - fxy[:, 0]], -1)
    # child origin in the parent's reference coordinates (structured meshes:
    # affine parents, one 2x2 solve per pair)
    rel = np.linalg.solve(cj[par], (fxy[chi, 0] - cxy[par, 0])[..., None])[..., 0]
    keyrows = np.concatenate([cj[par].reshape(len(par), -1), fj[chi].reshape(len(par), -1),
                              rel.round(12)], axis=1)
    first, inv = _unique_rows(keyrows)
    order = np.argsort(first)                    # ids by first occurrence
    remap = np.empty_like(order)
    remap[order] = np.arange(len(order))
    return remap[inv.ravel()].astype(np.int32), [(par[first[o]], chi[first[o]]) for o in order]


def _entries(coarse: fem.Space, fine: fem.Space, parent, child):
    """Fine dual functionals applied to the (mapped) coarse basis on one
    parent / child pair (reference ``_prolongation_entries``, mg.py:91-124)."""
    ce, fe = coarse.element, fine.element
    shape = coarse.mesh.topology.cell_shape
    cxy = coarse.mesh.geometry.cell_coords(parent)
    fxy = fine.mesh.geometry.cell_coords(child)
    all_pts = np.vstack(fe.dof_points)
    phys = fem.map_points(shape, fxy, all_pts)
    cref = fem.inverse_map(shape, cxy, phys)
    cvals, _ = ce.tabulate(cref)
    if ce.mapping == "piola":
        cjac = np.column_stack([cxy[1] - cxy[0], cxy[2] - cxy[0]])
        _, cdet, _ = fem.cell_jacobians(shape, cxy, cref)
        _, fdet, finv = fem.cell_jacobians(shape, fxy, all_pts)
        cvals = np.einsum("qab,qjb->qja", cjac[None] / cdet[:, None, None], cvals)
        cvals = np.einsum("q,qab,qjb->qja", fdet, finv, cvals)
    out = np.empty((fe.ndof, ce.ndof))
    start = 0
    for i in range(fe.ndof):
        stop = start + len(fe.dof_points[i])
        w = fe.dof_weights[i]
        out[i] = np.einsum("q,qj->j", w, cvals[start:stop]) if fe.value_shape == () else \
            np.einsum("qv,qjv->j", w, cvals[start:stop])
        start = stop
    return out


def build_prolongation(coarse: fem.Mixed, fine: fem.Mixed, children,
                       coarse_bc=None, fine_bc=None):
    """(full, masked) device prolongations of the mixed space
    (block_diag(P_velocity, P_pressure), reference ``mg.py:208-216``)."""
    import torch
    L.require_cuda()
    nrows, ncols = fine.ndof, coarse.ndof
    blocks = []
    for cs, fs, roff, coff in ((coarse.velocity, fine.velocity, 0, 0),
                               (coarse.pressure, fine.pressure, fine.velocity.ndof,
                                coarse.velocity.ndof)):
        cfg, firsts = _configurations(cs, fs, children)
        tables = np.stack([_entries(cs, fs, p, c) for p, c in firsts])
        blocks.append((cs, fs, roff, coff, cfg, tables))
    counts = [len(children) * 4 * b[1].element.ndof * b[0].element.ndof for b in blocks]
    keys = torch.empty(sum(counts), dtype=torch.int64, device="cuda")
    vals = torch.empty(sum(counts), dtype=torch.float64, device="cuda")
    st = L.stream_ptr()
    kids = _dev(children, np.int32)
    off = 0
    hold = []
    for (cs, fs, roff, coff, cfg, tables), cnt in zip(blocks, counts):
        args = [_dev(cfg, np.int32), _dev(tables, np.float64), _dev(cs.cell_dofs, np.int32),
                _dev(cs.cell_dof_scale, np.float64), _dev(fs.cell_dofs, np.int32),
                _dev(fs.cell_dof_scale, np.float64)]
        hold += args
        L.call("vk_prolong_entries", len(children), fs.element.ndof, cs.element.ndof,
               L.ptr(kids), *[L.ptr(t) for t in args], roff, coff, ncols,
               L.ptr(keys[off:]), L.ptr(vals[off:]), st)
        off += cnt
    out = []
    rmask = _mask(nrows, fine_bc.indices) if fine_bc is not None else None
    cmask = _mask(ncols, coarse_bc.indices) if coarse_bc is not None else None
    for rm, cm in ((None, None), (rmask, cmask)):
        h = C.c_void_p()
        L.call("vk_coo_to_csr", len(keys), L.ptr(keys), L.ptr(vals), nrows, ncols, 1, 1e-12,
               L.ptr(rm), L.ptr(cm), None, C.byref(h))
        out.append(DeviceCSR(_handle=h.value, _shape=(nrows, ncols), _nnz=_nnz(h)))
    return out[0], out[1]


# ----------------------------------------------------------------------------
# hierarchy (reference mg.py:177-234)
# ----------------------------------------------------------------------------

def build_hierarchy(case: str, k: int, levels: int, config: ProblemConfig | None = None, *,
                    nu: int = 2, weighting: str = "invmult", cheb_mode: str = "repeat",
                    seed: int = 0, est_steps: int = 10, damping: float | None = None):
    """Rediscretised hierarchy on the ``mg.COARSE_CELLS_PER_SIDE`` base mesh
    refined ``levels`` times, built entirely on the device (meshes / DoF
    maps on the host): per level the assembled operator, patches built and
    factored, transfers; Chebyshev bounds estimated on the device like the
    reference (``est_steps``, ``seed``), or pinned by ``damping`` (the
    BASELINE recipe: damp = 2 / (lower + upper) = damping)."""
    from . import mg
    if levels < 0:
        raise ValueError("need a nonnegative refinement count")
    if cheb_mode not in mg.CHEB_MODES:
        raise ValueError(f"unknown chebyshev mode {cheb_mode!r}")
    if config is None:
        config = ProblemConfig(case, k)
    if config.case != case or config.order != k:
        raise ValueError("problem config does not match the requested case")
    shape = "quad" if case == "th-quad" else "tri"
    n0 = mg.COARSE_CELLS_PER_SIDE
    lv = []
    for i in range(levels + 1):
        mesh = fem.structured_mesh(shape, n0 * 2 ** i)
        mixed = fem.build_mixed(case, mesh, k)
        system = assemble(mixed, config, rhs=(i == levels))   # the finest level's load
        masked = full = None
        if i > 0:
            prev = lv[-1]
            full, masked = build_prolongation(prev[0], mixed, fem.refine_links(shape, n0 * 2 ** (i - 1)),
                                              prev[1].bc, system.bc)
        lv.append((mixed, system, masked, full))
    if damping is None:
        hier = mg._build(lv, nu, weighting, cheb_mode, lambda i: None, config)
        return mg.estimate_spectra(hier, est_steps=est_steps, seed=seed)
    upper = 2.0 / damping - 1.0
    return mg._build(lv, nu, weighting, cheb_mode,
                     lambda i: mg.FixedDamping(1.0, upper) if i > 0 else None, config)
