"""Host-side discretisation data for device assembly: structured meshes,
quadrature, reference elements and global DoF maps.

Everything here is O(mesh size) integer bookkeeping or O(1) reference-cell
tabulation (a few hundred basis evaluations); the O(mesh size) floating-point
work — element matrices, facet terms, COO -> CSR, boundary elimination,
prolongation scatter — runs on the device (``assembly.py``,
``csrc/vk_assembly.cu``).

The definitions restate the reference discretisation (``stokesmg``) so that
global numbering and basis functions coincide with it:

* meshes: ``meshtopo.py:93-231`` (vertex / edge / cell numbering, local
  vertex order of the reference map, edge slots), refinement links
  ``meshtopo.py:234-288``;
* quadrature: ``elements.py:45-69`` (Gauss-Legendre, collapsed
  Gauss-Jacobi on the triangle);
* modal bases: orthonormal Dubiner on the triangle, tensor Legendre on the
  square (``elements.py:74-138``); nodal Lagrange elements on the
  entity-ordered equispaced lattice (``elements.py:189-280``); vector
  elements with interleaved components (``elements.py:300-341``);
  normal-moment BDM / RT elements (``elements.py:347-447``);
* spaces: entity-blocked global numbering, edge permutations / signs and
  length normalisation (``spaces.py:63-124``), boundary DoFs and strong BCs
  (``spaces.py:117-121, 203-220``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from numpy.polynomial.legendre import leggauss
from scipy.linalg import null_space
from scipy.special import eval_jacobi, eval_legendre, roots_jacobi

TRI_SLOTS = ((1, 2), (0, 2), (0, 1))          # local edge k = local vertices
QUAD_SLOTS = ((0, 1), (2, 3), (0, 2), (1, 3))
TRI_REF = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
QUAD_REF = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
MAX_QUAD_DEGREE = 20
CASES = ("th-tri", "th-quad", "bdm", "rt")


# ============================================================================
# structured meshes of the unit square
# ============================================================================

@dataclass
class Topology:
    """Reference ``MeshTopology`` attribute names; adjacency as CSR pairs
    (``*_ptr`` / ``*_idx``) with list views for reference-style callers."""
    cell_shape: str
    cells_per_side: int
    num_vertices: int
    num_edges: int
    num_cells: int
    cell_vertices: np.ndarray
    cell_edges: np.ndarray
    edge_vertices: np.ndarray
    edge_cells_ptr: np.ndarray
    edge_cells_idx: np.ndarray
    vertex_cells_ptr: np.ndarray
    vertex_cells_idx: np.ndarray
    boundary_vertex: np.ndarray
    boundary_edge: np.ndarray

    def entity_count(self, dim: int) -> int:
        return (self.num_vertices, self.num_edges, self.num_cells)[dim]

    @property
    def edge_cells(self):
        return _lists(self.edge_cells_ptr, self.edge_cells_idx)

    @property
    def vertex_cells(self):
        return _lists(self.vertex_cells_ptr, self.vertex_cells_idx)


def _lists(ptr, idx):
    return [idx[ptr[i]:ptr[i + 1]].tolist() for i in range(len(ptr) - 1)]


@dataclass
class Geometry:
    vertex_coords: np.ndarray     # (nv, 2)
    edge_length: np.ndarray
    edge_tangent: np.ndarray      # unit, lower -> higher vertex
    edge_normal: np.ndarray       # unit, away from the lower-indexed cell
    cell_map_vertices: np.ndarray  # (nc, 3|4) reference-map order
    cell_edge_ids: np.ndarray      # (nc, 3|4) per local edge slot
    cell_edge_aligned: np.ndarray  # slot direction == global direction

    def cell_coords(self, cell):
        return self.vertex_coords[self.cell_map_vertices[cell]]


@dataclass
class Mesh:
    topology: Topology
    geometry: Geometry

    def __iter__(self):            # unpacks as (topology, geometry)
        return iter((self.topology, self.geometry))


def _incidence(n_items, owners):
    """CSR of sorted owner lists per item from an (n_owner, k) item table."""
    k = owners.shape[1]
    items = owners.ravel()
    own = np.repeat(np.arange(owners.shape[0]), k)
    order = np.lexsort((own, items))
    ptr = np.zeros(n_items + 1, dtype=np.int64)
    np.add.at(ptr, items + 1, 1)
    return np.cumsum(ptr).astype(np.int32), own[order].astype(np.int32)


def structured_mesh(shape: str, n: int) -> Mesh:
    """n x n squares of the unit square; triangles split along the
    top-left / bottom-right diagonal (reference ``build_structured_tri`` /
    ``build_structured_quad``, ``meshtopo.py:177-231``)."""
    if n < 1:
        raise ValueError("need at least one cell per side")
    vid = np.arange((n + 1) ** 2).reshape(n + 1, n + 1)
    ii, jj = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    coords = np.column_stack([jj.ravel() / n, ii.ravel() / n])
    nh = n * (n + 1)
    hor = np.arange(nh).reshape(n + 1, n)
    ver = nh + np.arange(nh).reshape(n, n + 1)
    ev = [np.column_stack([vid[:, :-1].ravel(), vid[:, 1:].ravel()]),
          np.column_stack([vid[:-1, :].ravel(), vid[1:, :].ravel()])]
    a, b = vid[:-1, :-1], vid[:-1, 1:]             # bottom corners of square (i, j)
    c, d = vid[1:, :-1], vid[1:, 1:]               # top corners
    if shape == "tri":
        dia = 2 * nh + np.arange(n * n).reshape(n, n)
        ev.append(np.column_stack([b.ravel(), c.ravel()]))
        lower_v = np.stack([a, b, c], -1).reshape(-1, 3)
        upper_v = np.stack([b, d, c], -1).reshape(-1, 3)
        lower_e = np.stack([dia, ver[:, :-1], hor[:-1, :]], -1).reshape(-1, 3)
        upper_e = np.stack([hor[1:, :], dia, ver[:, 1:]], -1).reshape(-1, 3)
        cmv = np.empty((2 * n * n, 3), dtype=np.int64)
        cei = np.empty((2 * n * n, 3), dtype=np.int64)
        cmv[0::2], cmv[1::2] = lower_v, upper_v
        cei[0::2], cei[1::2] = lower_e, upper_e
        slots = TRI_SLOTS
    elif shape == "quad":
        cmv = np.stack([a, b, c, d], -1).reshape(-1, 4).astype(np.int64)
        cei = np.stack([hor[:-1, :], hor[1:, :], ver[:, :-1], ver[:, 1:]], -1)
        cei = cei.reshape(-1, 4).astype(np.int64)
        slots = QUAD_SLOTS
    else:
        raise ValueError(f"unknown cell shape {shape!r}")
    edge_vertices = np.vstack(ev).astype(np.int64)
    nv, ne, nc = len(coords), len(edge_vertices), len(cmv)
    bvert = np.zeros(nv, dtype=bool)
    bvert[vid[0, :]] = bvert[vid[n, :]] = bvert[vid[:, 0]] = bvert[vid[:, n]] = True
    bedge = np.zeros(ne, dtype=bool)
    bedge[hor[0, :]] = bedge[hor[n, :]] = bedge[ver[:, 0]] = bedge[ver[:, n]] = True
    ec_ptr, ec_idx = _incidence(ne, cei)
    vc_ptr, vc_idx = _incidence(nv, cmv)
    aligned = np.column_stack([cmv[:, la] < cmv[:, lb] for la, lb in slots])
    topo = Topology(shape, n, nv, ne, nc, np.sort(cmv, axis=1), np.sort(cei, axis=1),
                    edge_vertices, ec_ptr, ec_idx, vc_ptr, vc_idx, bvert, bedge)
    vec = coords[edge_vertices[:, 1]] - coords[edge_vertices[:, 0]]
    length = np.linalg.norm(vec, axis=1)
    tangent = vec / length[:, None]
    normal = np.column_stack([tangent[:, 1], -tangent[:, 0]])
    mid = 0.5 * (coords[edge_vertices[:, 0]] + coords[edge_vertices[:, 1]])
    first = ec_idx[ec_ptr[:-1]]
    centroid = coords[cmv[first]].mean(axis=1)
    flip = np.einsum("ij,ij->i", normal, mid - centroid) < 0
    normal[flip] = -normal[flip]
    geom = Geometry(coords, length, tangent, normal, cmv, cei, aligned)
    return Mesh(topo, geom)


def refine_links(shape: str, n: int) -> np.ndarray:
    """Children of every coarse cell in the n -> 2n refinement, in the
    reference order (``meshtopo.py:271-286``): (ncoarse, 4) fine cell ids."""
    m = 2 * n
    if shape == "quad":
        i, j = np.divmod(np.arange(n * n), n)
        base = 2 * i * m + 2 * j
        return np.column_stack([base, base + 1, base + m, base + m + 1])
    c = np.arange(2 * n * n)
    sq, t = np.divmod(c, 2)
    i, j = np.divmod(sq, n)
    fsq = lambda a, b: 2 * (a * m + b)  # noqa: E731
    lower = np.column_stack([fsq(2 * i, 2 * j), fsq(2 * i, 2 * j + 1), fsq(2 * i + 1, 2 * j),
                             fsq(2 * i, 2 * j) + 1])
    upper = np.column_stack([fsq(2 * i, 2 * j + 1) + 1, fsq(2 * i + 1, 2 * j + 1) + 1,
                             fsq(2 * i + 1, 2 * j) + 1, fsq(2 * i + 1, 2 * j + 1)])
    return np.where((t == 0)[:, None], lower, upper)


# ============================================================================
# quadrature
# ============================================================================

@dataclass
class Quadrature:
    points: np.ndarray
    weights: np.ndarray


def _gauss01(npts):
    x, w = leggauss(npts)
    return 0.5 * (x + 1.0), 0.5 * w


def quadrature(shape: str, degree: int) -> Quadrature:
    """Exact to ``degree``: Gauss-Legendre on [0,1], its tensor square, and
    on the triangle the collapsed rule (Gauss-Legendre x Gauss-Jacobi(1,0)
    through (u, v) -> (u (1 - v), v)) — reference ``elements.py:45-69``."""
    if not 0 <= degree <= MAX_QUAD_DEGREE:
        raise ValueError(f"unsupported quadrature degree {degree}")
    npts = degree // 2 + 1
    x, w = _gauss01(npts)
    if shape == "interval":
        return Quadrature(x[:, None], w)
    if shape == "quad":
        px, py = np.meshgrid(x, x, indexing="ij")
        return Quadrature(np.column_stack([px.ravel(), py.ravel()]), np.outer(w, w).ravel())
    if shape == "tri":
        t, wt = roots_jacobi(npts, 1.0, 0.0)
        v, wv = 0.5 * (t + 1.0), 0.25 * wt
        uu, vv = np.meshgrid(x, v, indexing="ij")
        pts = np.column_stack([(uu * (1.0 - vv)).ravel(), vv.ravel()])
        return Quadrature(pts, np.outer(w, wv).ravel())
    raise ValueError(f"unknown shape {shape!r}")


# ============================================================================
# orthonormal modal bases (values and gradients)
# ============================================================================

def _collapsed_legendre(k, u, s):
    """L_a = s^a P_a(u / s), a = 0..k, and its partials in u and s
    (three-term recurrence, regular at s = 0)."""
    L = np.zeros((k + 1,) + u.shape)
    Lu = np.zeros_like(L)
    Ls = np.zeros_like(L)
    L[0] = 1.0
    if k >= 1:
        L[1], Lu[1] = u, 1.0
    # the operation order of the recurrence is kept as published
    # ((2a+1) u L_a - a s^2 L_{a-1}) / (a+1): the H(div) interior moments come
    # from the null space of edge functionals evaluated on this basis, whose
    # orthonormal basis (an SVD) is not continuous in last-bit changes
    for a in range(1, k):
        L[a + 1] = ((2 * a + 1) * u * L[a] - a * s * s * L[a - 1]) / (a + 1)
        Lu[a + 1] = ((2 * a + 1) * (L[a] + u * Lu[a]) - a * s * s * Lu[a - 1]) / (a + 1)
        Ls[a + 1] = ((2 * a + 1) * u * Ls[a] - a * (2 * s * L[a - 1] + s * s * Ls[a - 1])) / (a + 1)
    return L, Lu, Ls


def dubiner(k: int, pts):
    """Orthonormal basis of P_k on the unit triangle, ordered by total degree
    d and then a = 0..d (b = d - a): c_ab L_a J_b^(2a+1,0)(2y-1).
    Returns values (nq, nb) and gradients (nq, nb, 2)."""
    x, y = pts[:, 0], pts[:, 1]
    u, s, z = 2.0 * x + y - 1.0, 1.0 - y, 2.0 * y - 1.0
    L, Lu, Ls = _collapsed_legendre(k, u, s)
    cols, dcols = [], []
    for d in range(k + 1):
        for a in range(d + 1):
            b = d - a
            J = eval_jacobi(b, 2 * a + 1, 0, z)
            dJ = 0.5 * (b + 2 * a + 2) * eval_jacobi(b - 1, 2 * a + 2, 1, z) if b else 0.0 * z
            c = np.sqrt(2.0 * (2 * a + 1) * (a + b + 1))
            cols.append(c * L[a] * J)
            # d/dx: u_x = 2;  d/dy: u_y = 1, s_y = -1, z_y = 2
            dcols.append(np.stack([c * 2.0 * Lu[a] * J,
                                   c * ((Lu[a] - Ls[a]) * J + 2.0 * L[a] * dJ)], -1))
    return np.stack(cols, 1), np.stack(dcols, 1)


def _legendre01(k, t):
    """sqrt(2a+1) P_a(2t-1), a = 0..k, and derivatives in t."""
    z = 2.0 * t - 1.0
    v = np.empty((k + 1,) + t.shape)
    dv = np.empty_like(v)
    for a in range(k + 1):
        sc = np.sqrt(2.0 * a + 1.0)
        v[a] = sc * eval_legendre(a, z)
        dv[a] = sc * (a + 1) * eval_jacobi(a - 1, 1, 1, z) if a else 0.0
    return v, dv


def tensor_legendre(k: int, pts):
    """Orthonormal basis of Q_k on the unit square, (a, b) with a outer."""
    px, dpx = _legendre01(k, pts[:, 0])
    py, dpy = _legendre01(k, pts[:, 1])
    vals = np.einsum("aq,bq->qab", px, py).reshape(len(pts), -1)
    gx = np.einsum("aq,bq->qab", dpx, py).reshape(len(pts), -1)
    gy = np.einsum("aq,bq->qab", px, dpy).reshape(len(pts), -1)
    return vals, np.stack([gx, gy], -1)


# ============================================================================
# reference elements
# ============================================================================

@dataclass
class Element:
    """Reference element (reference ``ReferenceElement``, ``elements.py:
    143-171``): basis = modal(x) @ coeffs."""
    family: str
    degree: int
    cell_shape: str
    value_shape: tuple
    ndof: int
    mapping: str                      # "identity" | "piola"
    entity_dofs: dict
    dof_entity: list                  # (dim, local entity, position)
    dof_points: list
    dof_weights: list
    edge_reverse_perm: np.ndarray
    edge_reverse_sign: np.ndarray
    modal: object = field(repr=False, default=None)   # pts -> (vals, grads) of the modal set
    coeffs: np.ndarray | None = None
    length_normalized: bool = False
    edge_ref_lengths: np.ndarray | None = None
    scalar: "Element | None" = None   # vector elements: the component element

    def edge_transform(self, aligned: bool):
        m = len(self.edge_reverse_perm)
        return (np.arange(m), np.ones(m)) if aligned else \
            (self.edge_reverse_perm, self.edge_reverse_sign)

    def tabulate(self, pts):
        """Values (nq, ndof[, 2]) and reference gradients (..., 2)."""
        pts = np.atleast_2d(np.asarray(pts, dtype=float))
        if self.scalar is not None:                     # interleaved vector element
            sv, sg = self.scalar.tabulate(pts)
            nq, ns = sv.shape
            vals = np.zeros((nq, 2 * ns, 2))
            grads = np.zeros((nq, 2 * ns, 2, 2))
            for comp in (0, 1):
                vals[:, comp::2, comp] = sv
                grads[:, comp::2, comp, :] = sg
            return vals, grads
        mv, mg = self.modal(pts)
        if self.value_shape == ():
            return mv @ self.coeffs, np.einsum("qpd,pj->qjd", mg, self.coeffs)
        return (np.einsum("qpv,pj->qjv", mv, self.coeffs),
                np.einsum("qpvd,pj->qjvd", mg, self.coeffs))


def _lattice(shape, k):
    """Entity-ordered equispaced lattice: vertices, edge interiors by slot,
    cell interior (reference ``elements.py:189-219``)."""
    verts, slots = (TRI_REF, TRI_SLOTS) if shape == "tri" else (QUAD_REF, QUAD_SLOTS)
    pts = [v for v in verts]
    owner = [(0, i) for i in range(len(verts))]
    for e, (la, lb) in enumerate(slots):
        for i in range(1, k):
            pts.append(verts[la] + (i / k) * (verts[lb] - verts[la]))
            owner.append((1, e))
    for i in range(1, k):
        for j in range(1, (k - i) if shape == "tri" else k):
            pts.append(np.array([i / k, j / k]))
            owner.append((2, 0))
    return np.array(pts), owner


def _entity_tables(owner, counts):
    ent = {d: [[] for _ in range(counts[d])] for d in range(3)}
    dof_entity = []
    for i, (dim, e) in enumerate(owner):
        dof_entity.append((dim, e, len(ent[dim][e])))
        ent[dim][e].append(i)
    return ent, dof_entity


def lagrange(shape: str, k: int, discontinuous: bool = False) -> Element:
    """Nodal Lagrange on the equispaced lattice (reference ``elements.py:
    222-280``); ``discontinuous``: all DoFs owned by the cell (dP_k)."""
    if discontinuous and k == 0:
        pts, owner = np.array([[1.0 / 3.0, 1.0 / 3.0]]), [(2, 0)]
    else:
        pts, owner = _lattice(shape, k)
        if discontinuous:
            owner = [(2, 0)] * len(pts)
    modal = (lambda p: dubiner(k, p)) if shape == "tri" else (lambda p: tensor_legendre(k, p))
    coeffs = np.linalg.inv(modal(pts)[0])
    counts = (3, 3, 1) if shape == "tri" else (4, 4, 1)
    ent, dof_entity = _entity_tables(owner, counts)
    m = 0 if discontinuous else k - 1
    fam = ("dlagrange-" if discontinuous else "lagrange-") + shape
    return Element(fam, k, shape, (), len(pts), "identity", ent, dof_entity,
                   [p[None, :] for p in pts], [np.ones(1) for _ in pts],
                   np.arange(m)[::-1].copy(), np.ones(m), modal, coeffs)


def vector(scalar: Element) -> Element:
    """Two components interleaved per scalar DoF (``elements.py:300-341``)."""
    ent = {d: [[2 * i + c for i in e for c in (0, 1)] for e in scalar.entity_dofs[d]]
           for d in range(3)}
    dof_entity = [(dim, e, 2 * pos + c) for (dim, e, pos) in scalar.dof_entity for c in (0, 1)]
    pts, wts = [], []
    for i in range(scalar.ndof):
        for c in (0, 1):
            pts.append(scalar.dof_points[i])
            w = np.zeros((len(scalar.dof_weights[i]), 2))
            w[:, c] = scalar.dof_weights[i]
            wts.append(w)
    rp = scalar.edge_reverse_perm
    perm = (2 * np.repeat(rp, 2) + np.tile([0, 1], len(rp))).astype(int)
    sign = np.repeat(scalar.edge_reverse_sign, 2)
    return Element("vector-" + scalar.family, scalar.degree, scalar.cell_shape, (2,),
                   2 * scalar.ndof, "identity", ent, dof_entity, pts, wts, perm, sign,
                   scalar=scalar)


def _hdiv_modal(family, k):
    """Modal spanning set of BDM_k (vector P_k) or RT_k (vector P_{k-1} +
    x * homogeneous P_{k-1}), as (vals (nq, np, 2), grads (nq, np, 2, 2))."""
    deg = k if family == "bdm-tri" else k - 1
    extra = 0 if family == "bdm-tri" else k
    nb = (deg + 1) * (deg + 2) // 2

    def modal(pts):
        sv, sg = dubiner(deg, pts)
        nq = len(pts)
        vals = np.zeros((nq, 2 * nb + extra, 2))
        grads = np.zeros((nq, 2 * nb + extra, 2, 2))
        for comp in (0, 1):
            vals[:, comp:2 * nb:2, comp] = sv
            grads[:, comp:2 * nb:2, comp, :] = sg
        x, y = pts[:, 0], pts[:, 1]
        for a in range(extra):
            b = k - 1 - a
            m = x ** a * y ** b
            mx = a * x ** (a - 1) * y ** b if a else np.zeros_like(x)
            my = b * x ** a * y ** (b - 1) if b else np.zeros_like(x)
            col = 2 * nb + a
            vals[:, col] = np.column_stack([x * m, y * m])
            grads[:, col, 0] = np.column_stack([m + x * mx, x * my])
            grads[:, col, 1] = np.column_stack([y * mx, m + y * my])
        return vals, grads
    return modal, 2 * nb + extra


def _apply_functionals(points, weights, modal):
    """Matrix of functionals (rows) applied to the modal set (columns)."""
    rows = []
    for p, w in zip(points, weights):
        vals, _ = modal(p)
        rows.append(np.einsum("qv,qpv->p", w, vals))
    return np.array(rows)


def hdiv(family: str, k: int) -> Element:
    """Normal-moment H(div) elements on the triangle (reference
    ``elements.py:372-447``): per edge slot, length-normalised moments of the
    normal component against Legendre P_0..P_{npe-1}; interior DoFs =
    moments against an L2-orthonormal basis of the zero-normal-trace
    subspace (null space of the edge functionals, orthonormalised by
    Cholesky of its Gram matrix)."""
    modal, nprime = _hdiv_modal(family, k)
    npe = k + 1 if family == "bdm-tri" else k
    s, w = _gauss01(max(k + 2, 10))
    pts, wts, owner = [], [], []
    lengths = np.empty(3)
    for e, (la, lb) in enumerate(TRI_SLOTS):
        va, vb = TRI_REF[la], TRI_REF[lb]
        lengths[e] = np.linalg.norm(vb - va)
        t = (vb - va) / lengths[e]
        nrm = np.array([t[1], -t[0]])
        ep = va + s[:, None] * (vb - va)
        for mm in range(npe):
            pts.append(ep)
            wts.append((w * eval_legendre(mm, 2.0 * s - 1.0))[:, None] * nrm[None, :])
            owner.append((1, e))
    nedge = len(pts)
    nint = nprime - nedge
    if nint > 0:
        emat = _apply_functionals(pts, wts, modal)
        bub = null_space(emat)
        if bub.shape[1] != nint:
            raise RuntimeError(f"{family} order {k}: interior space has dimension "
                               f"{bub.shape[1]}, expected {nint}")
        g = quadrature("tri", min(2 * k + 2, MAX_QUAD_DEGREE))
        gv, _ = modal(g.points)
        gram = np.einsum("q,qpv,qrv->pr", g.weights, gv, gv)
        chol = np.linalg.cholesky(bub.T @ gram @ bub)
        bub = bub @ np.linalg.inv(chol).T
        iq = quadrature("tri", MAX_QUAD_DEGREE)
        iv, _ = modal(iq.points)
        fields = np.einsum("qpv,pj->qjv", iv, bub)
        for j in range(nint):
            pts.append(iq.points)
            wts.append(iq.weights[:, None] * fields[:, j, :])
            owner.append((2, 0))
    coeffs = np.linalg.inv(_apply_functionals(pts, wts, modal))
    ent, dof_entity = _entity_tables(owner, (3, 3, 1))
    return Element(family, k, "tri", (2,), len(pts), "piola", ent, dof_entity, pts, wts,
                   np.arange(npe), np.array([(-1.0) ** (mm + 1) for mm in range(npe)]),
                   modal, coeffs, True, lengths)


_ELEMENTS: dict = {}


def element(family: str, k: int) -> Element:
    """Cached reference element: lagrange-tri / lagrange-quad / dlagrange-tri
    / vector-lagrange-tri / vector-lagrange-quad / bdm-tri / rt-tri."""
    key = (family, k)
    if key not in _ELEMENTS:
        if family in ("lagrange-tri", "lagrange-quad"):
            el = lagrange(family.split("-")[1], k)
        elif family == "dlagrange-tri":
            el = lagrange("tri", k, discontinuous=True)
        elif family.startswith("vector-"):
            el = vector(element(family[len("vector-"):], k))
        elif family in ("bdm-tri", "rt-tri"):
            el = hdiv(family, k)
        else:
            raise ValueError(f"unknown element family {family!r}")
        _ELEMENTS[key] = el
    return _ELEMENTS[key]


# ============================================================================
# cell maps
# ============================================================================

def cell_jacobians(shape, vertices, pts):
    """Per-point Jacobian (nq, 2, 2), determinant and inverse of the affine
    (triangle) / bilinear (square) reference map with the given vertices."""
    v = np.asarray(vertices, dtype=float)
    pts = np.atleast_2d(pts)
    jac = np.broadcast_to(np.column_stack([v[1] - v[0], v[2] - v[0]]),
                          (len(pts), 2, 2)).copy()
    if shape == "quad":
        tw = v[0] - v[1] - v[2] + v[3]
        jac[:, :, 0] += np.outer(pts[:, 1], tw)
        jac[:, :, 1] += np.outer(pts[:, 0], tw)
    det = jac[:, 0, 0] * jac[:, 1, 1] - jac[:, 0, 1] * jac[:, 1, 0]
    inv = np.stack([np.stack([jac[:, 1, 1], -jac[:, 0, 1]], -1),
                    np.stack([-jac[:, 1, 0], jac[:, 0, 0]], -1)], 1) / det[:, None, None]
    return jac, det, inv


def map_points(shape, vertices, pts):
    v = np.asarray(vertices, dtype=float)
    pts = np.atleast_2d(pts)
    out = v[0] + pts @ np.column_stack([v[1] - v[0], v[2] - v[0]]).T
    if shape == "quad":
        out = out + np.outer(pts[:, 0] * pts[:, 1], v[0] - v[1] - v[2] + v[3])
    return out


def inverse_map(shape, vertices, phys):
    v = np.asarray(vertices, dtype=float)
    phys = np.atleast_2d(phys)
    jac = np.column_stack([v[1] - v[0], v[2] - v[0]])
    ref = np.linalg.solve(jac, (phys - v[0]).T).T
    if shape == "quad" and not np.allclose(v[0] - v[1] - v[2] + v[3], 0.0, atol=1e-14):
        for _ in range(30):
            res = map_points(shape, v, ref) - phys
            if np.max(np.abs(res)) < 1e-14:
                break
            _, _, inv = cell_jacobians(shape, v, ref)
            ref = ref - np.einsum("qab,qb->qa", inv, res)
    return ref


def push_forward(el: Element, shape, vertices, pts, tab):
    """Reference basis values / gradients -> physical cell (identity map:
    gradients by J^-T; Piola: J v / det, gradients accordingly)."""
    vals, grads = tab
    jac, det, inv = cell_jacobians(shape, vertices, pts)
    if el.mapping == "identity":
        if el.value_shape == ():
            return vals, np.einsum("qib,qba->qia", grads, inv)
        return vals, np.einsum("qicb,qba->qica", grads, inv)
    pv = np.einsum("qcd,qid->qic", jac, vals) / det[:, None, None]
    pg = np.einsum("qcd,qidb,qba->qica", jac, grads, inv) / det[:, None, None, None]
    return pv, pg


# ============================================================================
# global function spaces
# ============================================================================

@dataclass
class Space:
    """Reference ``FunctionSpace`` attribute names (``spaces.py:25-38``)."""
    mesh: Mesh
    element: Element
    ndof: int
    entity_dofs: dict
    cell_dofs: np.ndarray
    cell_dof_scale: np.ndarray
    boundary_dof: np.ndarray


@dataclass
class Mixed:
    """Reference ``MixedSpace`` (``spaces.py:41-54``)."""
    velocity: Space
    pressure: Space
    case: str
    order: int

    @property
    def offset(self) -> int:
        return self.velocity.ndof

    @property
    def ndof(self) -> int:
        return self.velocity.ndof + self.pressure.ndof


def build_space(mesh: Mesh, el: Element) -> Space:
    """Entity-blocked numbering (vertices, edges, cells), edge DoFs permuted /
    signed by the edge orientation, H(div) DoFs length / area normalised
    (reference ``spaces.py:63-124``)."""
    topo, geom = mesh
    per = [len(el.entity_dofs[d][0]) if el.entity_dofs[d] else 0 for d in range(3)]
    counts = [topo.num_vertices, topo.num_edges, topo.num_cells]
    offs = np.concatenate([[0], np.cumsum([per[d] * counts[d] for d in range(3)])])
    ent = {d: offs[d] + per[d] * np.arange(counts[d])[:, None] + np.arange(per[d])[None, :]
           for d in range(3)}
    nc = topo.num_cells
    cell_dofs = np.empty((nc, el.ndof), dtype=np.int64)
    scale = np.ones((nc, el.ndof))
    fperm, fsign = el.edge_transform(True)
    rperm, rsign = el.edge_transform(False)
    if el.length_normalized:
        v = geom.vertex_coords[geom.cell_map_vertices]
        j = np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]], -1)
        area_scale = np.sqrt(np.linalg.det(j))
    for i, (dim, e, pos) in enumerate(el.dof_entity):
        if dim == 0:
            cell_dofs[:, i] = ent[0][geom.cell_map_vertices[:, e], pos]
        elif dim == 1:
            edges = geom.cell_edge_ids[:, e]
            al = geom.cell_edge_aligned[:, e]
            cell_dofs[:, i] = ent[1][edges, np.where(al, fperm[pos], rperm[pos])]
            scale[:, i] = np.where(al, fsign[pos], rsign[pos])
            if el.length_normalized:
                scale[:, i] *= geom.edge_length[edges] / el.edge_ref_lengths[e]
        else:
            cell_dofs[:, i] = ent[2][:, pos]
            if el.length_normalized:
                scale[:, i] = area_scale
    bdof = np.zeros(int(offs[-1]), dtype=bool)
    if per[0]:
        bdof[ent[0][topo.boundary_vertex].ravel()] = True
    if per[1]:
        bdof[ent[1][topo.boundary_edge].ravel()] = True
    return Space(mesh, el, int(offs[-1]), ent, cell_dofs, scale, bdof)


def build_mixed(case: str, mesh: Mesh, k: int) -> Mixed:
    """Velocity-pressure pair (reference ``spaces.py:127-151``)."""
    if case not in CASES:
        raise ValueError(f"unknown case {case!r}")
    shape = mesh.topology.cell_shape
    if case in ("th-tri", "th-quad"):
        want = "tri" if case == "th-tri" else "quad"
        if shape != want or k < 2:
            raise ValueError(f"{case} needs a {want} mesh and order >= 2")
        vel = element(f"vector-lagrange-{shape}", k)
        pres = element(f"lagrange-{shape}", k - 1)
    else:
        if shape != "tri" or k < 1:
            raise ValueError("normal-continuity pairs need a triangular mesh and order >= 1")
        vel = element("bdm-tri" if case == "bdm" else "rt-tri", k)
        pres = element("dlagrange-tri", k - 1)
    return Mixed(build_space(mesh, vel), build_space(mesh, pres), case, k)


@dataclass
class StrongBc:
    """Reference ``StrongBc`` (``spaces.py:57-60``): constrained velocity
    DoFs = every DoF on a boundary entity (Dirichlet) / the boundary normal
    moments (normal flux) — the same index set for both modes."""
    indices: np.ndarray
    values: np.ndarray


def strong_bc(space: Space) -> StrongBc:
    idx = np.flatnonzero(space.boundary_dof)
    return StrongBc(idx, np.zeros(len(idx)))
