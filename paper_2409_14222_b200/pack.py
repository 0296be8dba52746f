"""Problem packs: the assembled inputs the hot path consumes, serialised.

The hot path starts from an *assembled* global saddle-point CSR
matrix plus the topology / DoF maps that patch construction reads.  Producing
those (structured meshes, finite elements, assembly, natural-embedding
prolongation: reference ``meshtopo.py``, ``elements.py``, ``spaces.py``,
``assembly.py``, ``mg.py:91-234``) is out of scope, so a pack freezes exactly
what the reference hands to the hot path, level by level:

* ``A``      — ``BlockSystem.matrix`` (reference ``assembly.py:273-285``)
* ``P``      — ``TransferPair.masked`` (reference ``mg.py:159-167``)
* ``bc``     — ``StrongBc.indices`` (reference ``spaces.py:203-220``)
* ``cell_dofs`` / ``pres_ed{d}`` — ``FunctionSpace.cell_dofs`` /
  ``entity_dofs`` (reference ``spaces.py:63-124``)
* ``vertex_cells`` / ``edge_cells`` / ``cell_edges`` — ``MeshTopology``
  adjacency (reference ``meshtopo.py:35-50``)

Packs are written by ``tools/make_packs.py`` (which imports the reference in the
build container) and read here with numpy only, so the GPU box never needs the
reference.  CSR matrices are stored losslessly: row lengths, delta-coded column
indices and a bit-pattern dictionary of the values (structured meshes repeat a
few hundred distinct entries), then deflated by ``np.savez_compressed``.

The light classes below carry the same attribute names as the reference's
``MixedSpace`` / ``FunctionSpace`` / ``MeshTopology`` / ``StrongBc`` /
``BlockSystem`` so that every host entry point accepts either.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

PACK_VERSION = 1


# ----------------------------------------------------------------------------
# lossless CSR codec
# ----------------------------------------------------------------------------

def encode_csr(prefix: str, a) -> dict:
    a = sp.csr_matrix(a)
    if not a.has_sorted_indices:
        a = a.sorted_indices()
    indptr = a.indptr.astype(np.int64)
    rowlen = np.diff(indptr)
    cols = a.indices.astype(np.int64)
    rows = np.repeat(np.arange(a.shape[0], dtype=np.int64), rowlen)
    d = np.empty_like(cols)
    if cols.size:
        d[1:] = cols[1:] - cols[:-1]
        d[0] = cols[0]
        first = indptr[:-1][rowlen > 0]
        d[first] = cols[first] - rows[first]
    bits = np.ascontiguousarray(a.data, dtype=np.float64).view(np.uint64)
    out = {
        f"{prefix}_shape": np.array(a.shape, dtype=np.int64),
        f"{prefix}_rowlen": rowlen.astype(np.int32),
        f"{prefix}_dcol": d.astype(np.int32),
    }
    uniq, codes = np.unique(bits, return_inverse=True)
    if uniq.size * 4 < bits.size:
        out[f"{prefix}_vals"] = uniq
        out[f"{prefix}_code"] = codes.astype(np.int32)
    else:
        out[f"{prefix}_bits"] = bits
    return out


def decode_csr(prefix: str, z) -> sp.csr_matrix:
    shape = tuple(int(v) for v in z[f"{prefix}_shape"])
    rowlen = z[f"{prefix}_rowlen"].astype(np.int64)
    indptr = np.zeros(shape[0] + 1, dtype=np.int64)
    np.cumsum(rowlen, out=indptr[1:])
    d = z[f"{prefix}_dcol"].astype(np.int64)
    if d.size:
        starts = indptr[:-1][rowlen > 0]
        rows_nz = np.flatnonzero(rowlen > 0)
        d = d.copy()
        d[starts] += rows_nz
        total = np.cumsum(d)
        before = np.zeros(shape[0], dtype=np.int64)
        has_prev = indptr[:-1] > 0
        before[has_prev] = total[indptr[:-1][has_prev] - 1]
        # segment start values already absolute: remove the running prefix
        cols = total - np.repeat(before, rowlen)
    else:
        cols = d
    if f"{prefix}_vals" in z:
        bits = z[f"{prefix}_vals"][z[f"{prefix}_code"]]
    else:
        bits = z[f"{prefix}_bits"]
    data = np.ascontiguousarray(bits, dtype=np.uint64).view(np.float64)
    return sp.csr_matrix((data, cols.astype(np.int32), indptr.astype(np.int32)),
                         shape=shape)


def _ragged_to_csr(lists) -> tuple[np.ndarray, np.ndarray]:
    lens = np.fromiter((len(x) for x in lists), dtype=np.int64, count=len(lists))
    ptr = np.zeros(len(lists) + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    idx = np.fromiter((v for x in lists for v in x), dtype=np.int64,
                      count=int(ptr[-1]))
    return ptr.astype(np.int32), idx.astype(np.int32)


class _Ragged(list):
    """List-of-lists view over a CSR pair (reference ``edge_cells`` style)."""

    def __init__(self, ptr, idx):
        super().__init__(idx[ptr[i]:ptr[i + 1]].tolist()
                         for i in range(len(ptr) - 1))
        self.ptr = np.asarray(ptr, dtype=np.int32)
        self.idx = np.asarray(idx, dtype=np.int32)


# ----------------------------------------------------------------------------
# light stand-ins with the reference's attribute names
# ----------------------------------------------------------------------------

@dataclass
class LiteTopology:
    """Subset of reference ``MeshTopology`` (``meshtopo.py:35-56``)."""
    cell_shape: str
    cells_per_side: int
    num_vertices: int
    num_edges: int
    num_cells: int
    cell_edges: np.ndarray
    vertex_cells_ptr: np.ndarray
    vertex_cells_idx: np.ndarray
    edge_cells_ptr: np.ndarray
    edge_cells_idx: np.ndarray

    def entity_count(self, dim: int) -> int:
        return (self.num_vertices, self.num_edges, self.num_cells)[dim]

    @property
    def vertex_cells(self):
        return _Ragged(self.vertex_cells_ptr, self.vertex_cells_idx)

    @property
    def edge_cells(self):
        return _Ragged(self.edge_cells_ptr, self.edge_cells_idx)


@dataclass
class LiteMesh:
    topology: LiteTopology


@dataclass
class LiteSpace:
    """Subset of reference ``FunctionSpace`` (``spaces.py:25-38``)."""
    mesh: LiteMesh
    ndof: int
    entity_dofs: dict
    cell_dofs: np.ndarray | None = None


@dataclass
class LiteMixed:
    """Subset of reference ``MixedSpace`` (``spaces.py:41-54``)."""
    velocity: LiteSpace
    pressure: LiteSpace
    case: str
    order: int

    @property
    def offset(self) -> int:
        return self.velocity.ndof

    @property
    def ndof(self) -> int:
        return self.velocity.ndof + self.pressure.ndof


@dataclass
class LiteBc:
    """Reference ``StrongBc`` (``spaces.py:57-60``); values are irrelevant to
    the operator (identity rows, ``assembly.py:273-285``)."""
    indices: np.ndarray
    values: np.ndarray | None = None


@dataclass
class LiteSystem:
    """Reference ``BlockSystem`` (``assembly.py:38-51``) without rhs."""
    matrix: sp.csr_matrix
    mixed: LiteMixed
    bc: LiteBc | None
    rhs: np.ndarray | None = None

    @property
    def num_velocity(self) -> int:
        return self.mixed.velocity.ndof

    @property
    def num_pressure(self) -> int:
        return self.mixed.pressure.ndof


@dataclass
class PackLevel:
    mixed: LiteMixed
    system: LiteSystem
    prolong: sp.csr_matrix | None       # masked P: this level <- coarser level


@dataclass
class ProblemPack:
    case: str
    order: int
    levels: list                          # levels[0] is the coarsest
    meta: dict = field(default_factory=dict)

    @property
    def fine(self) -> PackLevel:
        return self.levels[-1]


# ----------------------------------------------------------------------------
# writer (build container only: takes reference objects) and reader
# ----------------------------------------------------------------------------

def level_arrays(i: int, mixed, system, masked=None) -> dict:
    """Flatten one reference level into pack arrays (duck-typed)."""
    vel, pres = mixed.velocity, mixed.pressure
    topo = vel.mesh.topology
    p = f"L{i}"
    out = {}
    out.update(encode_csr(f"{p}_A", system.matrix))
    if masked is not None:
        out.update(encode_csr(f"{p}_P", masked))
    bc = system.bc.indices if system.bc is not None else np.zeros(0, np.int64)
    out[f"{p}_bc"] = np.asarray(bc, dtype=np.int32)
    out[f"{p}_cell_dofs"] = np.asarray(vel.cell_dofs, dtype=np.int32)
    for d in range(3):
        out[f"{p}_pres_ed{d}"] = np.asarray(pres.entity_dofs[d], dtype=np.int32)
        out[f"{p}_vel_ed{d}"] = np.asarray(vel.entity_dofs[d].shape,
                                           dtype=np.int64)
    vptr, vidx = _ragged_to_csr(topo.vertex_cells)
    eptr, eidx = _ragged_to_csr(topo.edge_cells)
    out[f"{p}_vc_ptr"], out[f"{p}_vc_idx"] = vptr, vidx
    out[f"{p}_ec_ptr"], out[f"{p}_ec_idx"] = eptr, eidx
    out[f"{p}_cell_edges"] = np.asarray(topo.cell_edges, dtype=np.int32)
    out[f"{p}_meta"] = np.array([topo.cells_per_side, topo.num_vertices,
                                 topo.num_edges, topo.num_cells, vel.ndof,
                                 pres.ndof], dtype=np.int64)
    out[f"{p}_shape"] = np.array(topo.cell_shape)
    return out


def write_pack(path, case: str, order: int, levels, extra_meta=None) -> None:
    """``levels``: list of (mixed, system, masked_or_None), coarsest first."""
    arrays = {"version": np.array(PACK_VERSION), "case": np.array(case),
              "order": np.array(order), "num_levels": np.array(len(levels))}
    for i, (mixed, system, masked) in enumerate(levels):
        arrays.update(level_arrays(i, mixed, system, masked))
    for key, val in (extra_meta or {}).items():
        arrays[f"meta_{key}"] = np.asarray(val)
    np.savez_compressed(path, **arrays)


def _read_level(z, i: int, case: str, order: int) -> PackLevel:
    p = f"L{i}"
    n, nv, ne, nc, nvel, npres = (int(v) for v in z[f"{p}_meta"])
    topo = LiteTopology(str(z[f"{p}_shape"]), n, nv, ne, nc,
                        z[f"{p}_cell_edges"], z[f"{p}_vc_ptr"],
                        z[f"{p}_vc_idx"], z[f"{p}_ec_ptr"], z[f"{p}_ec_idx"])
    mesh = LiteMesh(topo)
    pres_ed = {d: z[f"{p}_pres_ed{d}"].astype(np.int64) for d in range(3)}
    vel_ed = {}
    for d in range(3):
        cnt, width = (int(v) for v in z[f"{p}_vel_ed{d}"])
        vel_ed[d] = np.zeros((cnt, width), dtype=np.int64)  # shape only
    vel = LiteSpace(mesh, nvel, vel_ed, z[f"{p}_cell_dofs"].astype(np.int64))
    pres = LiteSpace(mesh, npres, pres_ed)
    mixed = LiteMixed(vel, pres, case, order)
    bc = LiteBc(z[f"{p}_bc"].astype(np.int64))
    system = LiteSystem(decode_csr(f"{p}_A", z), mixed, bc)
    prolong = decode_csr(f"{p}_P", z) if f"{p}_P_shape" in z else None
    return PackLevel(mixed, system, prolong)


def read_pack(path_or_bytes) -> ProblemPack:
    src = io.BytesIO(path_or_bytes) if isinstance(path_or_bytes, bytes) \
        else path_or_bytes
    with np.load(src, allow_pickle=False) as z:
        case = str(z["case"])
        order = int(z["order"])
        nl = int(z["num_levels"])
        levels = [_read_level(z, i, case, order) for i in range(nl)]
        meta = {k[5:]: z[k] for k in z.files if k.startswith("meta_")}
    return ProblemPack(case, order, levels, meta)
