"""The host discretisation restatement (paper_2409_14222_b200/fem.py) against
the reference's own meshes, quadrature, elements and DoF maps, bit for bit
(fixtures: tools/make_fem_golden.py from the unmodified reference)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2409_14222_b200 import fem

G = np.load(os.path.join(GOLDEN, "fem_golden.npz"))


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        return a.shape == b.shape and np.array_equal(a.view(np.uint64), np.asarray(b, float).view(np.uint64))
    return np.array_equal(a, b)


@pytest.mark.parametrize("shape,n", [("tri", 3), ("tri", 4), ("quad", 3), ("quad", 4)])
def test_mesh_numbering_and_geometry(shape, n):
    t, g = fem.structured_mesh(shape, n)
    p = f"mesh_{shape}{n}"
    for name in ("cell_vertices", "cell_edges", "edge_vertices", "boundary_vertex",
                 "boundary_edge"):
        assert _eq(getattr(t, name), G[f"{p}_{name}"]), name
    for name in ("vertex_coords", "edge_length", "edge_tangent", "edge_normal",
                 "cell_map_vertices", "cell_edge_ids", "cell_edge_aligned"):
        assert _eq(getattr(g, name), G[f"{p}_{name}"]), name
    for name in ("edge_cells", "vertex_cells"):
        ptr, idx = getattr(t, f"{name}_ptr"), getattr(t, f"{name}_idx")
        assert _eq(np.diff(ptr), G[f"{p}_{name}_len"]) and _eq(idx, G[f"{p}_{name}_idx"])
    assert _eq(fem.refine_links(shape, n), G[f"{p}_children"])


@pytest.mark.parametrize("shape,deg", [("interval", 8), ("tri", 6), ("tri", 10), ("tri", 20),
                                       ("quad", 8)])
def test_quadrature(shape, deg):
    r = fem.quadrature(shape, deg)
    assert _eq(r.points, G[f"quad_{shape}{deg}_points"])
    assert _eq(r.weights, G[f"quad_{shape}{deg}_weights"])


ELEMENTS = [("lagrange-tri", 1), ("lagrange-tri", 2), ("lagrange-tri", 3), ("lagrange-tri", 4),
            ("lagrange-quad", 1), ("lagrange-quad", 2), ("lagrange-quad", 3),
            ("dlagrange-tri", 0), ("dlagrange-tri", 1), ("dlagrange-tri", 2),
            ("bdm-tri", 1), ("bdm-tri", 2), ("bdm-tri", 3), ("rt-tri", 1), ("rt-tri", 2)]


@pytest.mark.parametrize("fam,k", ELEMENTS)
def test_element_tabulation(fam, k):
    el = fem.element(fam, k)
    v, g = el.tabulate(G["tab_points"])
    assert _eq(v, G[f"el_{fam}{k}_vals"]) and _eq(g, G[f"el_{fam}{k}_grads"])
    assert _eq(np.array(el.dof_entity), G[f"el_{fam}{k}_dof_entity"])


@pytest.mark.parametrize("case,k,shape,n", [("th-tri", 2, "tri", 4), ("th-tri", 4, "tri", 3),
                                            ("th-quad", 3, "quad", 4), ("th-quad", 2, "quad", 3),
                                            ("bdm", 3, "tri", 4), ("rt", 2, "tri", 3),
                                            ("bdm", 1, "tri", 3)])
def test_dof_maps(case, k, shape, n):
    mixed = fem.build_mixed(case, fem.structured_mesh(shape, n), k)
    for sp in ("velocity", "pressure"):
        s = getattr(mixed, sp)
        p = f"sp_{case}{k}_{shape}{n}_{sp}"
        assert _eq(s.cell_dofs, G[f"{p}_cell_dofs"]) and _eq(s.cell_dof_scale, G[f"{p}_scale"])
        assert _eq(s.boundary_dof, G[f"{p}_boundary"])


def test_bad_inputs_raise_like_the_reference():
    with pytest.raises(ValueError):
        fem.structured_mesh("tri", 0)
    with pytest.raises(ValueError):
        fem.build_mixed("th-tri", fem.structured_mesh("quad", 2), 2)
    with pytest.raises(ValueError):
        fem.build_mixed("nope", fem.structured_mesh("tri", 2), 2)
    with pytest.raises(ValueError):
        fem.quadrature("tri", 21)
