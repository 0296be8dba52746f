#!/usr/bin/env python
"""Golden fixtures for the host discretisation restatement (build container
only: imports the unmodified reference from /root/reference).

Dumps, from the reference's own meshtopo / elements / spaces modules, the
mesh numbering and geometry, refinement links, quadrature rules, reference
element tabulations at fixed points and the global DoF maps of every
(case, order) the BASELINE configs and the small parity cases use, into
tests/golden/fem_golden.npz (tests/test_fem.py compares
paper_2409_14222_b200/fem.py against it bit for bit).

    python tools/make_fem_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")

MESHES = [("tri", 3), ("tri", 4), ("quad", 3), ("quad", 4)]
ELEMENTS = [("lagrange-tri", 1), ("lagrange-tri", 2), ("lagrange-tri", 3), ("lagrange-tri", 4),
            ("lagrange-quad", 1), ("lagrange-quad", 2), ("lagrange-quad", 3),
            ("dlagrange-tri", 0), ("dlagrange-tri", 1), ("dlagrange-tri", 2),
            ("bdm-tri", 1), ("bdm-tri", 2), ("bdm-tri", 3), ("rt-tri", 1), ("rt-tri", 2)]
SPACES = [("th-tri", 2, "tri", 4), ("th-tri", 4, "tri", 3), ("th-quad", 3, "quad", 4),
          ("th-quad", 2, "quad", 3), ("bdm", 3, "tri", 4), ("rt", 2, "tri", 3), ("bdm", 1, "tri", 3)]
QUADS = [("interval", 8), ("tri", 6), ("tri", 10), ("tri", 20), ("quad", 8)]


def main():
    import stokesmg.elements as E
    import stokesmg.meshtopo as M
    import stokesmg.spaces as S
    out = {}
    pts = np.random.default_rng(0).uniform(0.0, 0.5, (9, 2))
    out["tab_points"] = pts
    for shape, n in MESHES:
        mesh = (M.build_structured_tri if shape == "tri" else M.build_structured_quad)(n)
        t, g = mesh
        p = f"mesh_{shape}{n}"
        for name in ("cell_vertices", "cell_edges", "edge_vertices", "boundary_vertex",
                     "boundary_edge"):
            out[f"{p}_{name}"] = np.asarray(getattr(t, name))
        for name in ("vertex_coords", "edge_length", "edge_tangent", "edge_normal",
                     "cell_map_vertices", "cell_edge_ids", "cell_edge_aligned"):
            out[f"{p}_{name}"] = np.asarray(getattr(g, name))
        for name in ("edge_cells", "vertex_cells"):
            lists = getattr(t, name)
            out[f"{p}_{name}_len"] = np.array([len(x) for x in lists])
            out[f"{p}_{name}_idx"] = np.concatenate([np.asarray(x) for x in lists])
        out[f"{p}_children"] = M.refine_uniform(mesh)[1].parent_cells
    for shape, deg in QUADS:
        r = E.make_quadrature(shape, deg)
        out[f"quad_{shape}{deg}_points"], out[f"quad_{shape}{deg}_weights"] = r.points, r.weights
    for fam, k in ELEMENTS:
        el = E.make_element(fam, k)
        v, gr = E.tabulate(el, pts)
        out[f"el_{fam}{k}_vals"], out[f"el_{fam}{k}_grads"] = v, gr
        out[f"el_{fam}{k}_dof_entity"] = np.array(el.dof_entity)
    for case, k, shape, n in SPACES:
        mesh = (M.build_structured_tri if shape == "tri" else M.build_structured_quad)(n)
        mixed = S.build_mixed(case, mesh, k)
        for sp in ("velocity", "pressure"):
            s = getattr(mixed, sp)
            p = f"sp_{case}{k}_{shape}{n}_{sp}"
            out[f"{p}_cell_dofs"], out[f"{p}_scale"] = s.cell_dofs, s.cell_dof_scale
            out[f"{p}_boundary"] = s.boundary_dof
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "fem_golden.npz"), **out)


if __name__ == "__main__":
    main()
