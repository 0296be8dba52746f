"""Lossless problem-pack codec and light stand-in objects (CPU only)."""

import io

import numpy as np
import scipy.sparse as sp

from conftest import load_case
from paper_2409_14222_b200.pack import decode_csr, encode_csr, read_pack


def _roundtrip(a):
    z = encode_csr("M", a)
    buf = io.BytesIO()
    np.savez_compressed(buf, **z)
    buf.seek(0)
    with np.load(buf) as zz:
        return decode_csr("M", zz)


def _same(a, b):
    a, b = sp.csr_matrix(a), sp.csr_matrix(b)
    return (a.shape == b.shape and np.array_equal(a.indptr, b.indptr)
            and np.array_equal(a.indices, b.indices)
            and np.array_equal(a.data.view(np.uint64), b.data.view(np.uint64)))


def test_codec_random_and_special_values():
    rng = np.random.default_rng(0)
    dense = rng.standard_normal((50, 70)) * (rng.random((50, 70)) < 0.2)
    dense[3, :] = 0.0                       # empty row
    a = sp.csr_matrix(dense)
    a.data[:5] = [-0.0, np.inf, -np.inf, 1e-300, 5e-324]   # explicit specials
    assert _same(_roundtrip(a), a)


def test_codec_dictionary_path():
    # few distinct values -> dictionary coding
    rng = np.random.default_rng(1)
    dense = rng.choice([0.0, 0.0, 0.0, 1.5, -2.25, 3.0], size=(200, 200))
    a = sp.csr_matrix(dense)
    z = encode_csr("M", a)
    assert "M_vals" in z
    assert _same(_roundtrip(a), a)


def test_codec_empty():
    a = sp.csr_matrix((5, 7))
    assert _same(_roundtrip(a), a)


def test_pack_levels_and_topology():
    pack, g = load_case("s_thtri2")
    assert pack.case == "th-tri" and pack.order == 2
    assert len(pack.levels) == 3
    fine = pack.fine
    topo = fine.mixed.velocity.mesh.topology
    assert topo.num_vertices == 17 * 17
    # ragged views agree with the CSR arrays
    vc = topo.vertex_cells
    assert sum(len(x) for x in vc) == len(topo.vertex_cells_idx)
    assert fine.prolong.shape == (fine.system.matrix.shape[0],
                                  pack.levels[1].system.matrix.shape[0])
    assert pack.levels[0].prolong is None
    assert fine.mixed.ndof == fine.system.matrix.shape[0]


def test_read_pack_from_bytes():
    from conftest import case_paths
    pp, _ = case_paths("cfg1")
    with open(pp, "rb") as fh:
        raw = fh.read()
    p = read_pack(raw)
    assert p.fine.system.matrix.nnz == 248168
