"""Host-side logic of the device patch builder, checked on CPU: the candidate
arrays handed to vk_patches_build (entity -> cells incidence, pressure DoFs,
constrained mask), fed through a numpy emulation of the K1 kernel's
semantics, must reproduce the reference patch lists bit-exactly."""

import numpy as np
import pytest

from conftest import SMALL_MG, golden_weights, load_case
from paper_2409_14222_b200.vanka import (_constrained_mask, hdiv_candidates,
                                         taylor_hood_candidates)


def emulate_k1(cell_dofs, e2c_ptr, e2c, pptr, pdofs, constrained):
    """numpy restatement of build_stage_kernel + fill (not the oracle: the
    oracle works from the topology; this works from the flattened arrays)."""
    offs, idx, nv = [0], [], []
    for p in range(len(e2c_ptr) - 1):
        cells = e2c[e2c_ptr[p]:e2c_ptr[p + 1]]
        d = np.unique(cell_dofs[cells].ravel())
        v = d[constrained[d] == 0]
        pr = np.sort(pdofs[pptr[p]:pptr[p + 1]])
        if len(v) + len(pr) == 0:
            continue
        idx.append(np.concatenate([v, pr]))
        nv.append(len(v))
        offs.append(offs[-1] + len(v) + len(pr))
    return np.array(offs), np.concatenate(idx), np.array(nv)


@pytest.mark.parametrize("name", ["cfg1"] + SMALL_MG)
def test_candidates_reproduce_reference_patches(name):
    pack, g = load_case(name)
    mixed = pack.fine.mixed
    cand = (taylor_hood_candidates(mixed) if mixed.case in ("th-tri", "th-quad")
            else hdiv_candidates(mixed))
    e2c_ptr, e2c, pptr, pdofs, ents = cand
    con = _constrained_mask(mixed.ndof, pack.fine.system.bc)
    offs, idx, nv = emulate_k1(np.asarray(mixed.velocity.cell_dofs), e2c_ptr, e2c, pptr,
                               pdofs, con)
    assert np.array_equal(offs, g["patch_offsets"])
    assert np.array_equal(idx, g["patch_indices"])
    assert np.array_equal(nv, g["patch_nvel"])
    ent = np.array([(ents[k].dim, ents[k].index) for k in range(len(ents))])
    assert np.array_equal(ent, g["patch_entity"])   # no empty candidates here
    # multiplicity / weights exactly as the weights kernel computes them
    mult = np.bincount(idx, minlength=mixed.ndof).astype(float)
    assert np.array_equal(mult, g["multiplicity"])
    w = np.ones(len(idx))
    pos = np.arange(len(idx)) - np.repeat(offs[:-1], np.diff(offs))
    isvel = pos < np.repeat(nv, np.diff(offs))
    w[isvel] = 1.0 / mult[idx[isvel]]
    assert np.array_equal(w.view(np.uint64), golden_weights(g).view(np.uint64))


def test_candidate_capacity_fits_kernel():
    # every BASELINE discretisation stays within the 1024-entry stage
    for name in ["cfg1", "s_thtri4", "s_thquad3", "s_bdm3"]:
        pack, _ = load_case(name)
        mixed = pack.fine.mixed
        cand = (taylor_hood_candidates(mixed) if mixed.case in ("th-tri", "th-quad")
                else hdiv_candidates(mixed))
        e2c_ptr, _, pptr, _, _ = cand
        nloc = mixed.velocity.cell_dofs.shape[1]
        worst = np.max(np.diff(e2c_ptr) * nloc + np.diff(pptr))
        assert worst <= 1024
