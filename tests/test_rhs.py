"""Right-hand side of the manufactured problem (reference assembly.py:
136-172 load, 273-285 lift, spaces.py:170-220 boundary values) against the
reference's own vectors (tests/golden/rhs_golden.npz, tools/make_rhs_golden.py).

* host: Taylor-Hood boundary values by the elements' dual functionals —
  bit-exact with the reference (same numpy operations on the pinned element
  / mesh restatement); H(div) cases constrain to zero.
* device (gpu): the assembled rhs within 1e-13 of max |rhs| per entry (the
  forcing's sin / cos and the load's summation differ from numpy's in the
  last bits; the lift goes through the unconstrained operator, whose entries
  agree with the reference's to rounding).
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "rhs_golden.npz")
CASES = ["cfg1", "s_thtri2", "s_thtri4", "s_thquad3", "s_bdm3", "s_rt2", "s_thquad2",
         "t_thquad3_5", "t_bdm1_5", "t_rt1_5", "t_thtri3_3", "t_bdm2_3"]
CASE_OF = {"cfg1": "th-tri", "s_thtri2": "th-tri", "s_thtri4": "th-tri", "s_thquad3": "th-quad",
           "s_bdm3": "bdm", "s_rt2": "rt", "s_thquad2": "th-quad", "t_thquad3_5": "th-quad",
           "t_bdm1_5": "bdm", "t_rt1_5": "rt", "t_thtri3_3": "th-tri", "t_bdm2_3": "bdm"}


def _mixed(name, g):
    from paper_2409_14222_b200 import fem
    n, k = (int(v) for v in g[f"{name}_spec"])
    case = CASE_OF[name]
    shape = "quad" if case == "th-quad" else "tri"
    return fem.build_mixed(case, fem.structured_mesh(shape, n), k), case


@pytest.mark.parametrize("name", CASES)
def test_boundary_values_match_reference(name):
    from paper_2409_14222_b200 import fem
    from paper_2409_14222_b200.assembly import interpolate_boundary, manufactured_velocity
    g = np.load(GOLD)
    mixed, case = _mixed(name, g)
    bc = fem.strong_bc(mixed.velocity)
    assert np.array_equal(bc.indices, g[f"{name}_bc_indices"])
    if case in ("th-tri", "th-quad"):
        vals = interpolate_boundary(mixed.velocity, manufactured_velocity)[bc.indices]
    else:
        vals = bc.values
    ref = g[f"{name}_bc_values"]
    assert np.array_equal(vals.view(np.uint64), ref.view(np.uint64)), \
        float(np.max(np.abs(vals - ref)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_rhs_matches_reference(name, capsys):
    from paper_2409_14222_b200.assembly import assemble
    g = np.load(GOLD)
    mixed, _ = _mixed(name, g)
    system = assemble(mixed)
    b = system.rhs.cpu().numpy()
    ref = g[f"{name}_rhs"]
    scale = np.max(np.abs(ref))
    err = float(np.max(np.abs(b - ref)) / scale)
    idx = g[f"{name}_bc_indices"]
    assert np.array_equal(b[idx].view(np.uint64), ref[idx].view(np.uint64))
    with capsys.disabled():
        print(f"\n[{name}] rhs max |b - b_ref| / max |b_ref| = {err:.2e}")
    assert err <= 1e-13, err
