"""Reference-default Chebyshev bounds on the device.

The reference estimates every relaxed level's lam with ``estimate_lambda_max``
on A * apply_additive (``mg.py:214-221``, ``sparsela.py:194-226``); the
goldens (tools/make_spectra_golden.py) hold the reference's own lam per level
and its MG-FGMRES(30) history with those bounds, for both Chebyshev modes.

Gates: lam relative 1e-10 (10 Arnoldi steps on operators that differ from
the reference by ~1e-16 per application); history as test_gpu_parity:
iterations +-1 and max(1e-10, the reference's own floor recorded in the
golden: the largest history change the reference shows when only its coarse
solve is replaced by another valid factorization).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_case

RUNS = sorted(f[:-len("_spectra.json")] for f in os.listdir(GOLDEN) if f.endswith("_spectra.json"))
REL_LAM = 1e-10
REL_HIST = 1e-10


def _golden(run):
    with open(os.path.join(GOLDEN, f"{run}_spectra.json")) as fh:
        return json.load(fh)


def test_spectra_goldens_present():
    assert len(RUNS) >= 8
    for run in RUNS:
        g = _golden(run)
        assert g["lam"][0] is None and all(l > 0 for l in g["lam"][1:])
        assert g["converged"] and len(g["history"]) == g["iterations"] + 1
        assert g["history"][0] == 1.0


@pytest.mark.gpu
@pytest.mark.parametrize("run", RUNS)
def test_device_spectra_and_fgmres(run, capsys):
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.solver import FgmresSolver, mg_rhs
    g = _golden(run)
    name = g["name"]
    pack, _ = load_case(name)
    hier = V.hierarchy_from_pack(pack, cheb_mode=g["mode"], damping=None,
                                 est_steps=g["est_steps"], seed=g["seed"])
    lam = [lv.cheb.lam if lv.cheb is not None else None for lv in hier.levels]
    rel_lam = max(abs(a - b) / b for a, b in zip(lam[1:], g["lam"][1:]))
    x, its, conv, hist = FgmresSolver(hier).solve(mg_rhs(pack))
    ref = np.asarray(g["history"])
    m = min(len(hist), len(ref))
    rel = float(np.max(np.abs(hist[:m] - ref[:m]) / ref[:m]))
    floor = g["selfvar_history_max_rel"]
    tol = max(REL_HIST, floor)
    with capsys.disabled():
        print(f"\n[{run}] lam rel {rel_lam:.2e}; iterations {its} (ref {g['iterations']}); "
              f"history rel {rel:.2e} (strict 1e-10: {'pass' if rel <= REL_HIST else 'FAIL'}; "
              f"reference floor {floor:.2e}; tolerance {tol:.2e})")
    assert rel_lam <= REL_LAM
    assert conv and abs(its - g["iterations"]) <= 1
    assert rel <= tol
