import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "data")
sys.path.insert(0, ROOT)

SMALL_MG = ["s_thtri2", "s_thtri4", "s_thquad3", "s_thquad2", "s_bdm3", "s_rt2"]
FULL_MG = ["cfg2", "cfg3", "cfg4", "cfg5"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "full: BASELINE-size configs (data/ packs)")


def case_paths(name):
    d = GOLDEN if name not in FULL_MG else DATA
    return os.path.join(d, f"{name}_pack.npz"), os.path.join(d, f"{name}_golden.npz")


_PACKS = {}


def load_case(name):
    """(pack, golden dict) for a named case; full configs skip if absent."""
    if name in _PACKS:
        return _PACKS[name]
    from paper_2409_14222_b200.pack import read_pack
    pp, gp = case_paths(name)
    for p in (pp, gp):
        if not os.path.exists(p):
            pytest.skip(f"{p} not present (generate with tools/make_packs.py)")
    g = dict(np.load(gp))
    hp = os.path.join(GOLDEN, f"{name}_history.json")
    if os.path.exists(hp):
        g["info"] = json.load(open(hp))
    _PACKS[name] = (read_pack(pp), g)
    return _PACKS[name]


def seeded_residual(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def golden_residual(name, g, n):
    """The residual the golden sweep used (cfg1: seed 0; MG cases: seed 1)."""
    if "r" in g:
        return g["r"]
    return seeded_residual(n, 0 if name == "cfg1" else 1)


def golden_weights(g):
    if "patch_weights" in g:
        return g["patch_weights"]
    off, idx, nv, m = g["patch_offsets"], g["patch_indices"], g["patch_nvel"], g["multiplicity"]
    pos = np.arange(len(idx)) - np.repeat(off[:-1], np.diff(off))
    isvel = pos < np.repeat(nv, np.diff(off))
    w = np.ones(len(idx))
    w[isvel] = 1.0 / m[idx[isvel]]
    return w
