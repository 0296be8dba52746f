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
    """(pack, golden dict) for a named case.  Full configs: the full-size
    golden in data/ when present, else the committed compact stand-in
    tests/golden/<name>_compact.npz (tools/compact_golden.py: hashes, whole
    small arrays, sampled N-vectors); skip only if neither or no pack."""
    if name in _PACKS:
        return _PACKS[name]
    from paper_2409_14222_b200.pack import read_pack
    pp, gp = case_paths(name)
    if not os.path.exists(pp):
        pytest.skip(f"{pp} not present (generate with tools/make_packs.py)")
    if not os.path.exists(gp) or os.environ.get("VK_COMPACT_GOLDEN") == "1":
        cp = os.path.join(GOLDEN, f"{name}_compact.npz")
        if not os.path.exists(cp):
            pytest.skip(f"{gp} not present (generate with tools/make_packs.py)")
        gp = cp
    g = dict(np.load(gp))
    hp = os.path.join(GOLDEN, f"{name}_history.json")
    if os.path.exists(hp):
        g["info"] = json.load(open(hp))
    _PACKS[name] = (read_pack(pp), g)
    return _PACKS[name]


def golden_same(g, key, actual) -> bool:
    """Bit-equality of ``actual`` with the golden array ``key`` (float arrays
    compared as bit patterns); against its SHA-256 in a compact golden."""
    import hashlib
    if key in g:
        ref = np.asarray(g[key])
        a = np.ascontiguousarray(actual, dtype=ref.dtype)
        return a.shape == ref.shape and a.tobytes() == np.ascontiguousarray(ref).tobytes()
    a = np.ascontiguousarray(actual, dtype=np.dtype(str(g[key + "__dtype"])))
    if tuple(a.shape) != tuple(int(v) for v in g[key + "__shape"]):
        return False
    return hashlib.sha256(a.tobytes()).hexdigest() == str(g[key + "__sha256"])


def golden_rel(g, key, actual) -> float:
    """||actual - ref|| / ||ref|| against the golden N-vector ``key``.  Compact
    golden: the same ratio over the stored sample positions, or the relative
    difference of the full 2-norms / max-abs if that is larger."""
    actual = np.asarray(actual)
    if key in g:
        ref = g[key]
        return float(np.linalg.norm(actual - ref) / np.linalg.norm(ref))
    assert len(actual) == int(g[key + "__len"])
    idx, val = g[key + "__idx"], g[key + "__val"]
    rel = np.linalg.norm(actual[idx] - val) / np.linalg.norm(val)
    nrm = float(g[key + "__norm"])
    mx = float(g[key + "__maxabs"])
    return float(max(rel, abs(np.linalg.norm(actual) - nrm) / nrm,
                     abs(np.abs(actual).max() - mx) / mx))


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
