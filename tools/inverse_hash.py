#!/usr/bin/env python
"""SHA-256 of the exported patch inverses (every 53rd patch) of each config's
finest level — to check that two K3 builds produce bit-identical operators.

    python tools/inverse_hash.py [cfg2 ...]
"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.pack import read_pack
    from paper_2409_14222_b200.vanka import patch_inverses
    for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]:
        d = "data" if name in ("cfg2", "cfg3", "cfg4", "cfg5") else os.path.join("tests", "golden")
        pack = read_pack(os.path.join(ROOT, d, f"{name}_pack.npz"))
        lv = pack.fine
        ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), lv.system)
        h = hashlib.sha256()
        for p in range(0, ps.num_patches, 53):
            h.update(np.ascontiguousarray(patch_inverses(ps, p, 1)[0]).tobytes())
        print(name, h.hexdigest()[:16], flush=True)


if __name__ == "__main__":
    main()
