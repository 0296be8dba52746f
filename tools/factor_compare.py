#!/usr/bin/env python
"""Compare the patch inverses of two K3 kernel families on the finest level
of each config: eight ranges of 400 patches are exported from a run with the default
kernels and from a run with VK_FACTOR_ROWS=0 (round-2 register-tile / DMMA
kernels), per size class: fraction bit-identical, max |difference| relative
to max |inverse entry| of the patch.

    python tools/factor_compare.py [cfg2 ...]
"""
import os
import subprocess
import time
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
STEP = 11


def dump(name, out):
    import numpy as np
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.pack import read_pack
    from paper_2409_14222_b200.vanka import patch_inverses
    d = "data" if name in ("cfg2", "cfg3", "cfg4", "cfg5") else os.path.join("tests", "golden")
    lv = read_pack(os.path.join(ROOT, d, f"{name}_pack.npz")).fine
    ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), lv.system)
    J = ps.num_patches
    blocks = []
    for q in range(8):                      # eight ranges of 400 patches
        f = q * J // 8
        blocks += [np.ascontiguousarray(b).ravel() for b in patch_inverses(ps, f, min(400, J - f))]
    sizes = np.array([int(np.sqrt(b.size)) for b in blocks])
    np.savez(out, flat=np.concatenate(blocks), sizes=sizes)


def main():
    import numpy as np
    if len(sys.argv) > 2 and sys.argv[1] == "--dump":
        dump(sys.argv[2], sys.argv[3])
        return
    for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]:
        files = {}
        for tag, env in (("new", {}), ("old", {"VK_FACTOR_ROWS": "0", "VK_FACTOR_BLK": "0"})):
            f = f"/tmp/fc_{name}_{tag}.npz"
            t0 = time.time()
            subprocess.run([sys.executable, __file__, "--dump", name, f],
                           env=dict(os.environ, **env), check=True)
            print(f"{name} {tag}: dumped in {time.time() - t0:.1f} s", flush=True)
            files[tag] = np.load(f)
        a, b = files["new"], files["old"]
        assert np.array_equal(a["sizes"], b["sizes"])
        off = 0
        per = {}
        for s in a["sizes"]:
            x, y = a["flat"][off:off + s * s], b["flat"][off:off + s * s]
            off += s * s
            st = per.setdefault(int(s), [0, 0, 0.0])
            st[0] += 1
            st[1] += int(np.array_equal(x.view(np.uint64), y.view(np.uint64)))
            st[2] = max(st[2], float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300)))
        for s in sorted(per):
            n, same, rel = per[s]
            print(f"{name} s={s}: {n} patches, bit-identical {same}/{n}, max rel diff {rel:.2e}",
                  flush=True)


if __name__ == "__main__":
    main()
