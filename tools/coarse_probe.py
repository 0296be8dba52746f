#!/usr/bin/env python
"""Time the device coarse inverse (vk_coarse_operator + vk_dense_inverse)
against cuSOLVER's torch.linalg.inv (reference point only) on the coarse
operator of each BASELINE config, and report the coarse-solve difference to
the reference's LAPACK solve (golden coarse_x).

    python tools/coarse_probe.py [cfg2 cfg3 cfg4 cfg5] [--json out.json]
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def main(argv):
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.mg import coarse_inverse
    from paper_2409_14222_b200.pack import read_pack
    out = None
    if "--json" in argv:
        out = argv[argv.index("--json") + 1]
        argv = [a for a in argv if a not in ("--json", out)]
    names = argv or ["cfg2", "cfg3", "cfg4", "cfg5"]
    res = {}
    for name in names:
        d = "tests/golden" if name.startswith("s_") else "data"
        pack = read_pack(os.path.join(ROOT, d, f"{name}_pack.npz"))
        g = np.load(os.path.join(ROOT, d, f"{name}_golden.npz"))
        c = pack.levels[0]
        a0 = V.device_csr(c.system.matrix)
        q = torch.from_numpy(V.pressure_kernel(c.mixed)).cuda()
        shift = float(np.max(np.abs(c.system.matrix.data)))
        n = a0.shape[0]
        coarse_inverse(a0, q, shift)                      # warm-up (module load)
        torch.cuda.synchronize()
        t = []
        for _ in range(3):
            t0 = time.perf_counter()
            inv = coarse_inverse(a0, q, shift)
            torch.cuda.synchronize()
            t.append(time.perf_counter() - t0)
        m = a0.todense_device() + shift * torch.outer(q, q)
        torch.linalg.inv(m)
        torch.cuda.synchronize()
        tl = []
        for _ in range(3):
            t0 = time.perf_counter()
            li = torch.linalg.inv(m)
            torch.cuda.synchronize()
            tl.append(time.perf_counter() - t0)
        rc = np.random.default_rng(2).uniform(-1.0, 1.0, n)
        qq = q.cpu().numpy()
        b = rc - qq * (qq @ rc)
        x = inv.cpu().numpy() @ b
        x = x - qq * (qq @ x)
        xl = li.cpu().numpy() @ b
        xl = xl - qq * (qq @ xl)
        ref = g["coarse_x"]
        rel = float(np.linalg.norm(x - ref) / np.linalg.norm(ref))
        rel_l = float(np.linalg.norm(xl - ref) / np.linalg.norm(ref))
        flops = 2.0 * n ** 3
        import hashlib
        digest = hashlib.sha256(inv.cpu().numpy().tobytes()).hexdigest()[:16]
        res[name] = {"n": n, "device_gj_s": min(t), "device_gj_tflops": flops / min(t) / 1e12,
                     "inverse_sha256": digest, "cusolver_inv_s": min(tl), "coarse_rel_vs_reference_device": rel,
                     "coarse_rel_vs_reference_cusolver": rel_l}
        print(name, json.dumps(res[name]), flush=True)
        del inv, li, m
        torch.cuda.empty_cache()
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
