#!/usr/bin/env python
"""Separate the two error sources of the device coarse solve: the explicit
inverse itself (device LU inverse vs cuSOLVER vs LAPACK) and its application
(device vk_gemv vs numpy matvec), against the reference's LAPACK solve
(golden coarse_x).  Test-side probe; imports the oracle as the checker."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def main(names):
    import scipy.linalg as sl
    import torch
    from threadpoolctl import threadpool_limits
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    from paper_2409_14222_b200.mg import coarse_inverse
    from paper_2409_14222_b200.pack import read_pack
    for name in names:
        d = "tests/golden" if name.startswith("s_") else "data"
        pack = read_pack(os.path.join(ROOT, d, f"{name}_pack.npz"))
        g = np.load(os.path.join(ROOT, d, f"{name}_golden.npz"))
        c = pack.levels[0]
        q = V.pressure_kernel(c.mixed)
        a0 = c.system.matrix
        shift = float(np.max(np.abs(a0.data)))
        m = a0.toarray() + shift * np.outer(q, q)
        n = m.shape[0]
        rc = np.random.default_rng(2).uniform(-1.0, 1.0, n)
        b = rc - q * (q @ rc)
        ref = g["coarse_x"]
        rel = lambda x: float(np.linalg.norm(x - ref) / np.linalg.norm(ref))
        fin = lambda x: x - q * (q @ x)
        qd = torch.from_numpy(q).cuda()
        inv_dev = coarse_inverse(V.device_csr(a0), qd, shift)
        inv_cus = torch.linalg.inv(torch.from_numpy(m).cuda())
        with threadpool_limits(8):
            lu, piv = sl.lu_factor(m)
            inv_cpu = sl.lu_solve((lu, piv), np.eye(n))
        bd = torch.from_numpy(b).cuda()
        out = {}
        for tag, inv in (("device", inv_dev), ("cusolver", inv_cus)):
            y = torch.empty_like(bd)
            L.call("vk_gemv", n, n, L.ptr(inv), L.ptr(bd), L.ptr(y), L.stream_ptr())
            ih = inv.cpu().numpy()
            out[tag] = {"gemv_dev": rel(fin(y.cpu().numpy())), "matvec_np": rel(fin(ih @ b)),
                        "inv_vs_lapack": float(np.linalg.norm(ih - inv_cpu) /
                                               np.linalg.norm(inv_cpu))}
        y = torch.empty_like(bd)
        icd = torch.from_numpy(inv_cpu).cuda()
        L.call("vk_gemv", n, n, L.ptr(icd), L.ptr(bd), L.ptr(y), L.stream_ptr())
        out["lapack_inv"] = {"gemv_dev": rel(fin(y.cpu().numpy())), "matvec_np": rel(fin(inv_cpu @ b))}
        print(name, out, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["s_bdm3", "cfg5"])
