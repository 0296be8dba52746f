#!/usr/bin/env python
"""K6 probe: time prolong-add (x += P xc) and restriction (rc = P^T r) on the
finest transfer of each BASELINE config, with an L2 flush before every launch
(what the V-cycle sees: the residual SpMV streams A through L2 right before)
and back to back (L2-warm).  Also usable under ncu (-k regex:csr).

    python tools/transfer_probe.py [cfg2 cfg3 ...] [--reps 50] [--json out]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--json")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    from paper_2409_14222_b200.pack import read_pack

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6557.4) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6557.4
    st = torch.cuda.current_stream()
    sp_ = L.stream_ptr()
    # read-only flush: a memset would leave ~126 MB of dirty L2 lines whose
    # write-back lands inside the next timed kernel
    flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
    fsum = torch.empty((), dtype=torch.float64, device="cuda")
    out = {}
    for name in args.names:
        pack = read_pack(os.path.join(ROOT, "data", f"{name}_pack.npz"))
        pm = pack.fine.prolong
        P = V.device_csr(pm)
        PT = P.T
        nf, nc = pm.shape
        rng = np.random.default_rng(3)
        xc = torch.from_numpy(rng.uniform(-1, 1, nc)).cuda()
        xf = torch.from_numpy(rng.uniform(-1, 1, nf)).cuda()
        rc = torch.zeros(nc, dtype=torch.float64, device="cuda")

        A = V.device_csr(pack.fine.system.matrix)
        rr = torch.empty_like(xf)

        def res():
            L.call("vk_residual", A.handle, L.ptr(xf), L.ptr(xf), L.ptr(rr), sp_)

        def pro():
            L.call("vk_spmv", P.handle, L.ptr(xc), L.ptr(xf), 1.0, 1.0, sp_)

        def rst():
            L.call("vk_spmv", PT.handle, L.ptr(xf), L.ptr(rc), 1.0, 0.0, sp_)

        def timed(fn, cold):
            # all launches queued (no host gaps inside an event pair); with
            # cold=True a 256 MB read runs between launches (L2 flushed, clean)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ev = []
            for _ in range(args.reps):
                if cold:
                    torch.sum(flush, 0, out=fsum)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                fn()
                b.record(st)
                ev.append((a, b))
            torch.cuda.synchronize()
            return statistics.median(a.elapsed_time(b) for a, b in ev)

        nnz = int(P.nnz)
        b_p = 12 * nnz + 4 * (nf + 1) + 8 * (nf + nc) + 8 * nf
        b_t = 12 * nnz + 4 * (nc + 1) + 8 * (nf + nc)
        b_r = 12 * int(A.nnz) + 4 * (nf + 1) + 24 * nf
        rec = {"nnz": nnz, "rows": nf, "cols": nc, "bytes_prolong": b_p, "bytes_restrict": b_t,
               "nnz_A": int(A.nnz), "bytes_residual": b_r}
        # floor for a one-shot stream of the same size: torch device copy
        cs = torch.ones(b_p // 16, dtype=torch.float64, device="cuda")
        cd = torch.empty_like(cs)

        def cpy():
            cd.copy_(cs)

        for lab, fn, by in (("prolong", pro, b_p), ("restrict", rst, b_t), ("residual", res, b_r),
                            ("copy", cpy, 16 * (b_p // 16))):
            for cold in (True, False):
                t = timed(fn, cold)
                k = f"{lab}_{'cold' if cold else 'warm'}"
                rec[k + "_us"] = t * 1e3
                rec[k + "_frac"] = by / (t * 1e-3) / 1e9 / peak
        out[name] = rec
        print(name, json.dumps({k: (round(v, 3) if isinstance(v, float) else v)
                                for k, v in rec.items()}), flush=True)
        del P, PT, A
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
