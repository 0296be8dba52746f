#!/usr/bin/env python
"""Per-kernel timings of the hot path on the finest level of each config
(CUDA events on the launching stream, after warm-up).  GPU only.

    python tools/bench_kernels.py [cfg2 cfg3 cfg4 cfg5] [--reps 20] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def timed(fn, reps, stream):
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--json")
    ap.add_argument("--tts", action="store_true", help="also V-cycle time and MG-FGMRES TTS")
    args = ap.parse_args()
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import vanka as VV
    from paper_2409_14222_b200 import _lib as L
    from paper_2409_14222_b200.pack import read_pack
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    out = {}
    for name in args.names:
        d = "data" if name.startswith("cfg") and name != "cfg1" else "tests/golden"
        pack = read_pack(os.path.join(ROOT, d, f"{name}_pack.npz"))
        lv = pack.fine
        t0 = time.perf_counter()
        ps = V.build_patches(lv.mixed, lv.system.bc)
        torch.cuda.synchronize()
        t_build = time.perf_counter() - t0
        t0 = time.perf_counter()
        V.factor_patches(ps, lv.system)
        torch.cuda.synchronize()
        t_factor_first = time.perf_counter() - t0
        t0 = time.perf_counter()           # re-factor: operator storage already allocated
        V.factor_patches(ps, lv.system)
        torch.cuda.synchronize()
        t_factor = time.perf_counter() - t0
        ex = ps.export()
        sz = np.diff(ex["offsets"]).astype(np.int64)
        N, J = lv.system.matrix.shape[0], ps.num_patches
        s1, s2, s3 = int(sz.sum()), int((sz ** 2).sum()), int((sz ** 3).sum())
        A = V.device_csr(lv.system.matrix)
        st = torch.cuda.current_stream()
        sp_ = L.stream_ptr()
        r = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, N)).cuda()
        x = torch.zeros_like(r)
        y = torch.zeros_like(r)
        h = ps.handle
        t_solve = timed(lambda: L.call("vk_patches_solve", h, L.ptr(r), None, sp_), args.reps, st)
        t_acc = timed(lambda: L.call("vk_patches_accumulate", h, None, L.ptr(x), 0.5, L.VK_APPLY_XADD, sp_),
                      args.reps, st)
        t_res = timed(lambda: L.call("vk_residual", A.handle, L.ptr(r), L.ptr(x), L.ptr(y), sp_),
                      args.reps, st)
        # library reference point (not product code): cuSPARSE SpMV via torch
        m = lv.system.matrix
        tcsr = torch.sparse_csr_tensor(torch.from_numpy(m.indptr.astype(np.int32)).cuda(),
                                       torch.from_numpy(m.indices.astype(np.int32)).cuda(),
                                       torch.from_numpy(m.data).cuda(), size=m.shape)
        t_cusp = timed(lambda: torch.mv(tcsr, x), args.reps, st)
        del tcsr
        # library reference point for K3 (not product code): batched explicit
        # inverse of the dominant patch-size class via torch.linalg.inv
        # (cuSOLVER/cuBLAS batched getrf + getri), no pivot guard
        smode = int(np.bincount(sz).argmax())
        ids = np.flatnonzero(sz == smode)[:8192]
        blocks = VV.extract_blocks(ps, lv.system.matrix, int(ids[0]), int(ids[-1] - ids[0] + 1))
        batch = torch.from_numpy(np.stack([blocks[i - ids[0]] for i in ids])).cuda()
        t_inv = timed(lambda: torch.linalg.inv(batch), 3, st)
        del batch, blocks
        rec = {"N": N, "J": J, "nnz": int(A.nnz), "sum_s": s1, "sum_s2": s2, "smax": int(sz.max()),
               "cusparse_spmv_ms": t_cusp,
               "library_batched_inv": {"s": smode, "count": int(len(ids)), "ms": t_inv,
                                       "ms_per_1k": t_inv / len(ids) * 1000.0},
               "build_s": t_build, "factor_s": t_factor, "factor_first_s": t_factor_first,
               "factor_gflops_lu_equiv": (2.0 / 3.0) * s3 / t_factor / 1e9,
               "solve_ms": t_solve, "accumulate_ms": t_acc, "residual_ms": t_res}
        b_solve = 8 * s2 + 20 * s1 + 8 * N
        b_sweep = 8 * s2 + 12 * s1 + 16 * N
        b_res = 12 * A.nnz + 4 * (N + 1) + 24 * N
        rec["solve_gbps"] = b_solve / (t_solve * 1e-3) / 1e9
        rec["sweep_gbps"] = b_sweep / ((t_solve + t_acc) * 1e-3) / 1e9
        rec["residual_gbps"] = b_res / (t_res * 1e-3) / 1e9
        rec["solve_frac"] = rec["solve_gbps"] / peak
        rec["sweep_frac"] = rec["sweep_gbps"] / peak
        rec["residual_frac"] = rec["residual_gbps"] / peak
        rec["patch_solves_per_s"] = J / ((t_solve + t_acc) * 1e-3)
        if lv.prolong is not None:
            P = V.device_csr(lv.prolong)
            PT = P.T
            xc = torch.zeros(P.shape[1], dtype=torch.float64, device="cuda")
            t_pro = timed(lambda: L.call("vk_spmv", P.handle, L.ptr(xc), L.ptr(x), 1.0, 1.0, sp_),
                          args.reps, st)
            t_rst = timed(lambda: L.call("vk_spmv", PT.handle, L.ptr(r), L.ptr(xc), 1.0, 0.0, sp_),
                          args.reps, st)
            b_p = 12 * P.nnz + 4 * (P.shape[0] + 1) + 8 * (P.shape[0] + P.shape[1]) + 8 * P.shape[0]
            b_t = 12 * P.nnz + 4 * (P.shape[1] + 1) + 8 * (P.shape[0] + P.shape[1])
            rec.update({"prolong_ms": t_pro, "restrict_ms": t_rst,
                        "prolong_gbps": b_p / (t_pro * 1e-3) / 1e9,
                        "restrict_gbps": b_t / (t_rst * 1e-3) / 1e9, "nnz_P": int(P.nnz)})
        if args.tts and name != "cfg1":
            from paper_2409_14222_b200.solver import FgmresSolver, mg_rhs
            del ps
            t0 = time.perf_counter()
            hier = V.hierarchy_from_pack(pack)
            torch.cuda.synchronize()
            rec["mg_setup_s"] = time.perf_counter() - t0
            b = torch.from_numpy(mg_rhs(pack)).cuda()
            rec["vcycle_ms"] = timed(lambda: hier.vcycle_device(b), args.reps, st)
            solver = FgmresSolver(hier)
            solver.solve(b)
            tts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                _, its, conv, hist = solver.solve(b)
                e1.record(st)
                torch.cuda.synchronize()
                tts.append(e0.elapsed_time(e1))
            rec["tts_ms"] = statistics.median(tts)
            rec["tts_iterations"] = its
            ref = json.load(open(os.path.join(ROOT, "tests", "golden", f"{name}_history.json")))
            rec["tts_reference_iterations"] = ref["iterations"]
            rec["tts_reference_cpu_s"] = ref["solve_s"]
            h_ref = np.asarray(ref["history"])
            m = min(len(hist), len(h_ref))
            rec["history_max_rel"] = float(np.max(np.abs(hist[:m] - h_ref[:m]) / h_ref[:m]))
            del hier, solver
            torch.cuda.empty_cache()
        out[name] = rec
        print(name, json.dumps({k: (round(v, 4) if isinstance(v, float) else v)
                                for k, v in rec.items()}), flush=True)
        if "ps" in locals():
            del ps
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
