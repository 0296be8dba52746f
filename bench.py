#!/usr/bin/env python
"""Benchmark: additive Vanka sweep on the largest BASELINE config (cfg3) +
MG-FGMRES time-to-solution on every config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (the largest single-GPU BASELINE config, configs[2]):
Taylor-Hood P4/P3 on the 128x128 right-triangle grid, finest level of the
4-level hierarchy — N = 674,563 DoFs, J = 98,817 composite patches
(s = 13..123), 8*sum s^2 = 3.25 GB of patch operators streamed per sweep
(data/cfg3_pack.npz: the reference's assembled operators).  A *step* is one
additive Vanka sweep x = 0.5 * apply_additive(r) over every patch of that
level = two kernels (K4a patch solve, K4b patch-ordered accumulation).
value = patch-solves/s over all ranks.  Beside it, in the same line, every
BASELINE config (cfg2..cfg5): sweep patch-solves/s and GB/s, MG-FGMRES(30)
time-to-solution to 1e-8 (the reference's ``run_case`` solve window,
bench.py:177-187 of the reference), iterations and history parity.

Multi-GPU: replicas only — every rank runs the same sweep
workload on its own GPU, no collective on the data path; value = all ranks'
patch-solves / max-over-ranks time ("scaling": "weak").

--impl reference times the reference algorithm on the host cores: the CPU
oracle (oracle/vanka_oracle.py — the reference's factor_patches /
apply_additive restated, scipy getrf/getrs per patch, bit-exact with the
reference) over EVERY patch of the same level, split over all host cores
(rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "cfg3"
EXTRA_CONFIGS = ("cfg2", "cfg4", "cfg5")
DESCR = {
    "cfg2": "Taylor-Hood P2/P1, 256x256 right-triangle grid, finest level of the 5-level "
            "hierarchy (vertex-star patches)",
    "cfg3": "Taylor-Hood P4/P3, 128x128 right-triangle grid, finest level of the 4-level "
            "hierarchy (composite vertex/edge/cell patches)",
    "cfg4": "Taylor-Hood Q3/Q2, 128x128 quadrilateral grid, finest level of the 4-level "
            "hierarchy (composite vertex/edge/cell patches)",
    "cfg5": "BDM3/dP2 interior penalty, 128x128 right-triangle grid, finest level of the "
            "4-level hierarchy (extended cell patches)",
}


def workload(cfg):
    return (f"{cfg}: {DESCR[cfg]}; one additive Vanka sweep x = 0.5*apply_additive(r) over "
            "every patch per step, seeded uniform[-1,1] residual")


# (case, k, coarse cells per side, refinements) of each config's hierarchy
# and the reference's setup time
SETUP_SPEC = {"cfg2": ("th-tri", 2, 16, 4), "cfg3": ("th-tri", 4, 16, 3),
              "cfg4": ("th-quad", 3, 16, 3), "cfg5": ("bdm", 3, 16, 3)}
REF_SETUP_S = {"cfg2": 163.9, "cfg3": 193.3, "cfg4": 108.5, "cfg5": 154.5}

METRIC = "Vanka sweep patch-solves/s (P4/P3 128x128 finest level, damping 0.5)"
UNIT = "patch-solves/s"
CPU_SAMPLE_PER_WORKER = 2048   # ours-arm cpu_baseline: bounded sample per host core
CPU_SAMPLE_1THREAD = 2048
E2E_MIN_STEPS = 100   # e2e pipeline steps (fill/drain amortised; >= --steps)
FP64_PEAK_TFLOPS = 36.5  # measured DFMA peak on this B200 (profiles/r1_fp64_peak.json)


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _pack(cfg):
    from paper_2409_14222_b200.pack import read_pack
    return read_pack(os.path.join(ROOT, "data", f"{cfg}_pack.npz"))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}



# ----------------------------------------------------------------------------
# CPU reference arm / baseline (oracle = the reference algorithm restated)
# ----------------------------------------------------------------------------

_CPU = {}


def _cpu_worker(w, lo, hi, conn):
    """Forked worker owning patches [lo, hi): factor them once (reference
    vanka.factor_patches), then on every "apply" write
    out_w = sum_i R_i^T W_i A_i^-1 R_i r over its patches (reference
    vanka.py:145-147, scipy getrs per patch) into its shared-memory row."""
    import scipy.sparse as sp
    from multiprocessing import shared_memory
    from oracle import vanka_oracle as O
    ps, n = _CPU["ps"], _CPU["n"]
    a = sp.csr_matrix(_CPU["a"])
    facs = {}
    for j in range(lo, hi):
        ii = ps.patch(j)
        facs[j] = O.lu_factor(O.extract_submatrix(a, ii, ii))
    shm = shared_memory.SharedMemory(name=_CPU["shm"])
    buf = np.ndarray((_CPU["workers"] + 1, n), dtype=np.float64, buffer=shm.buf)
    r, out = buf[-1], buf[w]
    conn.send("ready")
    while conn.recv() == "apply":
        out[:] = 0.0
        for j in range(lo, hi):
            a_, b_ = ps.offsets[j], ps.offsets[j + 1]
            ii = ps.indices[a_:b_]
            out[ii] += ps.weights[a_:b_] * O.lu_solve(facs[j], r[ii])
        conn.send("done")
    del r, out, buf
    shm.close()


def cpu_sweep(pack, cfg, steps=3, warmup=1, sample=None, workers=None):
    """The reference algorithm (oracle port: scipy getrs per patch, weighted
    scatter in patch order) on the host cores: the (sampled) patches are split
    into contiguous slices, one forked worker process per core (each factors
    its slice once, outside the timed sweeps), partial sums in shared memory
    added by the parent.  sample=None: every patch of the level."""
    import multiprocessing as mp
    from multiprocessing import shared_memory
    from oracle import vanka_oracle as O
    lv = pack.fine
    ps = O.build_patches(lv.mixed, lv.system.bc)
    workers = workers or max(1, min(os.cpu_count() or 1, 64))
    sample = ps.num_patches if sample is None else min(ps.num_patches, sample)
    n = lv.system.matrix.shape[0]
    shm = shared_memory.SharedMemory(create=True, size=8 * (workers + 1) * n)
    buf = np.ndarray((workers + 1, n), dtype=np.float64, buffer=shm.buf)
    buf[-1] = np.random.default_rng(1).uniform(-1.0, 1.0, n)
    _CPU.update(ps=ps, a=lv.system.matrix, shm=shm.name, n=n, workers=workers)
    cuts = np.linspace(0, sample, workers + 1).astype(int)
    env_threads = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")}
    os.environ.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1")
    ctx = mp.get_context("fork")
    procs, conns = [], []
    try:
        for w in range(workers):
            parent, child = ctx.Pipe()
            p = ctx.Process(target=_cpu_worker, args=(w, int(cuts[w]), int(cuts[w + 1]), child),
                            daemon=True)
            p.start()
            procs.append(p)
            conns.append(parent)
        for c in conns:
            c.recv()                                   # factorised

        def sweep():
            for c in conns:
                c.send("apply")
            for c in conns:
                c.recv()
            return buf[:workers].sum(axis=0)

        for _ in range(warmup):
            sweep()
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            total = sweep()
            times.append(time.perf_counter() - t0)
        for c in conns:
            c.send("stop")
        for p in procs:
            p.join(timeout=30)
    finally:
        for p in procs:
            if p.is_alive():
                p.terminate()
        for k, v in env_threads.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        del buf
        shm.close()
        shm.unlink()
    t = statistics.median(times)
    what = ("every one" if sample == ps.num_patches else f"the first {sample}") + \
        f" of the {ps.num_patches} patches of the {cfg} finest level"
    return {"value": sample / t, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"{what}: the reference apply_additive loop (scipy getrs per patch, "
                      f"weighted scatter in patch order) split over {workers} forked "
                      f"single-threaded worker process(es), partial sums added; median of "
                      f"{steps} sweeps", "ms_per_step": t * 1e3, "steps": steps,
            "patches": sample, "checksum": float(np.sum(total))}


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    pack = _pack(CONFIG)
    cb = cpu_sweep(pack, CONFIG, steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic: reference-assembled operators (data/{CONFIG}_pack.npz), seeded "
                    "uniform[-1,1] residual",
            "config": {"workload": workload(CONFIG)},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

def _ev():
    import torch
    return torch.cuda.Event(enable_timing=True)


def _history_rel(cfg, hist):
    hp = os.path.join(ROOT, "tests", "golden", f"{cfg}_history.json")
    if not os.path.exists(hp):
        return None, None
    ref = np.asarray(json.load(open(hp))["history"])
    m = min(len(hist), len(ref))
    return float(np.max(np.abs(hist[:m] - ref[:m]) / ref[:m])), int(len(ref) - 1)


class Level:
    """One config's device state + the algorithmic byte counts."""

    def __init__(self, cfg, dev):
        import torch
        import paper_2409_14222_b200 as V
        from paper_2409_14222_b200 import _lib as L
        self.cfg = cfg
        self.pack = _pack(cfg)
        t0 = time.perf_counter()
        self.hier = V.hierarchy_from_pack(self.pack)
        torch.cuda.synchronize()
        self.setup_s = time.perf_counter() - t0
        fine = self.hier.fine
        self.ps = fine.patches
        ex = self.ps.export()
        self.sizes = np.diff(ex["offsets"]).astype(np.int64)
        self.J, self.N = int(self.ps.num_patches), int(fine.n)
        self.sum_s, self.sum_s2 = int(self.sizes.sum()), int((self.sizes ** 2).sum())
        # K4a: operators + idx + w + z + r once;  sweep: BASELINE.md §4
        self.bytes_solve = 8 * self.sum_s2 + 4 * self.sum_s + 8 * self.sum_s + 8 * self.sum_s \
            + 8 * self.N
        self.bytes_sweep = 8 * self.sum_s2 + 12 * self.sum_s + 16 * self.N
        self.kernel = L.lib().vk_patches_solve_kernel(self.ps.handle).decode()
        self.r = torch.from_numpy(np.random.default_rng(1).uniform(-1.0, 1.0, self.N)).to(dev)
        self.x = torch.empty_like(self.r)
        self.dev = dev

    def step(self):
        from paper_2409_14222_b200 import _lib as L
        sp = L.stream_ptr()
        h = self.ps.handle
        L.call("vk_patches_solve", h, L.ptr(self.r), None, sp)
        L.call("vk_patches_accumulate", h, None, L.ptr(self.x), 0.5, L.VK_APPLY_XSET, sp)

    def per_kernel(self, steps):
        """K4a / K4b launch durations: CUDA events on the launching stream."""
        import torch
        from paper_2409_14222_b200 import _lib as L
        stream = torch.cuda.current_stream()
        sp = L.stream_ptr()
        h = self.ps.handle
        ev = [(_ev(), _ev(), _ev()) for _ in range(steps)]
        for a, b, c in ev:
            a.record(stream)
            L.call("vk_patches_solve", h, L.ptr(self.r), None, sp)
            b.record(stream)
            L.call("vk_patches_accumulate", h, None, L.ptr(self.x), 0.5, L.VK_APPLY_XSET, sp)
            c.record(stream)
        torch.cuda.synchronize()
        return (statistics.mean(e[0].elapsed_time(e[1]) for e in ev),
                statistics.mean(e[1].elapsed_time(e[2]) for e in ev))

    def back_to_back(self, steps):
        import torch
        stream = torch.cuda.current_stream()
        for _ in range(3):
            self.step()
        a, b = _ev(), _ev()
        a.record(stream)
        for _ in range(steps):
            self.step()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    def sweep_entry(self, steps, peak):
        ms = self.back_to_back(steps)
        ms_solve, ms_acc = self.per_kernel(steps)
        ach = self.bytes_solve / (ms_solve * 1e-3) / 1e9
        return {"patches": self.J, "N": self.N, "sum_s2": self.sum_s2, "ms_per_sweep": ms,
                "patch_solves_per_s": self.J / (ms * 1e-3),
                "gbps": self.bytes_sweep / (ms * 1e-3) / 1e9,
                "frac_hbm": self.bytes_sweep / (ms * 1e-3) / 1e9 / peak,
                "k4a": {"kernel": self.kernel, "ms": ms_solve, "gbps": ach, "frac": ach / peak},
                "k4b_ms": ms_acc}

    def tts(self, reps=5):
        import torch
        from paper_2409_14222_b200.solver import FgmresSolver, mg_rhs
        stream = torch.cuda.current_stream()
        solver = FgmresSolver(self.hier)
        b = torch.from_numpy(mg_rhs(self.pack)).to(self.dev)
        solver.solve(b)                           # warm-up (graph capture)
        torch.cuda.synchronize()
        tts = []
        for _ in range(reps):
            s0, s1 = _ev(), _ev()
            s0.record(stream)
            _, its, conv, hist = solver.solve(b)
            s1.record(stream)
            torch.cuda.synchronize()
            tts.append(s0.elapsed_time(s1))
        rel, ref_its = _history_rel(self.cfg, hist)
        return {"tts_ms_median": statistics.median(tts), "tts_ms": tts, "iterations": its,
                "reference_iterations": ref_its, "converged": bool(conv),
                "history_max_rel_vs_reference": rel, "setup_s": self.setup_s}

    def residual(self, peak, reps=20):
        import torch
        from paper_2409_14222_b200 import _lib as L
        A = self.hier.fine.A
        sp = L.stream_ptr()
        y = torch.empty_like(self.r)
        for _ in range(3):
            L.call("vk_residual", A.handle, L.ptr(self.r), L.ptr(self.x), L.ptr(y), sp)
        a, b = _ev(), _ev()
        a.record(torch.cuda.current_stream())
        for _ in range(reps):
            L.call("vk_residual", A.handle, L.ptr(self.r), L.ptr(self.x), L.ptr(y), sp)
        b.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        byts = 12 * A.nnz + 4 * (self.N + 1) + 24 * self.N
        return {"ms": ms, "gbps": byts / (ms * 1e-3) / 1e9,
                "frac": byts / (ms * 1e-3) / 1e9 / peak, "nnz": int(A.nnz)}

    def transfers(self, peak):
        """Fine-level K6, each launch after a read-only 256 MB L2 flush (the
        V-cycle runs them right after a residual streamed A through L2), with
        a device copy of the same byte count as the one-shot floor."""
        import torch
        from paper_2409_14222_b200 import _lib as L
        stream = torch.cuda.current_stream()
        sp = L.stream_ptr()
        tr = self.hier.transfers[len(self.hier.levels) - 1]
        nf, nc = tr.P.shape
        dev = self.dev
        xc = torch.from_numpy(np.random.default_rng(3).uniform(-1.0, 1.0, nc)).to(dev)
        flush = torch.ones(32 << 20, dtype=torch.float64, device=dev)
        fsum = torch.empty((), dtype=torch.float64, device=dev)
        b_pro = 12 * tr.P.nnz + 4 * (nf + 1) + 8 * (nf + nc) + 8 * nf
        b_rst = 12 * tr.P.nnz + 4 * (nc + 1) + 8 * (nf + nc)
        cs = torch.ones(b_pro // 16, dtype=torch.float64, device=dev)
        cd = torch.empty_like(cs)

        def cold_ms(fn, reps=20):
            for _ in range(3):
                fn()
            pairs = []
            for _ in range(reps):
                torch.sum(flush, 0, out=fsum)
                a_, b_ = _ev(), _ev()
                a_.record(stream)
                fn()
                b_.record(stream)
                pairs.append((a_, b_))
            torch.cuda.synchronize()
            return statistics.median(a_.elapsed_time(b_) for a_, b_ in pairs)

        ms_pro = cold_ms(lambda: L.call("vk_spmv", tr.P.handle, L.ptr(xc), L.ptr(self.x), 1.0,
                                        1.0, sp))
        ms_rst = cold_ms(lambda: L.call("vk_spmv", tr.PT.handle, L.ptr(self.r), L.ptr(xc), 1.0,
                                        0.0, sp))
        ms_cpy = cold_ms(lambda: cd.copy_(cs))
        del flush, cs, cd

        # the fused V-cycle units (one cooperative launch each) against the
        # same two SpMVs as separate launches, back to back like the residual
        A = self.hier.fine.A
        rr = torch.empty_like(self.r)
        b_res = 12 * A.nnz + 4 * (nf + 1) + 24 * nf

        def warm_ms(fn, reps=20):
            for _ in range(3):
                fn()
            a_, b_ = _ev(), _ev()
            a_.record(stream)
            for _ in range(reps):
                fn()
            b_.record(stream)
            torch.cuda.synchronize()
            return a_.elapsed_time(b_) / reps

        ms_rr = warm_ms(lambda: L.call("vk_residual_restrict", A.handle, L.ptr(self.r),
                                       L.ptr(self.x), L.ptr(rr), tr.PT.handle, L.ptr(xc), sp))
        ms_rr2 = warm_ms(lambda: (L.call("vk_residual", A.handle, L.ptr(self.r), L.ptr(self.x),
                                         L.ptr(rr), sp),
                                  L.call("vk_spmv", tr.PT.handle, L.ptr(rr), L.ptr(xc), 1.0, 0.0,
                                         sp)))
        ms_pr = warm_ms(lambda: L.call("vk_prolong_residual", tr.P.handle, L.ptr(xc),
                                       L.ptr(self.x), A.handle, L.ptr(self.r), L.ptr(rr), sp))
        ms_pr2 = warm_ms(lambda: (L.call("vk_spmv", tr.P.handle, L.ptr(xc), L.ptr(self.x), 1.0,
                                         1.0, sp),
                                  L.call("vk_residual", A.handle, L.ptr(self.r), L.ptr(self.x),
                                         L.ptr(rr), sp)))
        g = lambda b, ms: b / (ms * 1e-3) / 1e9
        return {"note": "fine-level K6, one launch after an L2 flush, CUDA events; copy = device "
                        "memcpy of the prolong byte count (one-shot floor for this size)",
                "prolong_add": {"ms": ms_pro, "gbps": g(b_pro, ms_pro),
                                "frac": g(b_pro, ms_pro) / peak, "nnz": int(tr.P.nnz)},
                "restrict": {"ms": ms_rst, "gbps": g(b_rst, ms_rst),
                             "frac": g(b_rst, ms_rst) / peak},
                "copy_same_bytes": {"ms": ms_cpy, "gbps": g(b_pro, ms_cpy),
                                    "frac": g(b_pro, ms_cpy) / peak},
                "fused_residual_restrict": {
                    "ms": ms_rr, "gbps": g(b_res + b_rst, ms_rr), "frac": g(b_res + b_rst, ms_rr) / peak,
                    "unfused_ms": ms_rr2, "unfused_frac": g(b_res + b_rst, ms_rr2) / peak,
                    "note": "vk_residual_restrict: r = b - A x then rc = P^T r, one cooperative "
                            "launch (grid barrier between), back to back; bytes = residual + restrict"},
                "fused_prolong_residual": {
                    "ms": ms_pr, "gbps": g(b_res + b_pro, ms_pr), "frac": g(b_res + b_pro, ms_pr) / peak,
                    "unfused_ms": ms_pr2, "unfused_frac": g(b_res + b_pro, ms_pr2) / peak,
                    "note": "vk_prolong_residual: x += P xc then r = b - A x, one cooperative launch"}}

    def factor(self):
        """K3 re-factor of the fine level (schedule and operator storage
        cached), LU-equivalent flops (2/3) sum s^3; and the coarse inverse."""
        import torch
        import paper_2409_14222_b200 as V
        from paper_2409_14222_b200.mg import coarse_inverse
        fts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            V.factor_patches(self.ps, self.hier.fine.system)
            torch.cuda.synchronize()
            fts.append(time.perf_counter() - t0)
        ms = statistics.median(fts) * 1e3
        flops = (2.0 / 3.0) * float((self.sizes.astype(np.float64) ** 3).sum())
        c = self.hier.levels[0]
        shift = float(np.max(np.abs(c.system.matrix.data)))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        inv = coarse_inverse(c.A, self.hier.q, shift)
        torch.cuda.synchronize()
        t_c = time.perf_counter() - t0
        n0 = c.A.shape[0]
        del inv
        return {"kernel": "K2 extract_blocks_kernel + K3 factor_warp / factor_rows / factor_blk kernels (guard + Gauss-Jordan inverse), re-factorisation of every patch",
                "ms": ms, "lu_equiv_gflop": flops / 1e9,
                "tflops_lu_equiv": flops / (ms * 1e-3) / 1e12,
                "fp64_peak_tflops": FP64_PEAK_TFLOPS,
                "frac_fp64_peak": flops / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                "coarse_inverse": {"n": n0, "ms": t_c * 1e3,
                                   "tflops": 2.0 * n0 ** 3 / t_c / 1e12}}

    def device_setup(self):
        """The whole hierarchy built on the device from scratch (meshes / DoF
        maps on the host; assembly, prolongations, patches, factorisation,
        coarse inverse on the device) — SURVEY §8(f) 3-4 — timed against the
        reference's setup, and its MG-FGMRES iterations."""
        import torch
        import paper_2409_14222_b200 as V
        from paper_2409_14222_b200 import mg
        from paper_2409_14222_b200.solver import FgmresSolver, mg_rhs
        case, k, n0, refs = SETUP_SPEC[self.cfg]
        old = mg.COARSE_CELLS_PER_SIDE
        mg.COARSE_CELLS_PER_SIDE = n0
        try:
            import gc
            gc.collect()                   # earlier configs' buffers are freed outside the timing
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hier = V.build_hierarchy(case, k, refs, nu=2, damping=0.5)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        finally:
            mg.COARSE_CELLS_PER_SIDE = old
        _, its, conv, hist = FgmresSolver(hier).solve(
            torch.from_numpy(mg_rhs(self.pack)).to(self.dev))
        rel, ref_its = _history_rel(self.cfg, hist)
        del hier
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        return {"build_hierarchy_s": dt, "reference_setup_s": REF_SETUP_S.get(self.cfg),
                "iterations": its, "reference_iterations": ref_its, "converged": bool(conv),
                "history_max_rel_vs_reference": rel,
                "note": "device assembly of every level's operator + prolongations + patches "
                        "+ factorisation + coarse inverse (no pack); reference setup time "
                        "survey-measured (SURVEY.md §6)"}

    def full_entry(self, steps, peak):
        out = {"workload": workload(self.cfg), "sweep": self.sweep_entry(steps, peak)}
        out["mg_fgmres"] = self.tts()
        out["residual_spmv"] = self.residual(peak)
        out["transfers"] = self.transfers(peak)
        out["factor"] = self.factor()
        out["device_setup"] = self.device_setup()
        return out

    def close(self):
        import torch
        del self.hier, self.ps, self.r, self.x
        torch.cuda.synchronize()
        torch.cuda.empty_cache()


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    from paper_2409_14222_b200.replicas import job_throughput

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peak, peak_kind = _peak_hbm()

    lv = Level(CONFIG, dev)
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3)):
        lv.step()
    torch.cuda.synchronize()

    # ---- timed region: K sweeps back to back (no events between K4a and K4b
    # here: an event recorded between two kernels costs ~3 us of GPU time)
    start, stop = _ev(), _ev()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # VK_PROFILE_TIMED=1: bracket the timed region with cudaProfilerStart/Stop
    # (ncu --profile-from-start off captures exactly its launches)
    prof_region = os.environ.get("VK_PROFILE_TIMED") == "1"
    with ClockSampler(local) as clocks:
        if prof_region:
            torch.cuda.profiler.start()
        start.record(stream)
        for _ in range(args.steps):
            lv.step()
        stop.record(stream)
        torch.cuda.synchronize()
        if prof_region:
            torch.cuda.profiler.stop()
        # ---- per-kernel pass for the roofline
        ms_solve, ms_gather = lv.per_kernel(args.steps)
        # ---- e2e through the public API, pipelined (SweepStream): every step
        # copies its residual from pinned host memory and its result back,
        # the copies of neighbouring steps overlapped with the sweep
        N, J = lv.N, lv.J
        nbuf = 4
        r_host = [torch.from_numpy(np.random.default_rng(10 + i).uniform(-1.0, 1.0, N))
                  .pin_memory() for i in range(nbuf)]
        o_host = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
        sweeps = V.SweepStream(lv.ps, scale=0.5, mode=L.VK_APPLY_XSET)
        e2e_steps = max(args.steps, E2E_MIN_STEPS)
        ins = [r_host[k % nbuf] for k in range(e2e_steps)]
        outs = [o_host[k % nbuf] for k in range(e2e_steps)]
        sweeps.run(ins[:3], outs[:3])
        torch.cuda.synchronize()
        e0, e1 = _ev(), _ev()
        e0.record(stream)
        sweeps.run(ins, outs)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1) / e2e_steps
        chk = torch.empty(N, dtype=torch.float64, device=dev)
        V.apply_additive(lv.ps, ins[-1].to(dev), chk, scale=0.5, mode=L.VK_APPLY_XSET)
        assert torch.equal(chk.cpu(), outs[-1]), "pipelined e2e sweep differs from the device sweep"
        e2e_value, _ = job_throughput(J, ms_e2e, dev)
        # ---- e2e through the drop-in call itself, as a reference caller uses
        # it (vanka.py:142): numpy residual in, numpy result out, one call per step
        r_np = [np.random.default_rng(20 + i).uniform(-1.0, 1.0, N) for i in range(nbuf)]
        for i in range(3):
            V.apply_additive(lv.ps, r_np[i % nbuf], scale=0.5, mode=L.VK_APPLY_XSET)
        d_steps = max(args.steps, 20)
        torch.cuda.synchronize()
        d0, d1 = _ev(), _ev()
        d0.record(stream)
        for k in range(d_steps):
            out_np = V.apply_additive(lv.ps, r_np[k % nbuf], scale=0.5, mode=L.VK_APPLY_XSET)
        d1.record(stream)
        torch.cuda.synchronize()
        ms_drop = d0.elapsed_time(d1) / d_steps
        V.apply_additive(lv.ps, torch.from_numpy(r_np[(d_steps - 1) % nbuf]).to(dev), chk,
                         scale=0.5, mode=L.VK_APPLY_XSET)
        assert np.array_equal(chk.cpu().numpy(), out_np), "drop-in sweep differs"
        drop_value, _ = job_throughput(J, ms_drop, dev)
        # keep the GPU busy a little longer so the sampler sees load
        extra_t0 = time.perf_counter()
        while time.perf_counter() - extra_t0 < 1.0:
            for _ in range(10):
                lv.step()
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = start.elapsed_time(stop)
    value, ms_total = job_throughput(J * args.steps, ms_total, dev)
    ms_step = ms_total / args.steps

    per_config = {}
    if not args.headline_only:
        per_config[CONFIG] = lv.full_entry(args.steps, peak)
    lv_summary = {"N": lv.N, "patches": lv.J, "sum_s": lv.sum_s, "sum_s2": lv.sum_s2,
                  "kernel": lv.kernel, "bytes_solve": lv.bytes_solve,
                  "bytes_sweep": lv.bytes_sweep}
    lv.close()
    if not args.headline_only:
        for cfg in EXTRA_CONFIGS:
            other = Level(cfg, dev)
            per_config[cfg] = other.full_entry(args.steps, peak)
            other.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    achieved = lv_summary["bytes_solve"] / (ms_solve * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{CONFIG}:{lv_summary['kernel']}", {}) \
                .get("dram_bytes")
        except Exception:
            traffic = None
    cpu = cpu1 = None
    if world == 1 and not args.no_cpu:
        pack = _pack(CONFIG)
        workers = max(1, min(os.cpu_count() or 1, 64))
        cb = cpu_sweep(pack, CONFIG, steps=3, warmup=1, sample=CPU_SAMPLE_PER_WORKER * workers,
                       workers=workers)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        c1 = cpu_sweep(pack, CONFIG, steps=3, warmup=1, sample=CPU_SAMPLE_1THREAD, workers=1)
        cpu1 = {k: c1[k] for k in ("value", "unit", "cores", "kind", "sample")}
        cpu1["threads"] = "OMP_NUM_THREADS=OPENBLAS_NUM_THREADS=1 (BASELINE.md §5)"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: reference-assembled operators (data/{CONFIG}_pack.npz), seeded "
                "uniform[-1,1] residual",
        "config": {"workload": workload(CONFIG),
                   "N": lv_summary["N"], "patches": lv_summary["patches"],
                   "sum_s": lv_summary["sum_s"], "sum_s2": lv_summary["sum_s2"],
                   "l2": "inputs larger than L2 (8*sum s^2 = %.0f MB streamed per sweep)"
                         % (8 * lv_summary["sum_s2"] / 1e6),
                   "parallelism": f"replicas x{world}"},
        "roofline": {"bound": "hbm", "kernel": f"{lv_summary['kernel']} (K4a, TMA bulk copies)",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes": lv_summary["bytes_solve"], "ms": ms_solve,
                     "traffic_source": f"profiles/ncu_summary.json[{CONFIG}:"
                                       f"{lv_summary['kernel']}] (ncu --set full, dram bytes "
                                       "read+write of one launch)",
                     "timing": "K4a launch duration from per-kernel CUDA events on the launching "
                               "stream, in a pass of --steps sweeps right after the timed region"},
        "sweep": {"ms": ms_solve + ms_gather, "ms_solve": ms_solve, "ms_accumulate": ms_gather,
                  "gbps": lv_summary["bytes_sweep"] / ((ms_solve + ms_gather) * 1e-3) / 1e9,
                  "algorithmic_bytes": lv_summary["bytes_sweep"]},
        "per_config": per_config,
        "cpu_baseline": cpu,
        "cpu_baseline_1thread": cpu1,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                "d2h_bytes_per_step": 8 * N, "ms_per_step": ms_e2e, "steps": e2e_steps,
                "api": "SweepStream (pinned host buffers, copies overlapped on three streams)"},
        "e2e_dropin": {"value": drop_value, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                       "d2h_bytes_per_step": 8 * N, "ms_per_step": ms_drop, "steps": d_steps,
                       "api": "apply_additive(patchset, numpy residual) -> numpy, one "
                              "synchronous call per step (reference vanka.py:142 call shape)"},
        "gpu_launches": 2 * args.steps,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline samples")
    ap.add_argument("--headline-only", action="store_true",
                    help="only the headline sweep (no per-config TTS / SpMV / factor section)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
