#!/usr/bin/env python
"""Sweep (vk_patches_apply) time back to back on a config's finest level, and
bit-identity of its result against solve + accumulate — run with VK_SWEEP_SPLIT=0/90 etc..

    VK_SWEEP_SPLIT=90 python tools/sweep_probe.py [cfg2] [--steps 50]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    from paper_2409_14222_b200.pack import read_pack
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["cfg2"]
    steps = 50
    for name in names:
        pack = read_pack(os.path.join(ROOT, "data", f"{name}_pack.npz"))
        lv = pack.fine
        ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), lv.system)
        n = lv.system.matrix.shape[0]
        r = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
        x = torch.empty_like(r)
        sp_ = L.stream_ptr()
        st = torch.cuda.current_stream()
        h = ps.handle
        for mode in (L.VK_APPLY_XSET, L.VK_APPLY_XADD, L.VK_APPLY_OUT):
            ref = torch.full_like(r, 0.25)
            L.call("vk_patches_solve", h, L.ptr(r), sp_)
            L.call("vk_patches_accumulate", h, L.ptr(ref), 0.5, mode, sp_)
            got = torch.full_like(r, 0.25)
            L.call("vk_patches_apply", h, L.ptr(r), L.ptr(got), 0.5, mode, sp_)
            torch.cuda.synchronize()
            same = torch.equal(ref, got)
            print(f"{name} mode {mode}: apply == solve+accumulate: {same}", flush=True)
            assert same or os.environ.get("VK_PROBE_NOCHECK")
        for _ in range(5):
            L.call("vk_patches_apply", h, L.ptr(r), L.ptr(x), 0.5, L.VK_APPLY_XSET, sp_)
        torch.cuda.synchronize()
        reps = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(steps):
                L.call("vk_patches_apply", h, L.ptr(r), L.ptr(x), 0.5, L.VK_APPLY_XSET, sp_)
            b.record(st)
            torch.cuda.synchronize()
            reps.append(a.elapsed_time(b) / steps)
        ms = statistics.median(reps)
        print(f"{name} VK_SWEEP_SPLIT={os.environ.get("VK_SWEEP_SPLIT", "0")}: sweep {ms * 1e3:.1f} us, "
              f"{ps.num_patches / (ms * 1e-3):.3e} patch-solves/s", flush=True)


if __name__ == "__main__":
    main()
