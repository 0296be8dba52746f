#!/usr/bin/env python
"""e2e sweep pipeline probe (cfg2 finest level): host time spent issuing
SweepStream.run vs the device time of the whole run, for a few pipeline
depths — tells whether the e2e number is bound by the host, the copies or
the sweep.

    python tools/e2e_probe.py [--steps 100]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--hier", action="store_true", help="use the patches of a full 5-level hierarchy")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    from paper_2409_14222_b200.pack import read_pack
    pack = read_pack(os.path.join(ROOT, "data", "cfg2_pack.npz"))
    lv = pack.fine
    if args.hier:
        ps = V.hierarchy_from_pack(pack).fine.patches
    else:
        ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), lv.system)
    n = lv.system.matrix.shape[0]
    st = torch.cuda.current_stream()
    r_host = [torch.from_numpy(np.random.default_rng(10 + i).uniform(-1, 1, n)).pin_memory()
              for i in range(4)]
    o_host = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
    rd = r_host[0].cuda()
    xd = torch.empty_like(rd)
    # device-only sweep for reference
    for _ in range(5):
        V.apply_additive(ps, rd, xd, scale=0.5, mode=L.VK_APPLY_XSET)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        V.apply_additive(ps, rd, xd, scale=0.5, mode=L.VK_APPLY_XSET)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"device sweep: {e0.elapsed_time(e1) / args.steps * 1e3:.1f} us/step")
    # H2D / D2H alone
    for name, fn in (("h2d", lambda k: rd.copy_(r_host[k % 4], non_blocking=True)),
                     ("d2h", lambda k: o_host[k % 4].copy_(xd, non_blocking=True))):
        e0.record(st)
        for k in range(args.steps):
            fn(k)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        print(f"{name}: {ms * 1e3:.1f} us/step ({8 * n / (ms * 1e-3) / 1e9:.1f} GB/s)")
    for depth in (2, 3, 4, 6):
        sw = V.SweepStream(ps, scale=0.5, mode=L.VK_APPLY_XSET, depth=depth) \
            if "depth" in V.SweepStream.__init__.__code__.co_varnames else V.SweepStream(ps, scale=0.5, mode=L.VK_APPLY_XSET)
        ins = [r_host[k % 4] for k in range(args.steps)]
        outs = [o_host[k % 4] for k in range(args.steps)]
        sw.run(ins[:3], outs[:3])
        torch.cuda.synchronize()
        e0.record(st)
        t0 = time.perf_counter()
        sw.run(ins, outs)
        t1 = time.perf_counter()
        e1.record(st)
        torch.cuda.synchronize()
        print(f"SweepStream depth {getattr(sw, 'depth', '?')}: device {e0.elapsed_time(e1) / args.steps * 1e3:.1f} us/step, "
              f"host issue {(t1 - t0) / args.steps * 1e6:.1f} us/step")


if __name__ == "__main__":
    main()
