#!/usr/bin/env python
"""Host<->device copy bandwidth for the e2e leg (pinned, 4.7 MB = one cfg2 vector)."""
import json
import sys

import torch


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 592387
    reps = 50
    h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
    d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        cur = torch.cuda.current_stream()
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d[0].copy_(h[0], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h[1].copy_(d[1], non_blocking=True)

    def both():
        h2d()
        d2h()
    bytes_ = 8 * n
    for name, fn in (("h2d", h2d), ("d2h", d2h), ("h2d+d2h concurrent", both)):
        for s in (s1, s2):
            s.wait_stream(torch.cuda.current_stream())
        ms = timeit(fn)
        mult = 2 if "+" in name else 1
        out[name] = {"ms": ms, "GB/s": mult * bytes_ / (ms * 1e-3) / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
