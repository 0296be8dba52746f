#!/usr/bin/env python
"""Residual SpMV of one config's finest operator in a loop (for ncu captures
and VK_SPMV_MODE A/B timings).

    VK_SPMV_MODE=1 python tools/spmv_probe.py cfg3 [reps]
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
    from paper_2409_14222_b200.pack import read_pack
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    a = read_pack(os.path.join(ROOT, "data", f"{name}_pack.npz")).fine.system.matrix
    d = V.device_csr(a)
    n = a.shape[0]
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal(n)).cuda()
    b = torch.from_numpy(rng.standard_normal(n)).cuda()
    r = torch.empty_like(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.residual(b, x, r)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ref = b.cpu().numpy() - a @ x.cpu().numpy()
    same = np.array_equal(ref.view(np.uint64), r.cpu().numpy().view(np.uint64))
    nbytes = 12 * a.nnz + 4 * (n + 1) + 24 * n
    ms = statistics.median(ts)
    print(f"{name} mode={os.environ.get('VK_SPMV_MODE', 'default')} residual {ms * 1e3:.1f} us "
          f"{nbytes / ms / 1e6:.0f} GB/s bit-identical-to-scipy={same}")


if __name__ == "__main__":
    main()
