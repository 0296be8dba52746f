#!/usr/bin/env python
"""Captured V-cycle time (median of 30 replays) per config:
python tools/vcycle_time.py [cfg2 ...]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.pack import read_pack
    from paper_2409_14222_b200.solver import mg_rhs
    for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]:
        pack = read_pack(os.path.join(ROOT, "data", f"{name}_pack.npz"))
        hier = V.hierarchy_from_pack(pack)
        b = torch.from_numpy(mg_rhs(pack)).cuda()
        for _ in range(5):
            hier.vcycle_device(b)
        torch.cuda.synchronize()
        ts = []
        for _ in range(30):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hier.vcycle_device(b)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        x = hier.vcycle_device(b).cpu().numpy()
        import hashlib
        print(f"{name} VK_SPLIT_MAX={os.environ.get('VK_SPLIT_MAX', 'default')} V-cycle "
              f"{statistics.median(ts) * 1e3:.1f} us (min {min(ts) * 1e3:.1f}) "
              f"sha {hashlib.sha256(x.tobytes()).hexdigest()[:12]}")
        del hier


if __name__ == "__main__":
    main()
