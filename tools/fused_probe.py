#!/usr/bin/env python
"""V-cycle (captured graph) time with the fused transfer units on and off
(mg.FUSED_TRANSFERS), per BASELINE config.  python tools/fused_probe.py [cfgs]"""
import os
import statistics
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def main(names):
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import mg
    from paper_2409_14222_b200.pack import read_pack
    for name in names:
        pack = read_pack(os.path.join(ROOT, "data", f"{name}_pack.npz"))
        res = {}
        for mode in ("repeat", "degree"):
            for fused in (True, False):
                mg.FUSED_TRANSFERS = fused
                hier = V.hierarchy_from_pack(pack, cheb_mode=mode)
                v = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, hier.fine.n)).cuda()
                for _ in range(5):
                    hier.vcycle_device(v)
                torch.cuda.synchronize()
                ts = []
                for _ in range(30):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    hier.vcycle_device(v)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                res[(mode, fused)] = statistics.median(ts)
                del hier
                torch.cuda.empty_cache()
        mg.FUSED_TRANSFERS = False
        print(name, " ".join(f"{m}/{'fused' if f else 'unfused'}={t:.4f}ms"
                             for (m, f), t in res.items()), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"])
