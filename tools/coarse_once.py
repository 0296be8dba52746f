#!/usr/bin/env python
"""One coarse inverse of a config's coarse operator (for ncu launch lists)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2409_14222_b200 as V
from paper_2409_14222_b200.mg import coarse_inverse
from paper_2409_14222_b200.pack import read_pack
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
c = read_pack(os.path.join(ROOT, "data", f"{name}_pack.npz")).levels[0]
a0 = V.device_csr(c.system.matrix)
q = torch.from_numpy(V.pressure_kernel(c.mixed)).cuda()
shift = float(np.max(np.abs(c.system.matrix.data)))
coarse_inverse(a0, q, shift)
torch.cuda.synchronize()
torch.cuda.profiler.start()
coarse_inverse(a0, q, shift)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
