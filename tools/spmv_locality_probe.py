#!/usr/bin/env python
"""Upper bound for x-gather locality in the residual SpMV: the same row lengths
and values with every row's columns moved next to the diagonal (synthetic),
timed against the real matrix (CUDA events, back to back)."""
import os, sys, statistics, numpy as np, torch, scipy.sparse as sp
sys.path.insert(0, '/root/repo')
import paper_2409_14222_b200 as V
from paper_2409_14222_b200 import _lib as L
from paper_2409_14222_b200.pack import read_pack
st = torch.cuda.current_stream(); spp = L.stream_ptr()
for name in sys.argv[1:]:
    A = read_pack(f'/root/repo/data/{name}_pack.npz').fine.system.matrix.tocsr()
    n = A.shape[0]
    lens = np.diff(A.indptr)
    # synthetic local pattern: row i's k-th entry -> column (i - len/2 + k) clipped, sorted, same lengths
    rows = np.repeat(np.arange(n), lens)
    k = np.arange(A.nnz) - np.repeat(A.indptr[:-1], lens)
    cols = np.clip(rows - lens[rows] // 2 + k, 0, n - 1)
    cols = np.minimum(cols, n - 1)
    B = sp.csr_matrix((A.data, cols.astype(np.int32), A.indptr), shape=A.shape)
    x = torch.from_numpy(np.random.default_rng(0).uniform(-1,1,n)).cuda(); y = torch.empty_like(x)
    for lab, M in (("orig", A), ("local", B)):
        D = V.device_csr(M)
        for _ in range(3): L.call("vk_residual", D.handle, L.ptr(x), L.ptr(x), L.ptr(y), spp)
        ev = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); L.call("vk_residual", D.handle, L.ptr(x), L.ptr(x), L.ptr(y), spp); b.record(st); ev.append((a, b))
        torch.cuda.synchronize()
        t = statistics.median(a.elapsed_time(b) for a, b in ev)
        by = 12 * M.nnz + 4 * (n + 1) + 24 * n
        print(name, lab, f"{t*1e3:.1f} us  {by/(t*1e-3)/1e9:.0f} GB/s  frac {by/(t*1e-3)/1e9/6550:.3f}", flush=True)
        del D
