"""Compare device SpMV with scipy row by row on pack matrices (debug aid)."""
import sys, os
import numpy as np, scipy.sparse as sp
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14222_b200 as V
from paper_2409_14222_b200.pack import read_pack
pk = read_pack(sys.argv[1] if len(sys.argv) > 1 else "tests/golden/s_thtri2_pack.npz")
for name, M in [("A", pk.fine.system.matrix), ("P", pk.fine.prolong), ("PT", pk.fine.prolong.T.tocsr())] if pk.fine.prolong is not None else [("A", pk.fine.system.matrix)]:
    x = np.random.default_rng(0).standard_normal(M.shape[1])
    y = V.spmv(M, x); ref = M @ x
    bad = np.flatnonzero(y.view(np.uint64) != ref.view(np.uint64))
    print(name, M.shape, "nnz", M.nnz, "mismatch rows", len(bad), bad[:10], flush=True)
    if len(bad):
        i = bad[0]
        print("  row", i, "len", M.indptr[i+1]-M.indptr[i], "got", y[i], "ref", ref[i])
