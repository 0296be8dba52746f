"""README quick start, runnable: MG-FGMRES on cfg2 and the reference-style
patch API on its finest level (needs a B200 and data/cfg2_pack.npz)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.chdir(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2409_14222_b200 as V
from paper_2409_14222_b200.pack import read_pack
from paper_2409_14222_b200.solver import FgmresSolver, mg_rhs
pack = read_pack("data/cfg2_pack.npz")
hier = V.hierarchy_from_pack(pack)
x, its, converged, history = FgmresSolver(hier).solve(mg_rhs(pack))
print("its", its, "converged", converged, "final rel", history[-1], type(x))
# reference-style API on the fine level
lv = pack.fine
import numpy as np
ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), lv.system)
r = np.random.default_rng(0).uniform(-1, 1, lv.system.matrix.shape[0])
out = V.apply_additive(ps, r)
print("apply_additive ->", type(out), out.shape, float(np.linalg.norm(out)))
print("spmv ->", float(np.linalg.norm(V.spmv(lv.system.matrix, r))))
