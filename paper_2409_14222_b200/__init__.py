"""B200-native (sm_100a) Vanka patch relaxation + multigrid hot path.

Drop-in for the hot path of the reference package ``stokesmg``
(arXiv 2409.14222 companion code): the names below mirror
``stokesmg/__init__.py:15-35`` for ``sparsela``, ``vanka``, ``mg``, the
assembly entry points and the ``bench`` driver layer (``experiments.py``).  All
numerics run in ``libvanka_b200.so`` (hand-written CUDA behind a C ABI,
``include/vanka_b200.h``); importing works without a GPU, computing does not
(no CPU fallback).
"""

from .pack import ProblemPack, read_pack
from .sparsela import (DenseFactorization, DeviceCSR, FgmresWorkspace, KrylovReport,
                       NullspaceProjector,
                       SingularMatrixError, device_csr, estimate_lambda_max,
                       extract_submatrix, fgmres, lu_factor, lu_solve, nullspace_projector,
                       spmv, triple_product)
from .vanka import (EntityRef, Patch, PatchSet, SweepStream, apply_additive, build_patches,
                    build_patches_hdiv_extended, build_patches_taylor_hood, factor_patches)
from .mg import (ChebyshevParams, FixedDamping, Level, MgHierarchy, TransferPair,
                 chebyshev_iteration, chebyshev_relax, coarse_solve, hierarchy_from_pack,
                 hierarchy_from_reference, make_preconditioner, pressure_kernel, v_cycle)
from .assembly import (ProblemConfig, assemble, build_hierarchy, build_prolongation,
                       interpolate)
from .fem import build_mixed, strong_bc, structured_mesh
from .experiments import (RunRecord, RunSpec, error_norms, expand_grid, run_case, stopping_study,
                          sweep)

__version__ = "0.1.0"
