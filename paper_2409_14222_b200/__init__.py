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

from .assembly import System as BlockSystem, manufactured_data
from . import fem as _fem

# host discretisation objects under the reference's public names
# (stokesmg/__init__.py:15-35): same numbering, geometry and tabulations, bit
# for bit (tests/test_fem.py)
Mesh, MeshTopology, MeshGeometry = _fem.Mesh, _fem.Topology, _fem.Geometry
FunctionSpace, MixedSpace, StrongBc = _fem.Space, _fem.Mixed, _fem.StrongBc
QuadratureRule, ReferenceElement = _fem.Quadrature, _fem.Element
build_space, make_quadrature = _fem.build_space, _fem.quadrature


def build_structured_tri(n: int):
    """Reference ``meshtopo.build_structured_tri`` (``meshtopo.py:177-205``)."""
    return _fem.structured_mesh("tri", n)


def build_structured_quad(n: int):
    """Reference ``meshtopo.build_structured_quad`` (``meshtopo.py:208-231``)."""
    return _fem.structured_mesh("quad", n)


def tabulate(element, points):
    """Reference ``elements.tabulate``: (values, gradients) on the reference cell."""
    return element.tabulate(points)


__version__ = "0.1.0"
