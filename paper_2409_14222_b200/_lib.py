"""ctypes binding of ``libvanka_b200.so`` (declared in ``include/vanka_b200.h``).

This is the whole host<->device boundary: plain pointers, sizes and opaque
handles.  The library is built in-tree (``paper_2409_14222_b200/build.py``);
if it is missing or no CUDA device is present every compute entry point
raises — there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VK_LIB") or os.path.join(_HERE, "libvanka_b200.so")  # VK_LIB: experiment builds

VK_OK, VK_SINGULAR = 0, 1
VK_ERR_ARG, VK_ERR_CUDA, VK_ERR_ALLOC, VK_ERR_UNSUPPORTED = -1, -2, -3, -4
VK_PATCH_OK, VK_PATCH_ZERO_ROW, VK_PATCH_SMALL_PIVOT = 0, 1, 2
VK_WEIGHT_INVMULT, VK_WEIGHT_UNIT = 0, 1
VK_APPLY_OUT, VK_APPLY_XSET, VK_APPLY_XADD = 0, 1, 2
VK_REDUCE_SCRATCH = 320          # doubles of caller-owned reduction scratch

_p = C.c_void_p
_i32, _i64, _f64 = C.c_int32, C.c_int64, C.c_double
_P_i32 = C.POINTER(C.c_int32)

# name: (restype, argtypes) — mirrors include/vanka_b200.h line by line
SIGNATURES = {
    "vk_last_error": (C.c_char_p, []),
    "vk_version": (C.c_int, []),
    "vk_device_sync": (C.c_int, []),
    "vk_csr_create": (C.c_int, [_p, _p, _p, _i32, _i32, _i64, C.POINTER(_p)]),
    "vk_csr_transpose": (C.c_int, [_p, C.POINTER(_p)]),
    "vk_csr_info": (C.c_int, [_p, _P_i32, _P_i32, C.POINTER(_i64)]),
    "vk_csr_destroy": (C.c_int, [_p]),
    "vk_csr_max_abs": (C.c_int, [_p, _p]),
    "vk_csr_export": (C.c_int, [_p, _p, _p, _p]),
    "vk_spmv": (C.c_int, [_p, _p, _p, _f64, _f64, _p]),
    "vk_residual": (C.c_int, [_p, _p, _p, _p, _p]),
    "vk_residual_restrict": (C.c_int, [_p, _p, _p, _p, _p, _p, _p]),
    "vk_prolong_residual": (C.c_int, [_p, _p, _p, _p, _p, _p, _p]),
    "vk_patches_build": (C.c_int, [_p, _i32, _i32, _p, _p, _i32, _p, _p, _p, _i32, _i32,
                                   C.POINTER(_p)]),
    "vk_patches_from_lists": (C.c_int, [_p, _p, _p, _p, _i32, _i32, C.POINTER(_p)]),
    "vk_patches_info": (C.c_int, [_p, _P_i32, C.POINTER(_i64), _P_i32]),
    "vk_patches_export": (C.c_int, [_p, _p, _p, _p, _p, _p, _p]),
    "vk_extract": (C.c_int, [_p, _p, _i32, _p, _i32, _p, _p]),
    "vk_patches_extract": (C.c_int, [_p, _p, _i32, _i32, _p]),
    "vk_patches_factor": (C.c_int, [_p, _p, _p, _P_i32]),
    "vk_patches_export_inverse": (C.c_int, [_p, _i32, _i32, _p]),
    "vk_patches_apply": (C.c_int, [_p, _p, _p, _f64, _i32, _p, _p]),
    "vk_patches_solve": (C.c_int, [_p, _p, _p, _p]),
    "vk_patches_accumulate": (C.c_int, [_p, _p, _p, _f64, _i32, _p]),
    "vk_patches_apply_cheb": (C.c_int, [_p, _p, _p, _p, _f64, _f64, _i32, _p, _p]),
    "vk_patches_solve_kernel": (C.c_char_p, [_p]),
    "vk_patches_destroy": (C.c_int, [_p]),
    "vk_dot": (C.c_int, [_i64, _p, _p, _p, _p, _p]),
    "vk_axpy_dev": (C.c_int, [_i64, _p, _p, _p, _p]),
    "vk_axpy_dot": (C.c_int, [_i64, _p, _p, _p, _p, _p, _i32, _p, _p]),
    "vk_axpy": (C.c_int, [_i64, _f64, _p, _p, _p]),
    "vk_div_dev": (C.c_int, [_i64, _p, _p, _p, _p]),
    "vk_nrm2": (C.c_int, [_i64, _p, _p, _p, _p]),
    "vk_project": (C.c_int, [_i64, _p, _p, _p, _p]),
    "vk_cheb_update": (C.c_int, [_i64, _p, _p, _p, _f64, _f64, _i32, _p]),
    "vk_copy_index": (C.c_int, [_i64, _p, _p, _p, _p]),
    "vk_gemv": (C.c_int, [_i32, _i32, _p, _p, _p, _p]),
    "vk_combine": (C.c_int, [_i64, _i32, _p, _p, _p, _p]),
    "vk_csr_to_dense": (C.c_int, [_p, _p, _p]),
    "vk_assemble_cells": (C.c_int, [_i32, _i32, _i32, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p,
                                    _p, _p, _p, _p, _i32, _f64, _i64, _p, _p, _p]),
    "vk_assemble_load": (C.c_int, [_i32, _i32, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _f64,
                                   _p, _p, _p]),
    "vk_assemble_facets": (C.c_int, [_i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _f64,
                                     _f64, _i64, _p, _p, _p]),
    "vk_prolong_entries": (C.c_int, [_i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _i64, _i64,
                                     _i64, _p, _p, _p]),
    "vk_coo_to_csr": (C.c_int, [_i64, _p, _p, _i32, _i32, _i32, _f64, _p, _p, _p,
                                C.POINTER(_p)]),
    "vk_error_cells": (C.c_int, [_i32, _i32, _i32, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p,
                                 _p, _p, _p, _i32, _p, _p, _p]),
    "vk_error_jump": (C.c_int, [_i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "vk_error_reduce": (C.c_int, [_i64, _p, _i64, _p, _p, _p]),
    "vk_coarse_operator": (C.c_int, [_p, _p, _f64, _p, _p]),
    "vk_dense_inverse_workspace": (C.c_int64, [_i32]),
    "vk_dense_inverse": (C.c_int, [_i32, _p, _p, _p, _P_i32, _P_i32, _p]),
    "vk_dense_lu": (C.c_int, [_i32, _p, _p, _p, _p, _P_i32, _P_i32, _p]),
}

_lib = None


class VankaError(RuntimeError):
    """A C-ABI call failed (CUDA or unsupported configuration)."""


def load(path: str = LIB_PATH):
    """Load the shared library (no GPU needed to load and resolve symbols)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2409_14222_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _lib if _lib is not None else load()


def last_error() -> str:
    msg = lib().vk_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> int:
    if status == VK_OK or status == VK_SINGULAR:
        return status
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == VK_ERR_ARG:
        raise ValueError(msg)
    if status == VK_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise VankaError(msg)


def call(name: str, *args) -> int:
    return check(getattr(lib(), name)(*args), name)


# -------------------------------------------------------------- pointers --

def ptr(t) -> int:
    """Device (or host) address of a torch tensor / numpy array (None -> 0)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def reduce_scratch(count: int = 1):
    """Zero-filled device scratch for ``count`` independent reduction
    streams (``VK_REDUCE_SCRATCH`` doubles each); row k serves stream k."""
    import torch
    return torch.zeros((count, VK_REDUCE_SCRATCH), dtype=torch.float64, device="cuda")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise VankaError("paper_2409_14222_b200 needs a CUDA device (B200, sm_100a); "
                         "there is no CPU fallback")
    load()
    return torch
