"""Build the C-ABI shared library ``libvanka_b200.so`` in-tree for sm_100a.

    python -m paper_2409_14222_b200.build        # or __graft_entry__.build()

Plain ``nvcc -shared`` (no torch extension machinery): the library exports
only the ``extern "C"`` symbols declared in ``include/vanka_b200.h``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libvanka_b200.so")
SOURCES = ["vk_csr.cu", "vk_patches.cu", "vk_factor.cu", "vk_apply.cu", "vk_blas.cu",
           "vk_dense.cu", "vk_assembly.cu", "vk_errors.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + \
        [os.path.join(ROOT, "include", "vanka_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    objs = []
    tmp = os.path.join(PKG, "_build")
    os.makedirs(tmp, exist_ok=True)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler",
             "-fvisibility=hidden", "--expt-relaxed-constexpr", *ARCH]
    if verbose:
        flags += ["-Xptxas", "-v"]
    flags += os.environ.get("VK_NVCC_FLAGS", "").split()  # experiments only
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")] + \
        [os.path.join(ROOT, "include", "vanka_b200.h")]
    stamp = os.path.join(tmp, "flags.txt")
    same_flags = os.path.exists(stamp) and open(stamp).read() == " ".join(flags)
    for src in SOURCES:
        obj = os.path.join(tmp, src.replace(".cu", ".o"))
        objs.append(obj)
        deps = [os.path.join(CSRC, src), *headers]
        if not force and same_flags and os.path.exists(obj) and \
                all(os.path.getmtime(d) < os.path.getmtime(obj) for d in deps):
            continue                       # object is newer than its source and every header
        cmd = [nvcc(), *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
    with open(stamp, "w") as fh:
        fh.write(" ".join(flags))
    cmd = [nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcudart"]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
