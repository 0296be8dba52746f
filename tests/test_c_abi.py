"""The C ABI used from plain C (tests/c/abi_demo.c): compiles here (no GPU
needed), runs on the GPU box."""

import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "c", "abi_demo.c")
LIBDIR = os.path.join(ROOT, "paper_2409_14222_b200")


def _build(out):
    cmd = ["gcc", "-O2", "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", SRC,
           "-L" + LIBDIR, "-lvanka_b200", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
           "-Wl,-rpath," + LIBDIR, "-Wl,-rpath,/usr/local/cuda/lib64", "-o", out]
    subprocess.run(cmd, check=True)


def test_c_client_compiles_and_links(tmp_path):
    _build(str(tmp_path / "abi_demo"))


@pytest.mark.gpu
def test_c_client_runs(tmp_path):
    exe = str(tmp_path / "abi_demo")
    _build(exe)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr
