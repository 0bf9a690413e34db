"""The C++ drop-in's multi-device overloads (skewdx/multigpu.hpp over the
NCCL communicator of include/skx.h): the test program compiles against the
public headers here (CPU), and on a B200 box it must reproduce the
single-device results and the reference's first-bad-row errors."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1910_10063_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "multigpu_test.cpp")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_1910_10063_b200 import build
    build.build_all()
    out = str(tmp_path_factory.mktemp("mg") / "multigpu_test")
    subprocess.check_call(["g++", "-O2", "-std=c++20", "-I" + os.path.join(PKG, "cpp", "include"),
                           SRC, "-o", out, "-L" + PKG, "-lskewdx_b200", "-lskx",
                           "-Wl,-rpath," + PKG])
    return out


def test_multigpu_program_builds(exe):
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_multigpu_overloads_equal_single_device(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "multigpu ok" in r.stdout
