"""In-tree native build of libskx.so (sm_100a CUDA + C-ABI) and the C++
drop-in shim libskewdx_b200.so.

Everything is compiled explicitly with nvcc / g++ (no JIT cache), so the
built .so files live next to this module and travel with the repo snapshot
to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
CPP = os.path.join(PKG, "cpp")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIBSKX = os.path.join(PKG, "libskx.so")
LIBSHIM = os.path.join(PKG, "libskewdx_b200.so")
CLI = os.path.join(PKG, "skewdx_b200_cli")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-Wall", "-I" + INCLUDE]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: cannot build libskx.so")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def build_libskx(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    nvcc = _nvcc()
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers]):
            jobs.append([nvcc, *NVCC_FLAGS, "-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for r in ex.map(_run, jobs):
            if verbose and (r.stdout or r.stderr):
                print(r.stdout, r.stderr)
    if force or jobs or _stale(LIBSKX, objs):
        # NCCL: the libnccl.so.2 already mapped into the process is reused (torch's
        # in Python, the system one for C++ hosts) -- one soname, one library
        _run([nvcc, *ARCH, "-shared", "-o", LIBSKX, *objs, "-lcudart_static", "-lnccl", "-lrt",
              "-lpthread", "-ldl"])
    return LIBSKX


def build_shim(force: bool = False) -> str:
    """C++ drop-in (namespace skewdx, reference signatures) over the C-ABI,
    with the multi-device overloads (skewdx/multigpu.hpp)."""
    srcs = [os.path.join(CPP, "skewdx_b200.cpp"), os.path.join(CPP, "skewdx_b200_multigpu.cpp")]
    hdrs = glob.glob(os.path.join(CPP, "include", "skewdx", "*.hpp"))
    if not os.path.exists(srcs[0]):
        return ""
    if force or _stale(LIBSHIM, [*srcs, *hdrs, LIBSKX, os.path.join(INCLUDE, "skx.h")]):
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-Wall", "-Wextra", "-pthread",
              "-I" + INCLUDE, "-I" + os.path.join(CPP, "include"), *srcs, "-o", LIBSHIM,
              "-L" + PKG, "-lskx", "-Wl,-rpath,$ORIGIN"])
    return LIBSHIM


def build_cli(force: bool = False) -> str:
    """The reference CLI's `index build` / `index apply` over the drop-in."""
    src = os.path.join(CPP, "skewdx_b200_cli.cpp")
    hdrs = glob.glob(os.path.join(CPP, "include", "skewdx", "*.hpp"))
    if force or _stale(CLI, [src, *hdrs, LIBSHIM]):
        _run(["g++", "-O2", "-std=c++20", "-Wall", "-Wextra", "-I" + INCLUDE,
              "-I" + os.path.join(CPP, "include"), src, "-o", CLI, "-L" + PKG, "-lskewdx_b200",
              "-lskx", "-Wl,-rpath,$ORIGIN"])
    return CLI


def build_all(force: bool = False) -> None:
    build_libskx(force)
    build_shim(force)
    build_cli(force)


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv)
    print(LIBSKX)
