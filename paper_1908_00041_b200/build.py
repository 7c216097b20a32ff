"""Build the in-tree CUDA library ``libfavest_b200.so`` for sm_100a.

    python -m paper_1908_00041_b200.build [--force] [--verbose]

One translation unit (``csrc/plan.cu`` includes the kernel headers), compiled
with ``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked
against cuFFT from the CUDA toolkit (rpath baked in, so the .so loads on the
GPU box from the same image).  No JIT cache: the built file lives next to this
module and travels with the repository snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBNAME = "libfavest_b200.so"
LIBPATH = os.path.join(HERE, LIBNAME)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    out = []
    for d in (CSRC, INCLUDE):
        for name in sorted(os.listdir(d)):
            if name.endswith((".cu", ".cuh", ".h")):
                out.append(os.path.join(d, name))
    return out


def _nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libfavest_b200.so")
    return cand


def needs_build() -> bool:
    if not os.path.exists(LIBPATH):
        return True
    t = os.path.getmtime(LIBPATH)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the library if any source is newer than it; return its path."""
    if not force and not needs_build():
        return LIBPATH
    cuda_home = os.path.dirname(os.path.dirname(os.path.realpath(_nvcc())))
    libdir = os.path.join(cuda_home, "lib64")
    tmp = LIBPATH + ".tmp"
    cmd = [
        _nvcc(), *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
        "-Xptxas", "-v" if verbose else "-O3",
        "-o", tmp, os.path.join(CSRC, "plan.cu"),
        f"-L{libdir}", "-lcufft", "-ldl", "-Xlinker", f"-rpath,{libdir}",
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}) building {LIBNAME}")
    os.replace(tmp, LIBPATH)
    return LIBPATH


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(path)
