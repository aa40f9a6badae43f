"""In-tree build of the native library (sm_100a kernels + C-ABI host code).

The output, ``paper_1710_08314_b200/libpolar_b200.so``, is git-ignored but
travels to the GPU box with the gpurun snapshot.  nvcc cross-compiles here
without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpolar_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["host.cu", "kernels.cu", "channel.cu", "sim.cu"]
HEADERS = ["polar_dev.h", "channel.h", "primitives.cuh", "lanes.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-cudart", "static",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _deps():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "polar_b200.h"))
    files.append(os.path.join(ROOT, "include", "polar_b200_sim.h"))
    files.append(os.path.abspath(__file__))
    return [f for f in files if os.path.exists(f)]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile the library (``out``/``defines``: tuning variants)."""
    target = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    objs = []
    procs = []
    # variant builds (``out``) keep their objects out of the source tree
    objdir = CSRC if out is None else tempfile.mkdtemp(prefix="plb_build_")
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src),
               "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    tmp = target + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force=True, verbose=True)
