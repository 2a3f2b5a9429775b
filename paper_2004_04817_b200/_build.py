"""In-tree build of the sm_100a shared library (``_lib/librbf_b200.so``).

nvcc cross-compiles for sm_100a without a GPU, so this runs on the CPU
build host; the built ``.so`` travels with the repo snapshot to the GPU box.
"""

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "librbf_b200.so"
SOURCES = ["rbf_capi.cu", "rbf_eval.cu", "rbf_chol.cu", "rbf_gcb.cu", "rbf_meshio.cpp"]
HEADERS = ["rbf_common.cuh", "rbf_tri.cuh", "rbf_internal.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--extended-lambda",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
]


CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-pthread"]


def _nvcc():
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cand = Path(cuda) / "bin" / "nvcc"
    return str(cand) if cand.exists() else "nvcc"


def _stale():
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "rbf_b200.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force=False, verbose=False):
    """Compile every CUDA source into one shared library (idempotent)."""
    if not force and not _stale():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = LIBDIR / (Path(src).stem + ".o")
        if src.endswith(".cpp"):  # host code: the system C++ compiler
            cuda_inc = str(Path(_nvcc()).resolve().parent.parent / "include")
            cmd = [os.environ.get("CXX", "g++"), *CXX_FLAGS, "-I", cuda_inc, "-c", str(CSRC / src),
                   "-o", str(obj)]
        else:
            # RBF_NVCC_EXTRA: extra flags for experiments (e.g. -DRBF_DEBUG_CAND)
            cmd = [_nvcc(), *NVCC_FLAGS, *os.environ.get("RBF_NVCC_EXTRA", "").split(), "-c",
                   str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
           "-o", str(tmp), *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    for o in objs:
        os.unlink(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
