"""Build libks.so in-tree: nvcc for sm_100a only (-gencode arch=compute_100a,code=sm_100a), static cudart.

Each .cu is compiled to an object in parallel, then linked into paper_2404_19249_b200/libks.so.
Rebuilds only when a source or header is newer than the library.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libks.so")
OBJ = os.path.join(PKG, "build")

NVCC = os.environ.get("NVCC", "nvcc")
# cuSOLVER (NEXT-1 dense pencil eigensolver) is linked dynamically from the toolkit the library was built with
CUDA_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(
    __import__("shutil").which(NVCC) or "/usr/local/cuda/bin/nvcc"))), "lib64")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
         "-I" + os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "ks.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every csrc/*.cu for sm_100a and link the shared library. `defines` (e.g. ["-DKS_PCG_SUNR=1"])
    and `out` build an A/B variant with the same flags and link line (scripts/build_variant.sh)."""
    lib = out or LIB
    if not force and not defines and out is None and not needs_build():
        return LIB
    obj_dir = OBJ if not defines and out is None else os.path.join(OBJ, os.path.basename(lib).replace(".so", ""))
    os.makedirs(obj_dir, exist_ok=True)

    def one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *defines, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        with open(obj + ".ptxas.log", "w") as f:
            f.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(one, sources()))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lcusolver", "-lcublas",
           "-Xlinker", "-rpath," + CUDA_LIB]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    if verbose:
        print("built", lib)
    return lib


if __name__ == "__main__":
    build(force=True, verbose=True)
