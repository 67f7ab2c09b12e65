"""Builds the in-tree native library libmapfuse_b200.so (sm_100a).

nvcc compiles the CUDA kernel families for `-gencode arch=compute_100a,
code=sm_100a` (plus -lineinfo so ncu's source page maps to the code); g++
compiles the host C++ (the reference-compatible API, planner, codegen,
lowering, executor, C-ABI).  Everything links into ONE shared library with a
static CUDA runtime, so it loads next to torch without version coupling.
Cross-compiles without a GPU.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libmapfuse_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + os.path.join(CUDA, "include")]


def sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    return cu, cpp


def _digest(paths):
    h = hashlib.sha1()
    hdrs = sorted(glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True) +
                  glob.glob(os.path.join(ROOT, "include", "**", "*.h*"), recursive=True))
    for p in list(paths) + hdrs:
        with open(p, "rb") as f:
            h.update(p.encode() + f.read())
    return h.hexdigest()


def _compile(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("compile failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stderr


def build(verbose: bool = False, force: bool = False, defines=(), lib: str = LIB,
          obj: str = OBJ) -> str:
    """defines/lib/obj: diagnostic variants (e.g. -DMF_TIMELINE) build into
    their own object directory and library path."""
    cu, cpp = sources()
    OBJ = obj
    LIB = lib
    defs = ["-D" + d for d in defines]
    stamp = os.path.join(OBJ, "stamp")
    dig = _digest(cu + cpp + [__file__]) + " ".join(defs)
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == dig:
                return LIB
    os.makedirs(OBJ, exist_ok=True)
    jobs = []
    objs = []
    for src in cu:
        o = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(o)
        jobs.append([NVCC] + ARCH + ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC",
                                     "-Xptxas", "-v"] + defs + INC + ["-c", src, "-o", o])
    for src in cpp:
        o = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(o)
        jobs.append(["g++", "-O2", "-std=c++20", "-fPIC", "-Wall", "-Wno-unused-function"] + defs + INC +
                    ["-c", src, "-o", o])
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        logs = list(ex.map(_compile, jobs))
    if verbose:
        for l in logs:
            if l:
                sys.stderr.write(l)
    link = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + [
        "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"]
    _compile(link)
    with open(stamp, "w") as f:
        f.write(dig)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
