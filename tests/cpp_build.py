"""Builds C++ test executables against the product's host sources (CPU only).

Host sources: paper_1305_1183_b200/csrc/host/*.cpp (+ the plan / lowering
C++ that does not need a GPU), linked with the static CUDA runtime so the
device-query code links (it degrades gracefully without a device).
"""
import glob
import hashlib
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_1305_1183_b200", "csrc", "host")
CSRC = os.path.join(ROOT, "paper_1305_1183_b200", "csrc")
OUT = os.path.join(ROOT, "tests", "_build")
INC = ["-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ROOT, "tests", "cpp"), "-I" + CSRC,
       "-I/usr/local/cuda/include"]
LIBS = ["-L/usr/local/cuda/lib64", "-lcudart_static", "-ldl", "-lpthread", "-lrt"]
# product C++ that is pure host code (no CUDA kernels): native plan + lowering
EXTRA = ["mf_native.cpp", "mf_builtin.cpp"]


def _key(paths):
    h = hashlib.sha1()
    for p in sorted(paths) + sorted(glob.glob(os.path.join(ROOT, "include", "**", "*.h*"),
                                                recursive=True)) + \
            sorted(glob.glob(os.path.join(CSRC, "*.hpp"))):
        with open(p, "rb") as f:
            h.update(p.encode() + f.read())
    return h.hexdigest()[:16]


def host_sources():
    srcs = sorted(glob.glob(os.path.join(HOST, "*.cpp")))
    srcs += [os.path.join(CSRC, e) for e in EXTRA if os.path.exists(os.path.join(CSRC, e))]
    return srcs


def _obj(src):
    os.makedirs(OUT, exist_ok=True)
    with open(src, "rb") as f:
        d = hashlib.sha1(f.read() + _key([]).encode()).hexdigest()[:12]
    o = os.path.join(OUT, os.path.basename(src) + "." + d + ".o")
    if not os.path.exists(o):
        tmp = "%s.%d.tmp" % (o, os.getpid())
        r = subprocess.run(["g++", "-std=c++20", "-O1", "-fPIC", "-Wall"] + INC + ["-c", src, "-o", tmp],
                           capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        os.replace(tmp, o)
    return o


def _link(exe, args):
    """Links into a per-process temporary, then renames: concurrent test
    workers (pytest -n) never exec a half-written binary."""
    tmp = "%s.%d.tmp" % (exe, os.getpid())
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall"] + INC + args + ["-o", tmp],
                       capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr[-4000:])
    os.replace(tmp, exe)
    return exe


def build_tool(name, sources):
    """Compiles sources (with their own main) + host objects into OUT/name."""
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(_obj, host_sources()))
    return _link(os.path.join(OUT, name), list(sources) + objs + LIBS)


def build_test(name, test_sources):
    """Compiles test_sources + a doctest main + host objects into OUT/name."""
    main = os.path.join(OUT, "doctest_main.cpp")
    os.makedirs(OUT, exist_ok=True)
    if not os.path.exists(main):
        tmp = "%s.%d.tmp" % (main, os.getpid())
        with open(tmp, "w") as f:
            f.write('#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include "doctest.h"\n')
        os.replace(tmp, main)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(_obj, host_sources() + [main]))
    return _link(os.path.join(OUT, name), list(test_sources) + objs + LIBS)
