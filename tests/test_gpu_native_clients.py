"""GPU: the two native boundaries exercised from native callers.

* C++ -- vm::launch(KernelIR, DeviceConfig, LaunchArgs) with std::vector
  buffers (the reference's own call-site shape), linked against
  libmapfuse_b200.so;
* C    -- a plain C program against include/mapfuse_b200.h.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1305_1183_b200")
OUT = os.path.join(ROOT, "tests", "_build")
pytestmark = pytest.mark.gpu


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    return r.stdout


def test_cpp_vm_launch():
    os.makedirs(OUT, exist_ok=True)
    main = os.path.join(OUT, "doctest_main_gpu.cpp")
    with open(main, "w") as f:
        f.write('#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include "doctest.h"\n')
    exe = os.path.join(OUT, "vm_launch_gpu")
    _run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
          '-DMF_GENERIC_MF="%s"' % os.path.join(ROOT, "tests", "golden", "generic.mf"),
          "-I" + os.path.join(ROOT, "tests", "cpp"), "-I" + os.path.join(PKG, "csrc"),
          os.path.join(ROOT, "tests", "cpp_gpu", "test_vm_launch.cpp"), main,
          "-L" + PKG, "-lmapfuse_b200", "-Wl,-rpath," + PKG, "-o", exe])
    out = _run([exe])
    assert "failed: 0" in out


def test_c_abi_client():
    exe = os.path.join(OUT, "c_abi_client")
    os.makedirs(OUT, exist_ok=True)
    _run(["gcc", "-O1", "-I" + os.path.join(ROOT, "include"),
          os.path.join(ROOT, "tests", "cpp_gpu", "c_abi_client.c"), "-L" + PKG, "-lmapfuse_b200",
          "-Wl,-rpath," + PKG, "-o", exe])
    assert "c-abi client ok" in _run([exe])


def test_c_sharded_client_nccl():
    """mf_launch_sharded from plain C: one process, every visible GPU, NCCL
    communicators from ncclCommInitAll (on a one-GPU box the all-reduce runs
    over a single rank)."""
    exe = os.path.join(OUT, "c_sharded_client")
    os.makedirs(OUT, exist_ok=True)
    _run(["gcc", "-O1", "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
          os.path.join(ROOT, "tests", "cpp_gpu", "c_sharded_client.c"), "-L" + PKG, "-lmapfuse_b200",
          "-Wl,-rpath," + PKG, "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64",
          "-lnccl", "-lm", "-o", exe])
    assert "c sharded client ok" in _run([exe])
