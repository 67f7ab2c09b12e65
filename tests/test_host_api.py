"""Drop-in proof for the host C++ API (CPU).

The reference's own C++ suites (proj/tests/test_ir.cpp, test_script.cpp,
test_library.cpp) compile UNCHANGED against include/mapfuse/*.hpp and run
against the new implementation (paper_1305_1183_b200/csrc/host/).  They are
read in place from /root/reference (skipped where it is absent, e.g. on the
GPU box); tests/cpp/ holds our own suites that always run.
"""
import glob
import os
import subprocess

import pytest

from cpp_build import ROOT, build_test

REF_TESTS = "/root/reference/proj/tests"


@pytest.mark.parametrize("suite", ["test_ir", "test_script", "test_library"])
@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference sources absent")
def test_reference_suite_unchanged(suite):
    exe = build_test("ref_" + suite, [os.path.join(REF_TESTS, suite + ".cpp")])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout


OWN = sorted(glob.glob(os.path.join(ROOT, "tests", "cpp", "test_*.cpp")))


@pytest.mark.parametrize("src", OWN, ids=lambda p: os.path.basename(p)[:-4])
def test_own_cpp_suite(src):
    exe = build_test("own_" + os.path.basename(src)[:-4], [src])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr[-6000:]
