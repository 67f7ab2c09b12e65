"""Committed pins for host pieces the product relies on (CPU).

* blas::make_problem (csrc/host/blas.cpp) against the inputs the UNMODIFIED
  reference generated (proj/src/blas.cpp:107-139, via oracle/_ref) in every
  tests/golden fixture: every input buffer bit for bit, every scalar exactly,
  every other name allocated at the padded shape and zero-filled.
* The builtin elementary-function library (generated from compact
  descriptions, csrc/host/builtin_data.cpp) against the reference's manifest
  (proj/data/blas_library.mf:1-438): all 10 functions / 42 routines, each
  routine's declared maps and printed body.  Checked live against
  oracle/_ref when it is built, and against the committed digest
  (oracle/gen_host_pins.py) always.
"""
import glob
import hashlib
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

from cpp_build import ROOT, build_tool

GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.npz")))


@pytest.fixture(scope="module")
def dump_host():
    return build_tool("dump_host", [os.path.join(ROOT, "tests", "cpp_tools", "dump_host.cpp")])


def product_problem(exe, seq, rows, cols, seed):
    d = tempfile.mkdtemp(prefix="mfpin")
    subprocess.run([exe, "problem", seq, str(rows), str(cols), str(seed), d], check=True)
    bufs, scal, padded = {}, {}, None
    with open(os.path.join(d, "index.txt")) as f:
        for line in f:
            kind, *rest = line.split()
            if kind == "padded":
                padded = (int(rest[0]), int(rest[1]))
            elif kind == "buffer":
                name, r, c = rest[0], int(rest[1]), int(rest[2])
                a = np.fromfile(os.path.join(d, name + ".f32"), dtype=np.float32)
                assert a.size == r * c, name
                bufs[name] = a.reshape(r, c)
            else:
                scal[rest[0]] = float.fromhex(rest[1])
    return padded, bufs, scal


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_make_problem_matches_reference_inputs(dump_host, path):
    g = np.load(path)
    meta = json.loads(str(g["meta"]))
    rq = meta["requested"]
    padded, bufs, scal = product_problem(dump_host, meta["sequence"], rq[0], rq[1], meta["seed"])
    assert padded == (meta["rows"], meta["cols"])
    for name, shape in meta["inputs"]:
        if shape is None:  # scalar: 0.25 + 0.5|U| drawn after the buffers
            assert np.float32(scal[name]) == g["sc__" + name], name
            continue
        want = g["in__" + name]
        got = bufs[name]
        assert got.shape == tuple(shape), (name, got.shape, shape)
        assert np.array_equal(got.reshape(want.shape), want), name
    inputs = {n for n, _ in meta["inputs"]}
    for name in meta["outputs"]:  # reduce outputs must start at 0 (vm.hpp:91-93)
        assert name in bufs and not bufs[name].any(), name
        assert bufs[name].size == g["out__" + name].size, name
    for name, a in bufs.items():
        if name not in inputs:
            assert not a.any(), name


def _canonical(exe, manifest_text=None):
    args = [exe, "library"]
    if manifest_text is not None:
        fd, path = tempfile.mkstemp(suffix=".mf")
        with os.fdopen(fd, "w") as f:
            f.write(manifest_text)
        args.append(path)
    return subprocess.run(args, capture_output=True, text=True, check=True).stdout


def test_builtin_library_matches_reference_manifest(dump_host):
    mine = _canonical(dump_host)
    with open(os.path.join(ROOT, "tests", "golden", "library_canonical.json")) as f:
        pin = json.load(f)
    assert mine.count("  routine ") == pin["routines"] == 42
    assert mine.count("function ") == pin["functions"] == 10
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import RefOracle
    if RefOracle.available():  # live: the reference's own manifest text
        ref = _canonical(dump_host, RefOracle().L.mfr_manifest().decode())
        if ref != mine:
            import difflib
            diff = "".join(list(difflib.unified_diff(ref.splitlines(True), mine.splitlines(True),
                                                     "reference", "builtin"))[:60])
            pytest.fail("builtin library differs from the reference manifest:\n" + diff)
    assert hashlib.sha256(mine.encode()).hexdigest() == pin["sha256"]


@pytest.mark.parametrize("seq,rows,cols,seed", [("GEMVER", 100, 200, 3), ("GESUMMV", 64, 64, 9),
                                                ("AXPYDOT", 1, 4000, 5), ("MADD", 70, 33, 2)])
def test_make_problem_matches_live_reference(dump_host, seq, rows, cols, seed):
    """Shapes beyond the fixtures, against oracle/_ref directly (skipped when
    it is not built)."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import RefOracle
    if not RefOracle.available():
        pytest.skip("oracle/_ref not built")
    p = RefOracle().problem(seq, rows, cols, seed)
    padded, bufs, scal = product_problem(dump_host, seq, rows, cols, seed)
    assert padded == (p.rows, p.cols)
    for name in p.inputs:
        if name in p.scalars:
            assert np.float32(scal[name]) == np.float32(p.scalar(name)), name
        else:
            want = p.buffer(name)
            assert np.array_equal(bufs[name].reshape(want.shape), want), name
