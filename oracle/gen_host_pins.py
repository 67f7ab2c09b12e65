"""Pins the product's shipped elementary-function library to the reference's.

TEST INFRASTRUCTURE.  Run here (oracle/_ref built from /root/reference):
    python oracle/gen_host_pins.py
Writes tests/golden/library_canonical.json: the sha256 of the canonical dump
(tests/cpp_tools/dump_host.cpp `library`) of the reference's own manifest
text -- blas::library_manifest() from the UNMODIFIED reference
(proj/data/blas_library.mf:1-438 via oracle/_ref) -- so the GPU box, which
has no /root/reference, still checks the builtin library against it.
"""
import hashlib
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def canonical(exe, manifest_text=None):
    args = [exe, "library"]
    if manifest_text is not None:
        fd, path = tempfile.mkstemp(suffix=".mf")
        with os.fdopen(fd, "w") as f:
            f.write(manifest_text)
        args.append(path)
    r = subprocess.run(args, capture_output=True, text=True, check=True)
    return r.stdout


def main():
    from cpp_build import build_tool
    from oracle import RefOracle
    exe = build_tool("dump_host", [os.path.join(ROOT, "tests", "cpp_tools", "dump_host.cpp")])
    text = canonical(exe, RefOracle().L.mfr_manifest().decode())
    out = {"sha256": hashlib.sha256(text.encode()).hexdigest(),
           "functions": text.count("\nfunction ") + text.startswith("function "),
           "routines": text.count("  routine "),
           "source": "reference blas::library_manifest() (proj/data/blas_library.mf) via oracle/_ref, "
                     "canonicalised by tests/cpp_tools/dump_host.cpp"}
    p = os.path.join(ROOT, "tests", "golden", "library_canonical.json")
    with open(p, "w") as f:
        json.dump(out, f, indent=1)
    print(p, out)


if __name__ == "__main__":
    main()
