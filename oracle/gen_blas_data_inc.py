"""Generates blas_data.inc for the reference build (oracle/_ref only).

TEST INFRASTRUCTURE.  Mirrors what /root/reference/proj/CMakeLists.txt:13-33
does at configure time (embed data/blas_library.mf, data/device.cfg and the
sorted data/scripts/*.mfs as raw string literals), so the reference sources
can be compiled without running the reference's own build system.  The
output goes to oracle/_ref/gen/ (git-ignored); reference data is read in
place and never committed here.
"""
import os
import sys


def main(src_root: str, out_path: str) -> None:
    data = os.path.join(src_root, "data")
    def rd(p):
        with open(p, "r", encoding="utf-8") as f:
            return f.read()
    out = ["// generated from data/, do not edit", "#pragma once", "#include <map>",
           "#include <string>", "namespace mapfuse::blas_data {"]
    out.append('inline const char* kLibraryManifest = R"mfdata(%s)mfdata";' %
               rd(os.path.join(data, "blas_library.mf")))
    out.append('inline const char* kDeviceConfig = R"mfdata(%s)mfdata";' %
               rd(os.path.join(data, "device.cfg")))
    out.append("inline const std::map<std::string, std::string> kScripts = {")
    sdir = os.path.join(data, "scripts")
    for fn in sorted(os.listdir(sdir)):
        if fn.endswith(".mfs"):
            out.append('  {"%s", R"mfdata(%s)mfdata"},' % (fn[:-4], rd(os.path.join(sdir, fn))))
    out.append("};")
    out.append("}  // namespace mapfuse::blas_data")
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path, "w", encoding="utf-8") as f:
        f.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
