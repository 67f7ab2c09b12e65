"""Small launches of every kernel family / variant for compute-sanitizer.

  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
      python tools/sanitize_target.py [--generic] [--mutate]

--generic: every plan on the generic path (NVRTC-emitted KernelIR,
host/cudagen.cpp), plus the user functions of tests/golden/generic.mf.
--generic-fast: the generic path WITHOUT poisoning, so bounds are proved and
           the uninstrumented variant runs -- the round-2 rewrites (warp row
           reduction, deferred accumulators, global vectors, pruned barriers,
           late prefetch) -- on shapes with several serial iterations; each
           plan also with every rewrite mask of interest (generic_rewrite).
--cluster: the row-resident chain over CTA clusters (ATAX, mode b200, n >
           16384: the auto variants 4 / 5 at clusters of 2 .. 8).
--mutate:  fused BiCGK with codegen's barriers suppressed: the
           racecheck run is EXPECTED to report hazards.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

CASES = [("AXPYDOT", 1, 4096), ("VADD", 1, 4096), ("WAXPBY", 1, 2080), ("BICGK", 96, 2080),
         ("ATAX", 160, 96), ("GEMVER", 128, 4128), ("GESUMMV", 64, 2080), ("SGEMVT", 96, 160),
         ("MADD", 64, 96), ("SSCAL", 1, 96), ("SGEMV", 64, 64)]
GENERIC = "--generic" in sys.argv
FAST = "--generic-fast" in sys.argv
MUTATE = "--mutate" in sys.argv
if GENERIC or MUTATE:
    mf.set_option("generic", 1)
    mf.set_option("generic_poison", 1)
if FAST:
    mf.set_option("generic", 1)
    mf.set_option("generic_poison", 0)
    CASES = [("AXPYDOT", 1, 1 << 16), ("BICGK", 1024, 1024), ("ATAX", 512, 512), ("GEMVER", 512, 1024),
             ("GESUMMV", 512, 512), ("SGEMVT", 512, 256), ("BICGK", 256, 4096)]
if MUTATE:
    mf.set_option("codegen_barriers", 0)
    CASES = [("BICGK", 128, 128)]


def run(plan, sc):
    bufs = {}
    for i, b in enumerate(plan.describe()["buffers"]):
        if b["role"] == "intermediate":
            continue
        t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=i)
        bufs[b["name"]] = t
    plan.launch(bufs, sc)
    torch.cuda.synchronize()
    if GENERIC or FAST:
        plan.check()


if GENERIC:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tests"))
    from generic_util import GENERIC_MF, USER_SCRIPTS
    lib = open(GENERIC_MF).read()
    for s, m, n in USER_SCRIPTS.values():
        for mode in ("fused", "unfused"):
            run(mf.Plan.compile(s, m, n, mode, manifest=lib), {})
if "--cluster" in sys.argv:
    for m, n in [(32, 32768), (96, 49152), (64, 65536), (64, 131072)]:
        run(mf.Plan.sequence("ATAX", m, n, "b200"), {})
    print("sanitize target done")
    sys.exit(0)
if FAST:
    for mask in (55, 23, 31, 63, 119, 127):
        mf.set_option("generic_rewrite", mask)
        mf.set_option("generic_iterations", 0)
        for seq, m, n in CASES:
            run(mf.Plan.sequence(seq, m, n, "fused"), {"alpha": 0.5, "beta": 0.25})
        mf.set_option("generic_iterations", 8)  # several serial iterations even at these sizes
        for seq, m, n in CASES:
            run(mf.Plan.sequence(seq, m, n, "fused"), {"alpha": 0.5, "beta": 0.25})
    mf.set_option("generic_iterations", 0)
    mf.set_option("generic_rewrite", 55)
    print("sanitize target done")
    sys.exit(0)
for tma in ((0,) if GENERIC or MUTATE else (0, 1)):
    mf.set_option("tma", tma)
    for seq, m, n in CASES:
        for mode in (("fused",) if MUTATE else ("fused", "unfused")):
            run(mf.Plan.sequence(seq, m, n, mode), {"alpha": 0.5, "beta": 0.25})
print("sanitize target done")
