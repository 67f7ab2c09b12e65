"""Small launches of every kernel family / variant for compute-sanitizer.

  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
      python tools/sanitize_target.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

CASES = [("AXPYDOT", 1, 4096), ("VADD", 1, 4096), ("WAXPBY", 1, 2080), ("BICGK", 96, 2080),
         ("ATAX", 160, 96), ("GEMVER", 128, 4128), ("GESUMMV", 64, 2080), ("SGEMVT", 96, 160),
         ("MADD", 64, 96), ("SSCAL", 1, 96), ("SGEMV", 64, 64)]
for tma in (0, 1):
    mf.set_option("tma", tma)
    for seq, m, n in CASES:
        for mode in ("fused", "unfused"):
            plan = mf.Plan.sequence(seq, m, n, mode)
            bufs = {}
            for i, b in enumerate(plan.describe()["buffers"]):
                if b["role"] == "intermediate":
                    continue
                t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],),
                                device="cuda")
                if b["role"] == "input":
                    mf.generate(t, seed=i)
                bufs[b["name"]] = t
            plan.launch(bufs, {"alpha": 0.5, "beta": 0.25})
            torch.cuda.synchronize()
print("sanitize target done")
