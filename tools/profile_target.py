"""Runs one fused plan per listed sequence once (plus one warm-up) -- a short
target for `ncu --set full` captures.  Usage:
  python tools/profile_target.py BICGK:16384:16384 GEMVER:32768:32768 ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

mode = os.environ.get("MF_PROFILE_MODE", "fused")
for spec in sys.argv[1:]:
    seq, m, n = spec.split(":")
    plan = mf.Plan.sequence(seq, int(m), int(n), mode)
    d = plan.describe()
    bufs = {}
    for i, b in enumerate(d["buffers"]):
        if b["role"] == "intermediate":
            continue
        shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
        t = torch.empty(shp, device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=3 + i)
        bufs[b["name"]] = t
    sc = {"alpha": 0.5, "beta": 0.75}
    for _ in range(2):
        plan.launch(bufs, sc)
    torch.cuda.synchronize()
    del bufs
    torch.cuda.empty_cache()
print("profile target done")
