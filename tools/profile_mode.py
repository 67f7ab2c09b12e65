"""Like profile_target.py with a planner mode: python tools/profile_mode.py MODE SEQ:M:N ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

mode = sys.argv[1]
for spec in sys.argv[2:]:
    seq, m, n = spec.split(":")
    plan = mf.Plan.sequence(seq, int(m), int(n), mode)
    bufs = {}
    for i, b in enumerate(plan.describe()["buffers"]):
        if b["role"] == "intermediate":
            continue
        t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=3 + i)
        bufs[b["name"]] = t
    for _ in range(2):
        plan.launch(bufs, {"alpha": 0.5, "beta": 0.75})
    torch.cuda.synchronize()
    del bufs
    torch.cuda.empty_cache()
print("done")
