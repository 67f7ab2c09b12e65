"""One generic-path (NVRTC-emitted KernelIR) launch per listed sequence, for
ncu captures: python tools/profile_generic.py BICGK:16384:16384 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

mf.set_option("generic", 1)
for spec in sys.argv[1:]:
    seq, m, n = spec.split(":")
    plan = mf.Plan.sequence(seq, int(m), int(n), "fused")
    bufs = {}
    for i, b in enumerate(plan.describe()["buffers"]):
        t = torch.empty((b["rows"], b["cols"]), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=3 + i)
        bufs[b["name"]] = t
    for _ in range(2):
        plan.launch(bufs, {"alpha": 0.5, "beta": 0.75})
    torch.cuda.synchronize()
print("done")
