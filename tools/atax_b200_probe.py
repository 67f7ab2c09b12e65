"""ATAX 131072^2 mode b200 on one GPU: the plan launched directly (L2
flushed per step, median) vs the sharding layer's back-to-back steps at
world = 1 (bench.py's atax_b200 leg).  python tools/atax_b200_probe.py"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402
from matrix_overhead import make, plan_for, time_plan  # noqa: E402

n = 131072
p = plan_for("ATAX", n, n, "b200")
b = make(p)
print("plan, L2 flushed, median of 9: %.2f ms" % (time_plan(p, b) * 1.0), flush=True)
sc = {"alpha": 0.5, "beta": 0.75}
for _ in range(3):
    p.launch(b, sc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    p.launch(b, sc)
e1.record()
torch.cuda.synchronize()
print("plan, 20 back-to-back launches: %.2f ms each" % (e0.elapsed_time(e1) / 20), flush=True)
del b
torch.cuda.empty_cache()
from paper_1305_1183_b200.sharding import ShardedPlan  # noqa: E402
sp = ShardedPlan("ATAX", n, n, "b200", world=1, rank=0)
print("sharded plan kernels:", [k["name"] for k in sp.desc["kernels"]], flush=True)
