"""Cross-CTA finalize probe: fused matrix / row-resident plans (L2 flushed,
median of 15, three repeats) for option finalize_group (lanes per float4
slot: 0 auto, 8, 16, 32).  python tools/finalize_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from matrix_overhead import make, plan_for, time_plan  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

for seq, m, n, mode in [("ATAX", 16384, 16384, "b200"), ("MTV", 16384, 16384, "fused"),
                        ("BICGK", 16384, 16384, "fused"), ("ATAX", 8192, 8192, "b200")]:
    for g in (8, 16, 32, 0):
        mf.set_option("finalize_group", g)
        p = plan_for(seq, m, n, mode)
        b = make(p)
        ms = [time_plan(p, b, reps=15) for _ in range(3)]
        print("%-6s %6dx%-6d %-5s G=%-4s %s us" % (seq, m, n, mode, g or "auto",
                                                   " ".join("%.1f" % (x * 1e3) for x in ms)), flush=True)
        del b
mf.set_option("finalize_group", 0)
