"""Row-resident chain (n <= 16384): rows prefetched into L2 beyond the TMA
ring (option rowres_l2_ahead), ATAX mode b200, L2 flushed, median of 15.
python tools/rowres_l2_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from matrix_overhead import make, plan_for, time_plan  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

for m, n in [(16384, 16384), (32768, 16384), (65536, 8192), (8192, 8192), (131072, 4096)]:
    for ahead in (0, 1, 2, 3, 4, 6):
        mf.set_option("rowres_l2_ahead", ahead)
        p = plan_for("ATAX", m, n, "b200")
        b = make(p)
        ms = [time_plan(p, b, reps=15) for _ in range(2)]
        byts = p.describe()["bytes_loaded"] + p.describe()["bytes_stored"]
        print("ATAX %6dx%-6d l2_ahead=%d %s us  %.0f GB/s" % (m, n, ahead, " ".join("%.1f" % (x * 1e3) for x in ms),
                                                             byts / min(ms) / 1e6), flush=True)
        del b
mf.set_option("rowres_l2_ahead", -1)
