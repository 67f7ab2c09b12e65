"""Matrix-kernel tile schedule probe: device time of fused BiCGK / GESUMMV /
SGEMV / SGEMVT plans for option matrix_waves (tiles per co-resident CTA) x
matrix_dynamic (tiles after the first from a counter), L2 flushed, median of
15.  python tools/matrix_waves.py [SEQ:m:n ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from matrix_overhead import make, plan_for, time_plan  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

specs = sys.argv[1:] or ["BICGK:16384:16384", "MV:16384:16384", "MTV:16384:16384", "BICGK:8192:8192",
                         "GESUMMV:16384:16384"]
for spec in specs:
    seq, m, n = spec.split(":")
    m, n = int(m), int(n)
    for waves, dyn in [(1, 0), (2, 0), (2, 1), (4, 0), (4, 1), (8, 1)]:
        mf.set_option("matrix_waves", waves)
        mf.set_option("matrix_dynamic", dyn)
        p = plan_for(seq, m, n, "fused")
        bufs = make(p)
        ms = time_plan(p, bufs, reps=15)
        d = p.describe()
        byts = d["bytes_loaded"] + d["bytes_stored"]
        print("%-8s %6dx%-6d waves=%d dyn=%d  %8.1f us  %7.1f GB/s" % (seq, m, n, waves, dyn, ms * 1e3,
                                                                     byts / ms / 1e6), flush=True)
        del bufs
mf.set_option("matrix_waves", 1)
mf.set_option("matrix_dynamic", 0)
