"""GEMVER fused: stage-1 L2 policy for A (option matrix_l2_normal: -1 auto =
evict-normal for store shapes, 0 evict-first, 1 evict-normal) x the
consumer's bottom-up rows (matrix_reverse -1 auto / 0).  Per-kernel device
time, L2 flushed before every step, median of 9.  python tools/gemver_l2_probe.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from matrix_overhead import make, plan_for  # noqa: E402

import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

fa = torch.empty(256 << 20, device="cuda")
fb = torch.empty(256 << 20, device="cuda")
sc = {"alpha": 0.5, "beta": 0.75}
for m in (32768, 16384):
    p = plan_for("GEMVER", m, m, "fused")
    b = make(p)
    for l2n, rev in ((-1, -1), (0, -1), (-1, 0), (0, 0), (-1, -1), (0, -1)):
        mf.set_option("matrix_l2_normal", l2n)
        mf.set_option("matrix_reverse", rev)
        for _ in range(3):
            p.launch(b, sc)
        per = [[] for _ in range(p.num_kernels)]
        for _ in range(9):
            fa.zero_()
            fb.sum()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(p.num_kernels + 1)]
            ev[0].record()
            for k in range(p.num_kernels):
                p.launch_kernel(k, b, sc)
                ev[k + 1].record()
            torch.cuda.synchronize()
            for k in range(p.num_kernels):
                per[k].append(ev[k].elapsed_time(ev[k + 1]) * 1e3)
        med = [statistics.median(x) for x in per]
        print("GEMVER %d^2 l2_normal=%2d reverse=%2d total %.1f us  kernels %s" % (
            m, l2n, rev, sum(med), " ".join("%.1f" % v for v in med)), flush=True)
    del b
mf.set_option("matrix_l2_normal", -1)
mf.set_option("matrix_reverse", -1)
