"""Run-to-run spread of the fused AXPYDOT kernel (n = 2^24) under three
timing regimes: L2 flushed before each launch, back-to-back, and flushed with
an idle gap.  python tools/axpy_variance.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402
p = mf.Plan.sequence("AXPYDOT", 1, 1 << 24, "fused")
bufs = {}
for i, b in enumerate(p.describe()["buffers"]):
    t = torch.empty(b["rows"] * b["cols"], device="cuda")
    if b["role"] == "input": mf.generate(t, seed=i)
    bufs[b["name"]] = t
fa = torch.empty(256 << 20, device="cuda"); fb = torch.empty(256 << 20, device="cuda")
sc = {"alpha": 0.5}
for _ in range(3): p.launch(bufs, sc)
for mode in ("flush", "noflush", "flush-sleep"):
    ts = []
    for _ in range(30):
        if mode != "noflush":
            fa.zero_(); fb.sum()
        if mode == "flush-sleep":
            torch.cuda._sleep(2000000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.launch(bufs, sc); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(mode, "median %.1f min %.1f max %.1f" % (statistics.median(ts), min(ts), max(ts)), [round(t, 1) for t in ts[:12]])
