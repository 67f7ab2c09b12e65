"""Variant sweep on the B200 (implementation-generator evidence).

python tools/sweep.py [stream|matrix|all]
Times each fused plan at its BASELINE size for every engine variant; L2 is
flushed (write then read a 1 GiB buffer, so no dirty lines are written back
inside the timed kernel) before every timed launch; median of 7.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

PEAK = 6545.6
fa = torch.empty(256 << 20, device="cuda")
fb = torch.empty(256 << 20, device="cuda")


def make(plan):
    bufs = {}
    for i, b in enumerate(plan.describe()["buffers"]):
        if b["role"] == "intermediate":
            continue
        t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=i + 1)
        bufs[b["name"]] = t
    return bufs


def time_plan(plan, bufs, reps=7):
    sc = {"alpha": 0.5, "beta": 0.75}
    for _ in range(3):
        plan.launch(bufs, sc)
    ts = []
    for _ in range(reps):
        fa.zero_()
        fb.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.launch(bufs, sc)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def run(seq, m, n, settings, mode="fused"):
    plan = mf.Plan.sequence(seq, m, n, mode)
    d = plan.describe()
    byts = d["bytes_loaded"] + d["bytes_stored"]
    bufs = make(plan)
    for st in settings:
        for k, v in st.items():
            mf.set_option(k, v)
        ms = time_plan(plan, bufs)
        print("%-8s %-6s %-42s %9.1f us %7.0f GB/s  %.3f" % (seq, mode, st, ms * 1e3, byts / ms / 1e6,
                                                      byts / ms / 1e6 / PEAK), flush=True)
    del bufs
    torch.cuda.empty_cache()


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("stream", "all"):
    st = [{"stream_unroll": u, "stream_ctas_per_sm": c} for u in (0, 4, 8) for c in (0, 2, 4)]
    for seq, n in (("VADD", 1 << 28), ("WAXPBY", 1 << 28), ("AXPYDOT", 1 << 24)):
        run(seq, 1, n, st)
    mf.set_option("stream_unroll", 0)
    mf.set_option("stream_ctas_per_sm", 0)
if which in ("matrix", "all"):
    st = [{"tma": -1, "matrix_k": 2, "tma_consumers": 0}, {"tma": 0, "matrix_k": 2},
          {"tma": 0, "matrix_k": 4}, {"tma": 1, "matrix_k": 2}, {"tma": 1, "matrix_k": 4},
          {"tma": 1, "matrix_k": 2, "tma_consumers": 512}, {"tma": -1, "matrix_k": 2, "tma_consumers": 512}]
    for seq, m, n in (("BICGK", 16384, 16384), ("ATAX", 16384, 16384), ("GESUMMV", 32768, 32768),
                      ("GEMVER", 32768, 32768), ("BICGK", 4096, 131072)):
        run(seq, m, n, st)
    mf.set_option("tma_consumers", 0)
if which in ("rowres", "all"):
    for m, n in ((16384, 16384), (8192, 16384), (16384, 8192), (32768, 4096), (65536, 2048)):
        run("ATAX", m, n, [{"tma": -1}], "fused")
        run("ATAX", m, n, [{"rowres_variant": v} for v in (1, 2)], "b200")
    mf.set_option("rowres_variant", 0)
if which in ("occupancy", "all"):
    st = [{"tma": 0, "matrix_k": k, "occupancy": o} for k in (2, 4) for o in (1, 2, 3)]
    for seq, m, n in (("BICGK", 16384, 16384), ("SGEMV", 16384, 16384), ("SGEMVT", 16384, 16384),
                      ("GESUMMV", 16384, 16384)):
        run(seq, m, n, st)
    mf.set_option("tma", -1)
    mf.set_option("matrix_k", 2)
    mf.set_option("occupancy", 2)
