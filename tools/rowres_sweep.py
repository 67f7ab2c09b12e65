"""Row-resident chain variants (option MF_SWEEP_OPTION: "rowres_cluster",
the default, or "rowres_variant" for n <= 16384) on ATAX in planner mode
b200: device time (median of 7, back-to-back launches are L2-cold at these
sizes, the L2 is flushed anyway) and the outputs' agreement with variant 1.

python tools/rowres_sweep.py [M:N ...]   (default 131072:131072 32768:32768 65536:65536;
MF_VARIANTS=1,4,5,6,7 by default: round 1 and the st.async variants)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

fa = torch.empty(256 << 20, device="cuda")
fb = torch.empty(256 << 20, device="cuda")
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
    import json
    PEAK = float(json.load(f)["hbm_gbs"])


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


specs = sys.argv[1:] or ["131072:131072", "32768:32768", "65536:65536"]
variants = [int(v) for v in os.environ.get("MF_VARIANTS", "1,4,5,6,7").split(",")]
OPTION = os.environ.get("MF_SWEEP_OPTION", "rowres_cluster")  # or rowres_variant (n <= 16384)
for spec in specs:
    m, n = (int(x) for x in spec.split(":"))
    plan = mf.Plan.sequence("ATAX", m, n, "b200")
    d = plan.describe()
    byts = d["bytes_loaded"] + d["bytes_stored"]
    bufs = {}
    for i, b in enumerate(d["buffers"]):
        if b["role"] == "intermediate":
            continue
        t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=i + 1)
        bufs[b["name"]] = t
    ref = None
    for v in variants:
        mf.set_option(OPTION, v)
        try:
            ms = time_plan(plan, bufs)
        except Exception as ex:  # unsupported shape for this variant
            print("ATAX %dx%d variant %d: %s" % (m, n, v, str(ex)[:120]), flush=True)
            continue
        y = bufs["y"].clone()
        if ref is None:
            ref = y
            agree = "ref"
        else:
            diff = (y - ref).abs().max().item()
            scale = ref.abs().max().item()
            agree = "bit-identical" if torch.equal(y, ref) else "max|dy|/max|y| = %.2e" % (diff / scale)
        print("ATAX %6dx%-6d variant %d: %9.1f us %7.0f GB/s  %.3f of HBM  (%s)" % (
            m, n, v, ms * 1e3, byts / ms / 1e6, byts / ms / 1e6 / PEAK, agree), flush=True)
    mf.set_option(OPTION, 0)
    del bufs
    torch.cuda.empty_cache()
