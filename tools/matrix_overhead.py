"""Fixed-overhead probe for the matrix kernels: device time of a fused plan
as a function of the row count m at fixed n (L2 flushed, median of 9).  The
intercept of t(m) = t0 + m * t_row is the launch + ramp + cross-CTA finalize
cost, the slope the streaming rate.

python tools/matrix_overhead.py [SEQ ...]   (default BICGK MV MTV; MV/MTV = one sgemv / sgemtv call)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

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


def time_plan(plan, bufs, reps=9):
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


SCRIPTS = {
    "MV": "TILE32x32 A;\nsubvector32 p, q;\ninput A, p;\nq = sgemv(A, p);\nreturn q;\n",
    "MTV": "TILE32x32 A;\nsubvector32 r, s;\ninput A, r;\ns = sgemtv(A, r);\nreturn s;\n",
}


def plan_for(seq, m, n, mode):
    if seq in SCRIPTS:
        return mf.Plan.compile(SCRIPTS[seq], m, n, mode)
    return mf.Plan.sequence(seq, m, n, mode)


def fit(xs, ys):
    mx, my = statistics.mean(xs), statistics.mean(ys)
    b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    return my - b * mx, b


def main():
    seqs = sys.argv[1:] or ["BICGK", "MV", "MTV"]
    settings = [dict()]
    if os.environ.get("MF_SWEEP"):
        settings = [eval(s) for s in os.environ["MF_SWEEP"].split(";")]
    n = int(os.environ.get("MF_N", "16384"))
    ms_rows = [2048, 4096, 8192, 16384, 24576]
    mode = os.environ.get("MF_MODE", "fused")
    for st in settings:
        saved = {k: mf.get_option(k) for k in st}
        for k, v in st.items():
            mf.set_option(k, v)
        for seq in seqs:
            xs, ys = [], []
            for m in ms_rows:
                plan = plan_for(seq, m, n, mode)
                d = plan.describe()
                byts = d["bytes_loaded"] + d["bytes_stored"]
                bufs = make(plan)
                ms = time_plan(plan, bufs)
                xs.append(byts / 1e9)
                ys.append(ms * 1e3)
                print("%-7s %s m=%-6d n=%d  %8.1f us  %6.0f GB/s" % (seq, st, m, n, ms * 1e3,
                                                                    byts / ms / 1e6), flush=True)
                del bufs
            t0, per_gb = fit(xs, ys)
            print("%-7s %s  intercept %.1f us, slope -> %.0f GB/s" % (seq, st, t0, 1e6 / per_gb),
                  flush=True)
        for k, v in saved.items():
            mf.set_option(k, v)


if __name__ == "__main__":
    main()
