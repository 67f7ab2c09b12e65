"""Repeated-launch stress: thousands of back-to-back launches of small fused
plans (grid barriers, tickets and peer counters reset themselves between
launches); every output must stay bit-identical to the first launch's.
python tools/stress_repeat.py [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
# MF_STRESS_OPTIONS="key=value,..." runs the same cases under engine options
# (e.g. matrix_dynamic=1,matrix_waves=4: the counter-fed tile schedule resets
# its counters at the end of every launch; generic=1: the rewritten kernels)
for kv in filter(None, os.environ.get("MF_STRESS_OPTIONS", "").split(",")):
    k, v = kv.split("=")
    mf.set_option(k, int(v))
cases = [("BICGK", 256, 384, "fused"), ("AXPYDOT", 1, 1 << 16, "fused"), ("GEMVER", 128, 4128, "fused"),
         ("ATAX", 160, 96, "b200"), ("ATAX", 64, 32768, "b200"), ("GESUMMV", 96, 2080, "fused"),
         ("BICGK", 2048, 4096, "fused"), ("ATAX", 64, 65536, "b200")]
for seq, m, n, mode in cases:
    p = mf.Plan.sequence(seq, m, n, mode)
    bufs = {}
    for i, b in enumerate(p.describe()["buffers"]):
        t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=5 + i)
        bufs[b["name"]] = t
    sc = {"alpha": 0.5, "beta": 0.75}
    outs = [b["name"] for b in p.describe()["buffers"] if b["role"] == "output"]
    p.launch(bufs, sc)
    torch.cuda.synchronize()
    ref = {k: bufs[k].clone() for k in outs}
    bad = 0
    worst = 0.0
    # generic kernels sum accumulated outputs with global atomics in hardware
    # order: those are checked to 1e-5 of the output's scale, not bit for bit
    generic = mf.get_option("generic") == 1
    reps = N if m * n < 1 << 20 else N // 10
    for i in range(reps):
        p.launch(bufs, sc)
        if i % 997 == 0 or i == reps - 1:
            torch.cuda.synchronize()
            for k in outs:
                if generic:
                    scale = max(float(ref[k].abs().max()), 1e-30)
                    d = float((bufs[k] - ref[k]).abs().max()) / scale
                    worst = max(worst, d)
                    bad += d > 1e-5
                else:
                    bad += 0 if torch.equal(bufs[k], ref[k]) else 1
    torch.cuda.synchronize()
    print("%-8s %-6s %dx%d: %d launches, %d mismatching checks%s" % (
        seq, mode, m, n, reps, bad, " (max rel diff %.1e)" % worst if generic else ""), flush=True)
