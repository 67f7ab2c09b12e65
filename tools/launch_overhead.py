"""Host cost of one plan launch (tiny problem, so the GPU is never the
bottleneck): Plan.launch vs a bound plan vs one CUDA-graph launch.
python tools/launch_overhead.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402


def per_launch(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


for seq, m, n in [("VADD", 1, 4096), ("AXPYDOT", 1, 4096), ("BICGK", 256, 256), ("GEMVER", 256, 256)]:
    p = mf.Plan.sequence(seq, m, n, "fused")
    d = p.describe()
    bufs = {b["name"]: torch.zeros((b["rows"], b["cols"]), device="cuda") for b in d["buffers"]}
    sc = {"alpha": 0.5, "beta": 0.25}
    s = torch.cuda.Stream()
    bound = p.bind(bufs, sc)
    a = per_launch(lambda: p.launch(bufs, sc))
    b = per_launch(lambda: bound.launch(s))
    c = per_launch(lambda: bound.graph_launch(s))
    print("%-8s kernels %d: Plan.launch %.1f us, bound %.1f us, graph %.1f us per plan launch" % (
        seq, p.num_kernels, a, b, c), flush=True)
