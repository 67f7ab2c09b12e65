"""Per-kernel device time of a plan (median of 9, L2 flushed before every step):
python tools/plan_kernels.py SEQ M N [mode]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

seq, m, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
mode = sys.argv[4] if len(sys.argv) > 4 else "fused"
p = mf.Plan.sequence(seq, m, n, mode)
d = p.describe()
bufs = {}
for i, b in enumerate(d["buffers"]):
    t = torch.empty((b["rows"], b["cols"]), device="cuda")
    if b["role"] == "input":
        mf.generate(t, seed=3 + i)
    bufs[b["name"]] = t
sc = {"alpha": 0.5, "beta": 0.75}
fa, fb = torch.empty(256 << 20, device="cuda"), torch.empty(256 << 20, device="cuda")
for _ in range(2):
    p.launch(bufs, sc)
times = [[] for _ in range(p.num_kernels)]
for _ in range(9):
    fa.zero_()
    fb.sum()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(p.num_kernels + 1)]
    ev[0].record()
    for k in range(p.num_kernels):
        p.launch_kernel(k, bufs, sc)
        ev[k + 1].record()
    torch.cuda.synchronize()
    for k in range(p.num_kernels):
        times[k].append(ev[k].elapsed_time(ev[k + 1]) * 1e3)
for k, kern in enumerate(d["kernels"]):
    print("%-28s %9.1f us  variant %s" % (kern["name"], statistics.median(times[k]), kern.get("variant")))
print("total %.1f us for %d bytes -> %.1f GB/s" % (sum(statistics.median(t) for t in times),
      d["bytes_loaded"] + d["bytes_stored"],
      (d["bytes_loaded"] + d["bytes_stored"]) / sum(statistics.median(t) for t in times) / 1e3))
