"""Plan-level vs per-kernel device time (L2 flushed, median of 15): how much
launch gap a multi-kernel plan pays back to back -- the headroom programmatic
dependent launch could recover.  python tools/plan_gap_probe.py"""
import os, sys, statistics
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "tools"))
from matrix_overhead import make, plan_for
import torch
import paper_1305_1183_b200 as mf
fa = torch.empty(256 << 20, device="cuda"); fb = torch.empty(256 << 20, device="cuda")
sc = {"alpha": 0.5, "beta": 0.75}
for seq, m, n, mode in [("GEMVER", 16384, 16384, "fused"), ("GEMVER", 8192, 8192, "fused"), ("GESUMMV", 8192, 8192, "fused"),
                        ("BICGK", 8192, 8192, "unfused"), ("ATAX", 8192, 8192, "fused")]:
    p = plan_for(seq, m, n, mode); b = make(p)
    for _ in range(3): p.launch(b, sc)
    whole, parts = [], []
    for _ in range(15):
        fa.zero_(); fb.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.launch(b, sc); e1.record(); torch.cuda.synchronize()
        whole.append(e0.elapsed_time(e1) * 1e3)
        fa.zero_(); fb.sum()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(p.num_kernels + 1)]
        evs[0].record()
        for k in range(p.num_kernels):
            p.launch_kernel(k, b, sc); evs[k + 1].record()
        torch.cuda.synchronize()
        parts.append([evs[k].elapsed_time(evs[k + 1]) * 1e3 for k in range(p.num_kernels)])
    pm = [statistics.median(x[k] for x in parts) for k in range(p.num_kernels)]
    print("%-8s %5dx%-5d %-7s whole %.1f us  per-kernel %s (sum %.1f)" % (seq, m, n, mode, statistics.median(whole),
          " ".join("%.1f" % v for v in pm), sum(pm)), flush=True)
    del b
