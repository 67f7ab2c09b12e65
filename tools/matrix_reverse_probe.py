"""Register-fed matrix kernels reading a matrix an earlier kernel of the plan
stored: row batches bottom-up within each band (option matrix_reverse:
-1 auto = when an earlier kernel stored it, 0 never, 1 always), so the
consumer starts on the rows still in L2.  GEMVER fused plans, per-kernel
device time (L2 flushed before every step, median of 9).
python tools/matrix_reverse_probe.py"""
import os, sys, statistics
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "tools"))
from matrix_overhead import make, plan_for
import torch
import paper_1305_1183_b200 as mf
fa = torch.empty(256 << 20, device="cuda"); fb = torch.empty(256 << 20, device="cuda")
for seq, m, n in [("GEMVER", 32768, 32768), ("GEMVER", 16384, 16384)]:
    p = plan_for(seq, m, n, "fused")
    b = make(p)
    sc = {"alpha": 0.5, "beta": 0.75}
    for rev in (0, -1, 0, -1):
        mf.set_option("matrix_reverse", rev)
        for _ in range(3): p.launch(b, sc)
        tot, per = [], {}
        for _ in range(9):
            fa.zero_(); fb.sum()
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(p.num_kernels + 1)]
            evs[0].record()
            for k in range(p.num_kernels):
                p.launch_kernel(k, b, sc); evs[k + 1].record()
            torch.cuda.synchronize()
            ks = [evs[k].elapsed_time(evs[k + 1]) * 1e3 for k in range(p.num_kernels)]
            tot.append(sum(ks))
            for k, v in enumerate(ks): per.setdefault(k, []).append(v)
        print("%s %dx%d rev=%d total %.1f us  kernels %s" % (seq, m, n, rev, statistics.median(tot),
              " ".join("%.1f" % statistics.median(v) for v in per.values())), flush=True)
    del b
mf.set_option("matrix_reverse", 0)
