"""Row-resident ATAX: the single-CTA rows kernel (n <= 16384) against the
CTA-cluster kernel forced onto the same shapes (option rowres_force_cluster,
cluster variants 0 = by SM coverage, 4, 5, 6).  L2 flushed, median of 15."""
import os, sys
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "tools"))
from matrix_overhead import make, plan_for, time_plan
import paper_1305_1183_b200 as mf
for m, n in [(16384, 16384), (8192, 8192), (32768, 16384), (16384, 8192), (65536, 4096)]:
    for force, var in [(0, 0), (1, 0), (1, 4), (1, 5), (1, 6)]:
        mf.set_option("rowres_force_cluster", force)
        mf.set_option("rowres_cluster", var)
        try:
            p = plan_for("ATAX", m, n, "b200")
            b = make(p)
            ms = [time_plan(p, b, reps=15) for _ in range(2)]
            print("ATAX %6dx%-6d force=%d var=%d %s us" % (m, n, force, var, " ".join("%.1f" % (x * 1e3) for x in ms)), flush=True)
            del b
        except Exception as e:
            print("ATAX %dx%d force=%d var=%d error %s" % (m, n, force, var, str(e)[:100]), flush=True)
mf.set_option("rowres_force_cluster", 0)
mf.set_option("rowres_cluster", 0)
