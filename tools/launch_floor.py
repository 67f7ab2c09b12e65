"""Device time between CUDA events around one tiny plan launch (L2 flushed
before): the fixed floor every single-launch measurement carries.
python tools/launch_floor.py"""
import statistics, torch, sys
sys.path.insert(0, '.')
import paper_1305_1183_b200 as mf
fa = torch.empty(256 << 20, device="cuda"); fb = torch.empty(256 << 20, device="cuda")
for seq, m, n in [("VADD", 1, 32), ("BICGK", 32, 32), ("VADD", 1, 1 << 20)]:
    p = mf.Plan.sequence(seq, m, n, "fused")
    bufs = {}
    for i, b in enumerate(p.describe()["buffers"]):
        bufs[b["name"]] = torch.zeros((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
    for _ in range(3): p.launch(bufs, {})
    ts = []
    for _ in range(15):
        fa.zero_(); fb.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.launch(bufs, {}); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(seq, m, n, "median %.2f us" % statistics.median(ts))
