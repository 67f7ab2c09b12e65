"""End-to-end (mf_launch_host) VADD + WAXPBY bench step, the two host launches
sequential vs from two threads (their pipelines overlap).  python tools/e2e_concurrent.py"""
import threading, time, sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1305_1183_b200 as mf
n = 1 << 28
specs = []
for s in ("VADD", "WAXPBY"):
    p = mf.Plan.sequence(s, 1, n, "fused")
    host = {}
    for b in p.describe()["buffers"]:
        if b["role"] == "intermediate": continue
        t = torch.empty(n, dtype=torch.float32).pin_memory(); a = t.numpy(); a[:] = 0.25
        host[b["name"]] = (t, a)
    specs.append((p, {k: v[1] for k, v in host.items()}, host))
sc = {"alpha": 0.5, "beta": 0.75}
for p, hb, _ in specs: p.launch_host(hb, sc)
nbytes = 28 * n
for mode in ("seq", "thr", "seq", "thr"):
    t0 = time.perf_counter()
    for _ in range(5):
        if mode == "seq":
            for p, hb, _ in specs: p.launch_host(hb, sc)
        else:
            ths = [threading.Thread(target=p.launch_host, args=(hb, sc)) for p, hb, _ in specs]
            [t.start() for t in ths]; [t.join() for t in ths]
    el = (time.perf_counter() - t0) / 5
    print(mode, "%.1f GB/s" % (nbytes / el / 1e9))
