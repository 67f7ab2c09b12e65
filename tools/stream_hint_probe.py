"""Element-wise kernels: plain ld.global.nc vs the .L2::256B prefetch-size
hint (option stream_ld_hint).  VADD / WAXPBY / SSCAL at n = 2^28 launched
back to back (inputs >> L2), CUDA events over 50 launches, 3 repeats.
python tools/stream_hint_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

n = 1 << 28
for seq in ("VADD", "WAXPBY", "SSCAL", "MADD"):
    m_, n_ = (1, n) if seq != "MADD" else (16384, 16384)
    p = mf.Plan.sequence(seq, m_, n_, "fused")
    d = p.describe()
    bufs = {}
    for i, b in enumerate(d["buffers"]):
        if b["role"] == "intermediate":
            continue
        t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=i + 1)
        bufs[b["name"]] = t
    byts = d["bytes_loaded"] + d["bytes_stored"]
    for hint in (0, 1, 0, 1):
        mf.set_option("stream_ld_hint", hint)
        sc = {"alpha": 0.5, "beta": 0.75}
        for _ in range(3):
            p.launch(bufs, sc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            p.launch(bufs, sc)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 50
        print("%-7s hint=%d %8.1f us %7.0f GB/s" % (seq, hint, us, byts / us / 1e3), flush=True)
    del bufs
    torch.cuda.empty_cache()
mf.set_option("stream_ld_hint", 0)
