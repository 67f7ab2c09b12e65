"""Per-CTA timeline of one matrix-kernel launch (diagnostic build).

  python tools/matrix_timeline.py build          # here: builds the -DMF_TIMELINE library
  python tools/matrix_timeline.py SEQ:m:n ...    # on the B200

The diagnostic library (paper_1305_1183_b200/_build_tl/libmapfuse_tl.so)
records %globaltimer on thread 0 of every CTA at kernel entry, end of the
streaming loop, after the grid barrier, and at exit.  Printed: the spread of
each stamp over CTAs relative to the earliest entry, which splits the
kernel's time into ramp / streaming / barrier wait / cross-CTA finalize.
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
TL_OBJ = os.path.join(ROOT, "paper_1305_1183_b200", "_build_tl")
TL_LIB = os.path.join(TL_OBJ, "libmapfuse_tl.so")


def build():
    from paper_1305_1183_b200 import build as b
    print(b.build(defines=("MF_TIMELINE",), lib=TL_LIB, obj=TL_OBJ))


def main(specs):
    import ctypes as C

    import torch

    from paper_1305_1183_b200 import runtime
    runtime.LIB_PATH = TL_LIB
    import paper_1305_1183_b200 as mf
    L = mf.lib()
    L.mf_debug_timeline.argtypes = [C.c_void_p]
    fa = torch.empty(256 << 20, device="cuda")
    fb = torch.empty(256 << 20, device="cuda")
    host = (C.c_ulonglong * (5 * 4096))()
    for spec in specs:
        seq, m, n = spec.split(":")[:3]
        mode = spec.split(":")[3] if spec.count(":") >= 3 else "fused"
        plan = mf.Plan.sequence(seq, int(m), int(n), mode)
        d = plan.describe()
        bufs = {}
        for i, b in enumerate(d["buffers"]):
            if b["role"] == "intermediate":
                continue
            t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
            if b["role"] == "input":
                mf.generate(t, seed=i + 1)
            bufs[b["name"]] = t
        sc = {"alpha": 0.5, "beta": 0.75}
        L.mf_debug_timeline(C.cast(host, C.c_void_p))
        for rep in range(4):
            fa.zero_()
            fb.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.launch_kernel(0, bufs, sc)
            e1.record()
            torch.cuda.synchronize()
            if rep < 2:
                continue
            assert L.mf_debug_timeline(C.cast(host, C.c_void_p)) == 0
            rows = [[host[s * 4096 + b] for b in range(4096)] for s in range(4)]
            nb = sum(1 for x in rows[0] if x)
            if nb == 0:
                print(spec, "no stamps (kernel family not instrumented)")
                break
            t0 = min(rows[0][:nb])

            def us(s):
                v = [(x - t0) / 1e3 for x in rows[s][:nb] if x >= t0]
                return v

            out = ["%s %s k0=%s events %.1f us, CTAs %d" % (seq, spec, d["kernels"][0]["name"],
                                                          e0.elapsed_time(e1) * 1e3, nb)]
            for s, nm in enumerate(("entry", "loop_end", "barrier", "exit")):
                v = us(s)
                if v:
                    out.append("  %-8s min %7.2f  med %7.2f  max %7.2f us" % (nm, min(v),
                                                                        statistics.median(v), max(v)))
            print("\n".join(out), flush=True)
            if os.environ.get("MF_TL_DUMP") and rep == 3:
                sm = [host[4 * 4096 + b] for b in range(nb)]
                le = [(rows[1][b] - t0) / 1e3 for b in range(nb)]
                print("  per-CTA (block smid loop_end_us):", " ".join(
                    "%d:%d:%.1f" % (b, sm[b], le[b]) for b in range(nb)), flush=True)
                by_sm = {}
                for b in range(nb):
                    by_sm.setdefault(sm[b], []).append(le[b])
                slow = sorted(by_sm.items(), key=lambda kv: -max(kv[1]))[:12]
                print("  slowest SMs:", slow, flush=True)
        del bufs


if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:
        build()
    else:
        main(sys.argv[1:])
