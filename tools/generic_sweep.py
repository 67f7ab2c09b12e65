"""Generic-path (NVRTC-emitted KernelIR) throughput on the B200 per sequence
and serial-iteration count -- the measurement behind the cost model's
"generic" efficiency (host/select.cpp) and generic_params().

  python tools/generic_sweep.py [--its 0,1,4,16,64]
Prints one line per (sequence, iterations): us, GB/s, fraction of HBM."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1305_1183_b200 as mf  # noqa: E402

CASES = [("AXPYDOT", 1, 1 << 24), ("VADD", 1, 1 << 26), ("BICGK", 16384, 16384),
         ("ATAX", 8192, 8192), ("GEMVER", 8192, 8192), ("GESUMMV", 8192, 8192), ("MADD", 8192, 8192)]


def run(seq, m, n, reps=15):
    p = mf.Plan.sequence(seq, m, n, "fused")
    d = p.describe()
    bufs = {}
    for i, b in enumerate(d["buffers"]):
        t = torch.empty((b["rows"], b["cols"]), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=3 + i)
        bufs[b["name"]] = t
    sc = {"alpha": 0.5, "beta": 0.75}
    p.prepare()
    p.launch(bufs, sc)
    p.check()
    flush = torch.empty(256 << 20, device="cuda")
    times = []
    for _ in range(reps):
        flush.zero_()  # also keeps the device busy while the launch is issued
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        p.launch(bufs, sc)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    ms = sorted(times)[len(times) // 2]  # median
    byts = d["bytes_loaded"] + d["bytes_stored"]
    its = [l.split()[1] for l in "\n".join(p.kernel_text(k) for k in range(p.num_kernels)).splitlines()
           if l.strip().startswith("iterations")]
    return ms, byts, its


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--its", default="0,1,4,16,64")
    ap.add_argument("--bys", default="0")
    ap.add_argument("--only", default="", help="comma-separated sequences")
    ap.add_argument("--opt", action="append", default=[], help="engine option key=value (repeatable)")
    a = ap.parse_args()
    mf.set_option("generic", 1)
    for kv in a.opt:
        k, v = kv.split("=")
        mf.set_option(k, int(v))
    if a.opt:
        print("# options: " + " ".join(a.opt), flush=True)
    only = set(a.only.upper().split(",")) if a.only else None
    for seq, m, n in CASES:
        if only and seq not in only:
            continue
        for by in [int(x) for x in a.bys.split(",")]:
            if by and m == 1:
                continue  # block rows only shape depth-2 kernels
            mf.set_option("generic_by", by)
            for it in [int(x) for x in a.its.split(",")]:
                mf.set_option("generic_iterations", it)
                ms, byts, its = run(seq, m, n)
                print("%-8s %6dx%-8d by=%-4s it=%-4s (%s)  %9.1f us  %7.1f GB/s  %.3f of 6650" % (
                    seq, m, n, by or "dflt", it or "auto", ",".join(its), ms * 1e3, byts / ms / 1e6,
                    byts / ms / 1e6 / 6650), flush=True)


if __name__ == "__main__":
    main()
