"""mapfuse-b200 command line (retargeted to the B200).

  python -m paper_1305_1183_b200.cli compile  --sequence BICGK --rows 16384 --cols 16384 -o bicgk.mfp [--emit-source DIR]
  python -m paper_1305_1183_b200.cli run      bicgk.mfp [--reps 20]
  python -m paper_1305_1183_b200.cli search   --sequence GEMVER --rows 32768 --cols 32768 --top 5
  python -m paper_1305_1183_b200.cli verify   [--size 256] [--seed 1] [--top 0]
  python -m paper_1305_1183_b200.cli tune     --script s.mfs --manifest lib.mf --rows 8192 --cols 8192 [-o tuned.mfp]
  python -m paper_1305_1183_b200.cli bench-db -o cost.db      (then MF_COST_DB=cost.db)

--script FILE / --manifest FILE replace --sequence / the built-in library.
Exit codes: 0 success, 1 verification failure, 2 usage / parse error.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

from . import runtime as rt
from .runtime import MapfuseError, ParseError, Plan

SEQS = ["AXPYDOT", "VADD", "WAXPBY", "BICGK", "ATAX", "GEMVER", "GESUMMV", "SGEMV", "SGEMVT",
        "SSCAL", "MADD"]


def _script(args):
    manifest = open(args.manifest).read() if getattr(args, "manifest", None) else None
    if getattr(args, "script", None):
        return open(args.script).read(), manifest
    if not getattr(args, "sequence", None):
        raise SystemExit("need --sequence or --script")
    # the shipped script text: compile the sequence once and read it back
    return None, manifest


def _plan(args, rank=0, mode="fused"):
    text, manifest = _script(args)
    if text is None:
        if rank == 0:
            return Plan.sequence(args.sequence, args.rows, args.cols, mode)
        text = _sequence_text(args.sequence)
    return Plan.compile_ranked(text, args.rows, args.cols, rank, mode, manifest)


def _sequence_text(name):
    return rt.sequence_script(name)


def _device_buffers(plan, seed=1):
    import torch
    bufs = {}
    for i, b in enumerate(plan.describe()["buffers"]):
        if b["role"] == "intermediate":
            continue
        t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
        if b["role"] == "input":
            rt.generate(t, seed=seed + i)
        bufs[b["name"]] = t
    return bufs


def _time(plan, bufs, scalars, reps=10):
    import torch
    fa = torch.empty(256 << 20, device="cuda")
    fb = torch.empty(256 << 20, device="cuda")
    for _ in range(3):
        plan.launch(bufs, scalars)
    ts = []
    for _ in range(reps):
        fa.zero_()
        fb.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.launch(bufs, scalars)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3  # us


def cmd_compile(args):
    plan = _plan(args, 0, args.mode)
    text = plan.save()
    with open(args.output, "w") as f:
        f.write(text)
    if args.emit_source:
        os.makedirs(args.emit_source, exist_ok=True)
        for k in range(plan.num_kernels):
            with open(os.path.join(args.emit_source, "kernel%d.kir" % k), "w") as f:
                f.write(plan.kernel_text(k))
            src = plan.kernel_source(k)  # generic kernels: the emitted CUDA C++
            if src:
                with open(os.path.join(args.emit_source, "kernel%d.cu" % k), "w") as f:
                    f.write(src)
    d = plan.describe()
    print(json.dumps({"plan": args.output, "kernels": [k["name"] for k in d["kernels"]],
                      "predicted_us": plan.predicted_us,
                      "bytes": d["bytes_loaded"] + d["bytes_stored"]}))
    return 0


def cmd_run(args):
    plan = Plan.load(open(args.plan).read())
    bufs = _device_buffers(plan)
    sc = {s: 0.5 for s in plan.describe()["scalars"]}
    us = _time(plan, bufs, sc, args.reps)
    d = plan.describe()
    b = d["bytes_loaded"] + d["bytes_stored"]
    print(json.dumps({"plan": args.plan, "us": round(us, 2), "GBps": round(b / us / 1e3, 1),
                      "predicted_us": plan.predicted_us}))
    return 0


def cmd_search(args):
    """Empirical top-k search: time the k best predicted combinations, report
    the measured ranking (Table 4 analogue)."""
    text, manifest = _script(args)
    if text is None:
        text = _sequence_text(args.sequence)
    total = Plan.count_combinations(text, args.rows, args.cols, manifest)
    rows = []
    for r in range(min(args.top, total)):
        plan = Plan.compile_ranked(text, args.rows, args.cols, r, "fused", manifest)
        bufs = _device_buffers(plan)
        sc = {s: 0.5 for s in plan.describe()["scalars"]}
        us = _time(plan, bufs, sc, args.reps)
        rows.append({"rank": r, "predicted_us": round(plan.predicted_us, 2), "measured_us": round(us, 2),
                     "kernels": [k["name"] for k in plan.describe()["kernels"]]})
        del bufs
    best = min(rows, key=lambda x: x["measured_us"])
    out = {"combinations": total,
           "implementation_space": Plan.count_implementation_space(text, args.rows, args.cols, manifest),
           "evaluated": len(rows), "results": rows,
           "best_measured_rank": best["rank"],
           "rank1_vs_best": round(best["measured_us"] / rows[0]["measured_us"], 4),
           "inversions": [r["rank"] for r in rows[1:] if r["measured_us"] < rows[0]["measured_us"]]}
    print(json.dumps(out))
    return 0


def _time_kernel(plan, k, bufs, scalars, reps=7):
    """Median device time of kernel k alone, L2 flushed before each launch."""
    import torch
    fa = torch.empty(256 << 20, device="cuda")
    fb = torch.empty(256 << 20, device="cuda")
    for _ in range(2):
        plan.launch_kernel(k, bufs, scalars)
    ts = []
    for _ in range(reps):
        fa.zero_()
        fb.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.launch_kernel(k, bufs, scalars)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3  # us


def cmd_tune(args):
    """Empirical implementation search (section 5: the best of the
    generated implementations is found by measuring them): for every kernel of
    the plan that runs on the generic path, time its implementations (routine
    orders, block shapes, instances, serial iterations, memory plans; at most
    --max of them, spread evenly) on the GPU and keep the fastest.  Kernels a
    hand-written family covers are reported as such (their implementations
    lower to the same sm_100a kernel).  -o saves the tuned plan file."""
    import torch
    text, manifest = _script(args)
    if text is None:
        text = _sequence_text(args.sequence)
    chosen = {}

    def rebuild():
        p = Plan.compile(text, args.rows, args.cols, args.mode, manifest=manifest)
        for kk, ii in chosen.items():
            p.set_implementation(kk, ii)
        return p

    plan = rebuild()
    bufs = _device_buffers(plan)
    for b in plan.describe()["buffers"]:  # intermediates too: kernels run one at a time
        if b["name"] not in bufs:
            bufs[b["name"]] = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],),
                                          device="cuda")
    sc = {s_: 0.5 for s_ in plan.describe()["scalars"]}
    report = []
    for k, kern in enumerate(plan.describe()["kernels"]):
        if kern["kind"] != "generic":
            report.append({"kernel": kern["name"], "kind": kern["kind"], "tuned": False})
            continue
        cnt = plan.implementations(k)
        idx = sorted(set(range(0, cnt, max(1, cnt // args.max))) | {cnt - 1})
        base_us = _time_kernel(plan, k, bufs, sc, args.reps)
        best = (base_us, None)
        tried = []
        for i in idx:
            plan.set_implementation(k, i)
            us = _time_kernel(plan, k, bufs, sc, args.reps)
            tried.append({"implementation": i, "us": round(us, 2), **plan.implementation(k, i)})
            if us < best[0]:
                best = (us, i)
        if best[1] is not None:
            chosen[k] = best[1]
        plan = rebuild()  # the planner's choice for k unless an implementation beat it
        report.append({"kernel": kern["name"], "kind": "generic", "implementations": cnt,
                       "measured": len(tried), "default_us": round(base_us, 2),
                       "best_us": round(best[0], 2), "best_implementation": best[1],
                       "speedup": round(base_us / best[0], 3),
                       "best": tried[[t["implementation"] for t in tried].index(best[1])]
                       if best[1] is not None else None})
    if args.output:
        with open(args.output, "w") as f:
            f.write(plan.save())
    print(json.dumps({"kernels": report}))
    return 0


def cmd_verify(args):
    """Every sequence x every combination (or --top k) against the oracle."""
    import numpy as np
    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    from gpu_util import check_output, scale_bound  # test-side checkers
    from oracle import COracle
    co = COracle()
    failures = 0
    for seq in SEQS:
        m, n = (1, args.size * 16) if seq in ("AXPYDOT", "VADD", "WAXPBY", "SSCAL") else (args.size, args.size)
        text = _sequence_text(seq)
        total = Plan.count_combinations(text, m, n)
        k = total if args.top <= 0 else min(args.top, total)
        rng = np.random.default_rng(args.seed)
        for r in range(k):
            plan = Plan.compile_ranked(text, m, n, r)
            d = plan.describe()
            vals = {}
            for b in d["buffers"]:
                if b["role"] == "input":
                    shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
                    vals[b["name"]] = rng.uniform(-1, 1, shp).astype(np.float32)
            for s in d["scalars"]:
                vals[s] = float(np.float32(0.25 + 0.5 * rng.random()))
            bufs = {}
            for b in d["buffers"]:
                shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
                v = vals.get(b["name"])
                bufs[b["name"]] = (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray)
                                   else torch.zeros(shp, device="cuda"))
            plan.launch(bufs, {s: vals[s] for s in d["scalars"]})
            torch.cuda.synchronize()
            want = co.execute(seq, m, n, vals)
            S = scale_bound(co, seq, m, n, vals)
            status = "ok"
            for name in want:
                try:
                    check_output(seq, name, bufs[name].cpu().numpy(), want[name], S[name],
                                 exact=False)
                except AssertionError as e:
                    status = "FAIL %s" % e
                    failures += 1
            print("%-8s combination %d/%d (%d kernels): %s" % (seq, r + 1, total, plan.num_kernels, status))
    return 1 if failures else 0


def cmd_bench_db(args):
    """Measures per-family efficiency (fraction of HBM copy bandwidth) and
    writes the cost-model DB (MF_COST_DB format: '<key> <eta>' lines)."""
    peak = 6545.6
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = float(json.load(open(p))["hbm_gbs"])
    cases = {"stream": ("VADD", 1, 1 << 26), "stream.dot": ("AXPYDOT", 1, 1 << 24), "matrix.ldg.read": ("BICGK", 8192, 16384),
             "matrix.tma.read": ("BICGK", 8192, 16384), "matrix.ldg.rank": ("GEMVER", 8192, 16384),
             "matrix.tma.rank": ("GEMVER", 8192, 16384)}
    lines = []
    for key, (seq, m, n) in cases.items():
        rt.set_option("tma", 1 if ".tma." in key else (0 if ".ldg." in key else -1))
        plan = Plan.sequence(seq, m, n, "fused")
        d = plan.describe()
        k0 = d["kernels"][0]
        bufs = _device_buffers(plan)
        sc = {s: 0.5 for s in d["scalars"]}
        one = Plan.from_kernel_text(plan.kernel_text(0), m, n)
        names = set(k0["inputs"]) | set(k0["outputs"])
        import torch
        kb = {nm: bufs.get(nm) if nm in bufs else torch.zeros(1, device="cuda") for nm in names}
        for nm in names:
            if nm not in bufs:
                b = next(x for x in d["buffers"] if x["name"] == nm)
                kb[nm] = torch.zeros((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],),
                                     device="cuda")
        us = _time(one, kb, sc, args.reps)
        byts = one.describe()["bytes_loaded"] + one.describe()["bytes_stored"]
        eta = byts / us / 1e3 / peak
        lines.append("%s %.4f" % (key, eta))
        print("%-18s %8.1f us  eta %.3f" % (key, us, eta))
    rt.set_option("tma", -1)
    with open(args.output, "w") as f:
        f.write("\n".join(lines) + "\n")
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="mapfuse-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--sequence")
        p.add_argument("--script")
        p.add_argument("--manifest")
        p.add_argument("--rows", type=int, default=256)
        p.add_argument("--cols", type=int, default=256)

    c = sub.add_parser("compile")
    common(c)
    c.add_argument("-o", "--output", required=True)
    c.add_argument("--mode", default="fused", choices=["fused", "unfused"])
    c.add_argument("--emit-source")
    r = sub.add_parser("run")
    r.add_argument("plan")
    r.add_argument("--reps", type=int, default=20)
    s = sub.add_parser("search")
    common(s)
    s.add_argument("--top", type=int, default=5)
    s.add_argument("--reps", type=int, default=10)
    t = sub.add_parser("tune")
    common(t)
    t.add_argument("--mode", default="fused", choices=["fused", "unfused", "b200"])
    t.add_argument("--max", type=int, default=24)
    t.add_argument("--reps", type=int, default=5)
    t.add_argument("-o", "--output")
    v = sub.add_parser("verify")
    v.add_argument("--size", type=int, default=256)
    v.add_argument("--seed", type=int, default=1)
    v.add_argument("--top", type=int, default=0)
    b = sub.add_parser("bench-db")
    b.add_argument("-o", "--output", required=True)
    b.add_argument("--reps", type=int, default=10)
    args = ap.parse_args(argv)
    try:
        return {"compile": cmd_compile, "run": cmd_run, "search": cmd_search, "verify": cmd_verify,
                "bench-db": cmd_bench_db, "tune": cmd_tune}[args.cmd](args)
    except ParseError as e:
        print("error: %s" % e, file=sys.stderr)
        return 2
    except MapfuseError as e:
        print("error: %s" % e, file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
