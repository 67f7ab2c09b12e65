#!/usr/bin/env python
"""bench.py -- fused-sequence effective GB/s on B200 (BASELINE.json metric).

N = 1 (default workload, BASELINE.json configs[1]): the BLAS-1 chains at
n = 2^28 fp32 -- VADD (x = w + y + z) and WAXPBY (w = alpha x + beta y) --
each compiled by the planner into ONE fused sm_100a kernel.  A step is one
pass of both fused sequences over resident synthetic inputs (device-side
counter-based generator; inputs 4 GiB and 3 GiB, far larger than the 126 MB
L2, so no flush is needed between steps).

N > 1 (torchrun; default workload "auto" -> bicgk-sharded): BASELINE.json
configs[4], BiCGK 131072^2 row-sharded over the N ranks -- strong scaling,
the north star's multi-GPU path.  Every rank runs the planner's fused kernel
on its row panel; the column partials A^T r are all-reduced (NCCL) after the
kernel.  Rank 0 first times the whole problem alone on its GPU (T(1)), so
the line carries t1_ms, tN_ms and efficiency = T(1) / (N T(N)).

  value            algorithmic bytes of the step (every input read once, every
                   output written once) / device time  [GB/s, whole job]
  e2e              same metric through the public API with host buffers:
                   N = 1 the C-ABI host entry point mf_launch_host (pinned host
                   inputs copied H2D, kernels, outputs copied D2H); N > 1 the
                   row panels copied H2D from pinned host memory, the sharded
                   plan, the outputs copied D2H -- every step timed
  roofline         dominant kernel: achieved GB/s vs the measured HBM copy
                   bandwidth in MEASURED_PEAKS.json
  cpu_baseline     the reference's own CPU oracle (oracle/_ref, compiled from
                   /root/reference/proj/src) on a bounded sample, all host
                   cores, plus the serial code's 1-core figure
  speedup_vs_unfused  same step as one kernel per elementary call
  suite            the other BASELINE configs (AXPYDOT 2^24, BiCGK/ATAX 16384^2,
                   GEMVER/GESUMMV 32768^2), fused vs unfused, for context
  sharded          N = 1: BiCGK 131072^2 through the sharding layer on one GPU
                   (T(1) of the strong-scaling line), with a sampled fp64 parity
                   check
  parity           sampled rows / columns of the sharded outputs re-derived in
                   fp64 on the CPU from the counter-based generator

--workload bicgk-sharded | atax-sharded | gemver-sharded runs that sharded
line at any N (gemver: proj/data/scripts/gemver.mfs:8-11, one all-reduce of
t = B^T y per step).  --impl reference: rank 0 times the reference's CPU
implementation (reference_execute from oracle/_ref) on the same workload.
MF_BENCH_SHARED_GPU=1: every rank on cuda:0 over gloo (a one-GPU smoke run of
the multi-rank code path; numbers are not meaningful).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

N_DEFAULT = 1 << 28
METRIC = "fused-sequence effective GB/s"
WORKLOAD = "BLAS-1 chains fp32 n=2^28: VADD (x=w+y+z) + WAXPBY (w=alpha*x+beta*y), planner-fused"


# MF_BENCH_SHARED_GPU=1: every rank on cuda:0 with a gloo process group -- a
# one-GPU smoke run of the multi-rank code path (numbers are not meaningful)
SHARED_GPU = os.environ.get("MF_BENCH_SHARED_GPU", "0") == "1"


def env_rank():
    return (int(os.environ.get("RANK", "0")),
            0 if SHARED_GPU else int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def measured_peak():
    """HBM roofline denominator: the driver-measured copy bandwidth, else the
    fallback figure /opt/skills/guides/B200_PROFILING.md states (6.65 TB/s)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md, MEASURED_PEAKS.json absent)"


def host_info():
    """CPU model, logical cores and RAM of the box the CPU baseline ran on."""
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            mem_kb = int(f.readline().split()[1])
    except Exception:
        mem_kb = 0
    return {"cpu": model, "nproc": os.cpu_count(), "ram_gb": round(mem_kb / 2 ** 20, 1)}


# ---------------------------------------------------------------------------
# CPU reference arm / baseline: the reference's reference_execute from
# oracle/_ref, run on independent element slices in parallel threads (ctypes
# releases the GIL; the reference itself is serial code).

def _parallel(fn, items):
    out = [None] * len(items)

    def run(i):
        out[i] = fn(items[i])

    ths = [threading.Thread(target=run, args=(i,)) for i in range(len(items))]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return out


def cpu_reference(n_total: int, threads: int, reps: int, warmup: int):
    """VADD + WAXPBY through the reference's reference_execute over
    n_total elements split into `threads` independent slices, one thread
    each (make_problem excluded from the timing)."""
    from oracle import RefOracle
    ref = RefOracle()
    per = max(32, (n_total // threads) // 32 * 32)
    probs = _parallel(lambda t: (ref.problem("VADD", 1, per, 1 + t), ref.problem("WAXPBY", 1, per, 101 + t)),
                      list(range(threads)))

    def one(pair):
        pair[0].L.mfr_execute(pair[0].h)
        pair[1].L.mfr_execute(pair[1].h)

    for _ in range(warmup):
        _parallel(one, probs)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        _parallel(one, probs)
        times.append(time.perf_counter() - t0)
    nbytes = 28 * per * threads  # VADD 16n + WAXPBY 12n
    sec = statistics.median(times)
    return {"value": nbytes / sec / 1e9, "unit": "GB/s", "cores": threads, "kind": "reference",
            "host": host_info(),
            "sample": "reference_execute (oracle/_ref) VADD+WAXPBY on %d x %d-element slices "
                      "(%d threads, %d elements), make_problem excluded" % (threads, per, threads,
                                                                           per * threads),
            "sec_per_step": sec, "elements": per * threads}


def cpu_reference_matrix(seq: str, n: int, threads: int, rows_per_thread: int, reps: int, warmup: int):
    """`seq` (a row-shardable matrix sequence) at n columns through the
    reference's reference_execute, one independent row panel of
    `rows_per_thread` x n per host thread -- a bounded sample of the n x n
    workload with the same per-element work (make_problem excluded)."""
    from oracle import RefOracle
    ref = RefOracle()
    probs = _parallel(lambda t: ref.problem(seq, rows_per_thread, n, 1 + t), list(range(threads)))

    def one(p):
        p.L.mfr_execute(p.h)

    for _ in range(warmup):
        _parallel(one, probs)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        _parallel(one, probs)
        times.append(time.perf_counter() - t0)
    m = rows_per_thread
    per = {"BICGK": 4 * (m * n + 2 * m + 2 * n), "ATAX": 4 * (2 * m * n + m + 2 * n),
           "GEMVER": 4 * (3 * m * n + 4 * m + 7 * n)}[seq]
    sec = statistics.median(times)
    return {"value": per * threads / sec / 1e9, "unit": "GB/s", "cores": threads, "kind": "reference",
            "host": host_info(),
            "sample": "reference_execute (oracle/_ref) %s on %d independent %d x %d row panels "
                      "(%d threads), make_problem excluded" % (seq, threads, m, n, threads),
            "sec_per_step": sec, "rows": m * threads}


# ---------------------------------------------------------------------------
def make_buffers(torch, mf, plan, seed, skip_intermediate=True):
    d = plan.describe()
    bufs = {}
    for i, b in enumerate(d["buffers"]):
        if skip_intermediate and b["role"] == "intermediate":
            continue
        shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
        t = torch.empty(shp, device="cuda", dtype=torch.float32)
        if b["role"] == "input":
            mf.generate(t, seed=seed * 131 + i)
        bufs[b["name"]] = t
    return bufs, d


def time_kernels(torch, plans, steps, warmup, flush=None):
    """Runs `steps` steps; each step launches every kernel of every plan.
    Returns (total_ms over the timed region, per-kernel-name list of ms)."""
    for _ in range(warmup):
        for plan, bufs, sc in plans:
            plan.launch(bufs, sc)
    torch.cuda.synchronize()
    nk = sum(p.num_kernels for p, _, _ in plans)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps * (nk + 1))]
    per = {}
    t_total = 0.0
    if flush is None:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
    e = 0
    for s in range(steps):
        if flush is not None:
            flush[0].zero_()
            flush[1].sum()
        evs[e].record()
        for plan, bufs, sc in plans:
            for k in range(plan.num_kernels):
                plan.launch_kernel(k, bufs, sc)
                e += 1
                evs[e].record()
        e += 1
    if flush is None:
        end.record()
    torch.cuda.synchronize()
    e = 0
    for s in range(steps):
        for plan, bufs, sc in plans:
            d = plan.describe()
            for k in range(plan.num_kernels):
                ms = evs[e].elapsed_time(evs[e + 1])
                per.setdefault((d["sequence"], k, d["kernels"][k]["name"]), []).append(ms)
                e += 1
        e += 1
    if flush is None:
        t_total = start.elapsed_time(end)
    else:
        t_total = sum(sum(v) for v in per.values())
    return t_total, per


def soak_steps(torch, step, seconds, world):
    """How many untimed steps fill `seconds` (agreed over the ranks, so
    collectives inside a step stay matched): the clock sampler's window
    around the timed region is then >= `seconds` of the same load."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    n = max(1, int(seconds / max(time.perf_counter() - t0, 1e-6)))
    if world > 1:
        t = torch.tensor([n], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        n = int(t.item())
    return min(n, 100000)


def run_workload(args, torch, mf, rank, world):
    n = args.n
    sc = {"alpha": 0.5, "beta": 0.75}
    fused = [mf.Plan.sequence(s, 1, n, "fused") for s in ("VADD", "WAXPBY")]
    plans = []
    for i, p in enumerate(fused):
        bufs, d = make_buffers(torch, mf, p, seed=1 + rank * 17 + i)
        plans.append((p, bufs, sc))
    step_bytes = sum(p.describe()["bytes_loaded"] + p.describe()["bytes_stored"] for p in fused)

    def step():
        for plan, bufs, scal in plans:
            plan.launch(bufs, scal)

    n_soak = soak_steps(torch, step, 1.5, world)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    gpu_index = env_rank()[1]
    with ClockSampler(gpu_index) as clk:
        # the sampler's window: >= 1.5 s of the same load, then the timed region
        for _ in range(n_soak):
            step()
        total_ms, per = time_kernels(torch, plans, args.steps, args.warmup)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    res = {"total_ms": total_ms, "step_bytes": step_bytes, "per": per, "clocks": clk.summary(),
           "launches": args.steps * sum(p.num_kernels for p in fused)}
    # unfused chain (speedup context), same data; bytes-saved ratio from the
    # two plans' own algorithmic bytes
    unf = []
    unf_bytes = 0
    for (p, bufs, _), s in zip(plans, ("VADD", "WAXPBY")):
        up = mf.Plan.sequence(s, 1, n, "unfused")
        unf_bytes += up.describe()["bytes_loaded"] + up.describe()["bytes_stored"]
        unf.append((up, bufs, sc))
    u_ms, _ = time_kernels(torch, unf, max(2, args.steps // 2), 1)
    res["unfused_ms_per_step"] = u_ms / max(2, args.steps // 2)
    res["bytes_saved_ratio"] = unf_bytes / step_bytes
    del plans, unf
    torch.cuda.empty_cache()
    return res


def run_e2e(args, torch, mf, steps, world=1):
    """Host buffers through mf_launch_host: H2D + kernels + D2H per step.
    Under torchrun every rank runs its own slice at the same time (after a
    barrier); the time is the max over ranks and the bytes the sum."""
    import numpy as np
    n = args.n
    sc = {"alpha": 0.5, "beta": 0.75}
    h2d = d2h = 0
    specs = []
    for s in ("VADD", "WAXPBY"):
        p = mf.Plan.sequence(s, 1, n, "fused")
        d = p.describe()
        host = {}
        for b in d["buffers"]:
            if b["role"] == "intermediate":
                continue
            t = torch.empty(b["rows"] * b["cols"], dtype=torch.float32).pin_memory()
            a = t.numpy()
            if b["role"] == "input":
                a[:] = np.float32(0.25)
                h2d += a.nbytes
            else:
                d2h += a.nbytes
            host[b["name"]] = (t, a)
        specs.append((p, {k: v[1] for k, v in host.items()}, host, d))
    for p, hb, _, _ in specs:  # warm-up (allocates device mirrors)
        p.launch_host(hb, sc)
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        for p, hb, _, _ in specs:
            p.launch_host(hb, sc)
    el = time.perf_counter() - t0
    step_bytes = sum(d["bytes_loaded"] + d["bytes_stored"] for _, _, _, d in specs)
    if world > 1:
        t = torch.tensor([el], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        el = float(t.item())
    return {"value": step_bytes * world * steps / el / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world, "steps": steps,
            "path": "C-ABI mf_launch_host (pinned host buffers, H2D + fused kernels + D2H)" +
                    ("; all %d ranks concurrently, max time over ranks" % world if world > 1 else "")}


# ---------------------------------------------------------------------------
# Row-sharded sequences (BASELINE configs[4]; GEMVER per proj/data/scripts/gemver.mfs)

SHARDED_SEQ = {"bicgk-sharded": "BICGK", "atax-sharded": "ATAX", "gemver-sharded": "GEMVER"}
SHARDED_N = {"BICGK": 131072, "ATAX": 131072, "GEMVER": 65536}
SHARDED_SC = {"alpha": 0.625, "beta": 0.375}


def sharded_buffers(torch, mf, sp, n):
    """This rank's shard on the device, generated by the counter-based
    generator at GLOBAL indices (tile element (r0 + i) * n + j, row-indexed
    vector element r0 + k, column-indexed vector element j), so the CPU can
    re-derive any sampled row or column.  Returns (buffers, seed per input)."""
    d = sp.desc
    bufs, seeds = {}, {}
    for i, b in enumerate(d["buffers"]):
        if b["role"] == "intermediate":
            continue
        shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
        t = torch.empty(shp, device="cuda", dtype=torch.float32)
        if b["role"] == "input":
            seeds[b["name"]] = 11 + i
            sl = sp.local_slice(b["name"])
            if b["rows"] > 1:
                mf.generate(t, seed=11 + i, row0=sp.r0, ncols_global=n)
            elif sl is not None:
                mf.runtime._check(mf.lib().mf_generate(mf.runtime.C.c_void_p(t.data_ptr()),
                                                       t.numel(), 1, 1, 11 + i, sp.r0, 1, None))
            else:
                mf.generate(t, seed=11 + i)
        else:
            t.fill_(float("nan"))
        bufs[b["name"]] = t
    return bufs, seeds


def sharded_parity(torch, seq, sp, bufs, seeds, m, n, rank, world, k=16):
    """Sampled fp64 check of the sharded outputs:
    row outputs on k of this rank's rows, replicated column outputs on k
    columns (rank 0), against the counter-based generator's values.
    |got - ref| <= 2^-17 S + ulp(ref) elementwise and 1e-5 normwise.
    Returns the worst ratio over all ranks."""
    import numpy as np
    from oracle import COracle
    co = COracle()
    lr = sp.r1 - sp.r0
    rows_l = np.sort(np.random.default_rng(1234 + rank).choice(lr, min(k, lr), replace=False))
    rows_g = rows_l + sp.r0
    cols = np.sort(np.random.default_rng(99).choice(n, min(k, n), replace=False))
    g = lambda name, length: co.hash_fill(seeds[name], 0, length).astype(np.float64)
    host = lambda name: bufs[name].cpu().numpy()
    worst = [0.0, 0.0]  # elementwise ratio err / (tau S + ulp), normwise
    checked = []
    sc = SHARDED_SC

    def chk(name, got, ref, S):
        got = np.asarray(got, np.float64)
        err = np.abs(got - ref)
        lim = 2.0 ** -17 * S + np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
        worst[0] = max(worst[0], float(np.max(err / lim)) if np.all(np.isfinite(got)) else float("inf"))
        worst[1] = max(worst[1], float(np.max(err) / max(float(np.max(np.abs(ref))), 1e-30)))
        checked.append(name)

    if seq == "BICGK":
        qr, qa = co.hash_rows(seeds["A"], n, rows_g, g("p", n).astype(np.float32))
        chk("q", host("q")[rows_l], qr, qa)
        if rank == 0:
            sr, sa = co.hash_cols(seeds["A"], n, 0, m, cols, g("r", m).astype(np.float32))
            chk("s", host("s")[cols], sr, sa)
    elif seq == "ATAX":
        if rank == 0:
            t64, tabs = co.hash_matvec_all(seeds["A"], m, n, g("x", n).astype(np.float32))
            yr, ya = co.hash_cols_f64(seeds["A"], n, m, cols, t64, tabs)
            chk("y", host("y")[cols], yr, ya)
    elif seq == "GEMVER":
        al, be = sc["alpha"], sc["beta"]
        u1, u2, y = g("u1", m), g("u2", m), g("y", m)
        v1, v2, z = g("v1", n), g("v2", n), g("z", n)
        Arows = np.stack([co.hash_fill(seeds["A"], int(r) * n, n) for r in rows_g]).astype(np.float64)
        Brows = bufs["B"][torch.from_numpy(rows_l).cuda()].cpu().numpy()
        Bexp = (Arows + u1[rows_g, None] * v1[None, :] + u2[rows_g, None] * v2[None, :]).astype(np.float32)
        if not np.array_equal(Brows, Bexp):  # the rank-2 update is exact (fp64, rounded once)
            worst[0] = float("inf")
        checked.append("B")
        x = host("x").astype(np.float64)
        wr = al * (Brows.astype(np.float64) @ x)
        wa = abs(al) * (np.abs(Brows.astype(np.float64)) @ np.abs(x))
        chk("w", host("w")[rows_l], wr, wa)
        if rank == 0:  # x = beta B^T y + z, B = A + u1 v1^T + u2 v2^T
            ay, aya = co.hash_cols(seeds["A"], n, 0, m, cols, y.astype(np.float32))
            xr = be * (ay + v1[cols] * (u1 @ y) + v2[cols] * (u2 @ y)) + z[cols]
            xa = abs(be) * (aya + np.abs(v1[cols]) * (np.abs(u1) @ np.abs(y)) +
                            np.abs(v2[cols]) * (np.abs(u2) @ np.abs(y))) + np.abs(z[cols])
            chk("x", host("x")[cols], xr, xa)
    if world > 1:
        t = torch.tensor(worst, device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        worst = [float(v) for v in t.tolist()]
    return {"checked": checked, "rows_per_rank": int(len(rows_l)), "cols": int(len(cols)),
            "max_err_over_tol": round(worst[0], 4), "normwise": worst[1],
            "ok": bool(worst[0] <= 1.0 and worst[1] <= 1e-5),
            "oracle": "oracle/mf_oracle.c counter-based generator, fp64 (tau = 2^-17, normwise 1e-5)"}


def time_sharded(torch, sp, bufs, steps, warmup, world):
    """Device time of `steps` sharded steps (kernels + collectives) after a
    barrier, max over ranks; clocks sampled over a >= 1.5 s window of the
    same load ending with the timed region."""
    for _ in range(warmup):
        sp.launch(bufs, SHARDED_SC)
    n_soak = soak_steps(torch, lambda: sp.launch(bufs, SHARDED_SC), 1.5, world)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(env_rank()[1]) as clk:
        for _ in range(n_soak):
            sp.launch(bufs, SHARDED_SC)
        if world > 1:
            torch.cuda.synchronize()
            torch.distributed.barrier()
        start.record()
        for _ in range(steps):
            sp.launch(bufs, SHARDED_SC)
        end.record()
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    return ms / steps, clk.summary()


def run_sharded(args, torch, mf, rank, world, seq, collective="nccl", parity=True, e2e_steps=0):
    """`seq` at n_matrix^2 row-sharded over the ranks.  Each rank generates its
    row panel on the device (counter-based, global row offset), runs the
    planner's fused kernels on it and reduces the column partials after the
    kernel that produced them (NCCL all-reduce, or in-kernel over peer
    memory with collective="fused")."""
    from paper_1305_1183_b200.sharding import ShardedPlan
    m = n = args.n_matrix or SHARDED_N[seq]
    sp = ShardedPlan(seq, m, n, args.mode, collective=collective)
    d = sp.desc
    bufs, seeds = sharded_buffers(torch, mf, sp, n)
    local_bytes = d["bytes_loaded"] + d["bytes_stored"]
    ms, clocks = time_sharded(torch, sp, bufs, args.steps, args.warmup, world)
    sp.check()  # collective="fused": a peer barrier that timed out is an error, not a number
    if world > 1:
        tb = torch.tensor([local_bytes], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tb)
        total_bytes = float(tb.item())
    else:
        total_bytes = float(local_bytes)
    out = {"ms_per_step": ms, "value": total_bytes / (ms / 1e3) / 1e9, "step_bytes": total_bytes,
           "clocks": clocks, "launches": args.steps * sp.plan.num_kernels,
           "kernels": [k["name"] for k in d["kernels"]], "rows_per_rank": sp.r1 - sp.r0,
           "collectives_per_step": sum(len(c) for c in sp.collective_after), "m": m, "n": n}
    if parity:
        out["parity"] = sharded_parity(torch, seq, sp, bufs, seeds, m, n, rank, world)
    if e2e_steps > 0:
        out["e2e"] = sharded_e2e(torch, sp, bufs, e2e_steps, world, total_bytes)
    del bufs
    torch.cuda.empty_cache()
    return out


def sharded_e2e(torch, sp, bufs, steps, world, total_bytes):
    """The sharded step through the public API (ShardedPlan.launch) with the
    inputs in pinned host memory: every step copies this rank's shard H2D,
    runs the kernels + collectives and copies the outputs D2H; wall time,
    max over ranks."""
    d = sp.desc
    ins = [b["name"] for b in d["buffers"] if b["role"] == "input"]
    outs = [b["name"] for b in d["buffers"] if b["role"] == "output"]
    host = {k: torch.empty_like(bufs[k], device="cpu").pin_memory() for k in ins + outs}
    for k in ins:
        host[k].copy_(bufs[k])
    h2d = sum(host[k].numel() * 4 for k in ins)
    d2h = sum(host[k].numel() * 4 for k in outs)

    def step():
        for k in ins:
            bufs[k].copy_(host[k], non_blocking=True)
        sp.launch(bufs, SHARDED_SC)
        for k in outs:
            host[k].copy_(bufs[k], non_blocking=True)
        torch.cuda.synchronize()

    step()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        hd = torch.tensor([h2d, d2h], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(hd)
        el, h2d, d2h = float(t.item()), int(hd[0].item()), int(hd[1].item())
    del host
    return {"value": total_bytes * steps / el / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "path": "ShardedPlan.launch with every rank's shard copied H2D from pinned host memory "
                    "and the outputs copied D2H each step; wall time, max over ranks"}


def run_t1(args, torch, mf, rank, world, seq):
    """T(1): rank 0 runs the whole problem alone on its GPU (the other ranks
    wait at a barrier), before any shard is allocated."""
    res = None
    if rank == 0:
        import copy
        a1 = copy.copy(args)
        from paper_1305_1183_b200.sharding import ShardedPlan
        m = n = args.n_matrix or SHARDED_N[seq]
        sp = ShardedPlan(seq, m, n, args.mode, world=1, rank=0, collective="nccl")
        bufs, _ = sharded_buffers(torch, mf, sp, n)
        ms, _ = time_sharded(torch, sp, bufs, max(5, a1.steps), 3, 1)
        byts = sp.desc["bytes_loaded"] + sp.desc["bytes_stored"]
        res = {"t1_ms": ms, "t1_value": byts / (ms / 1e3) / 1e9}
        del bufs
        torch.cuda.empty_cache()
    if world > 1:
        torch.distributed.barrier()
    return res


def run_fused_child(args, rank, world, steps, seq):
    """Every rank starts `bench.py --workload <seq>-sharded --collective fused`
    with its own RANK / WORLD_SIZE on another rendezvous port; rank 0 returns
    the child's JSON summary (or the error).  The in-kernel peer barriers
    time out (MF_PEER_TIMEOUT_MS, a clear error instead of a hang), and the
    child itself is bounded by a wall-clock timeout."""
    import torch
    env = dict(os.environ)
    env["MASTER_PORT"] = str(int(env.get("MASTER_PORT", "29500")) + 17)
    env.setdefault("MF_PEER_TIMEOUT_MS", "2000")
    cmd = [sys.executable, os.path.abspath(__file__), "--workload", seq.lower() + "-sharded",
           "--collective", "fused", "--steps", str(steps), "--warmup", "3", "--gpus", str(world),
           "--no-t1"]
    torch.distributed.barrier()
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240)
        out = r.stdout.strip().splitlines()
        if rank != 0:
            return None
        if r.returncode != 0 or not out:
            return {"error": ("rc=%d " % r.returncode) + (r.stderr or "")[-300:]}
        d = json.loads(out[-1])
        return {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"],
                "frac_per_gpu": d["roofline"]["frac"], "workload": d["config"]["workload"],
                "parity": d.get("parity")}
    except Exception as ex:
        return {"error": str(ex)[:300]} if rank == 0 else None
    finally:
        torch.distributed.barrier()


SUITE = [("AXPYDOT", 1, 1 << 24), ("BICGK", 16384, 16384), ("ATAX", 16384, 16384),
         ("GEMVER", 32768, 32768), ("GESUMMV", 32768, 32768)]


def median_step_ms(torch, plan, bufs, sc, flush, reps=9):
    """Median over `reps` steps of the device time of one pass of the plan,
    L2 flushed before every step."""
    _, per = time_kernels(torch, [(plan, bufs, sc)], reps, 2, flush=flush)
    steps = [sum(v[i] for v in per.values()) for i in range(reps)]
    return statistics.median(steps)


def run_suite(args, torch, mf):
    # L2 flush between timed launches: write 1 GiB, then read another 1 GiB so
    # the L2 holds clean lines (no write-backs land inside the timed kernel)
    flush = (torch.empty(256 << 20, dtype=torch.float32, device="cuda"),
             torch.empty(256 << 20, dtype=torch.float32, device="cuda"))
    sc = {"alpha": 0.5, "beta": 0.75}
    peak, _ = measured_peak()
    out = {}
    for seq, m, n in SUITE:
        r = {}
        for mode in ("fused", "unfused"):
            p = mf.Plan.sequence(seq, m, n, mode)
            bufs, d = make_buffers(torch, mf, p, seed=7)
            ms = median_step_ms(torch, p, bufs, sc, flush)
            byts = d["bytes_loaded"] + d["bytes_stored"]
            r[mode] = {"us": round(ms * 1e3, 1), "GBps": round(byts / ms / 1e6, 1),
                       "bytes": byts, "kernels": p.num_kernels}
            del bufs
            torch.cuda.empty_cache()
        if seq == "ATAX":  # beyond the paper: row-resident single pass (planner mode "b200")
            p = mf.Plan.sequence(seq, m, n, "b200")
            bufs, d = make_buffers(torch, mf, p, seed=7)
            ms = median_step_ms(torch, p, bufs, sc, flush)
            byts = d["bytes_loaded"] + d["bytes_stored"]
            r["b200"] = {"us": round(ms * 1e3, 1), "GBps": round(byts / ms / 1e6, 1), "bytes": byts,
                         "kernels": p.num_kernels, "frac_of_hbm": round(byts / ms / 1e6 / peak, 3),
                         "speedup_vs_fused": round(r["fused"]["us"] / (ms * 1e3), 3)}
            del bufs
            torch.cuda.empty_cache()
        r["fused"]["frac_of_hbm"] = round(r["fused"]["GBps"] / peak, 3)
        r["speedup_vs_unfused"] = round(r["unfused"]["us"] / r["fused"]["us"], 3)
        r["bytes_saved_ratio"] = round(r["unfused"]["bytes"] / r["fused"]["bytes"], 3)
        out["%s %dx%d" % (seq, m, n) if m > 1 else "%s n=%d" % (seq, n)] = r
    del flush
    torch.cuda.empty_cache()
    return out


def traffic_entry(kernel_key):
    """roofline.traffic: DRAM bytes per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/ncu_traffic.json), with the
    capture it came from -- ncu is not run inside the bench."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    for k, v in d.items():
        if kernel_key in k and isinstance(v, dict):
            return v.get("dram_bytes_per_launch"), "profiles/ncu_traffic.json: %s (%s)" % (
                v.get("source", "?"), v.get("captured", "round-1 capture"))
    return None, None


def sharded_line(args, r, t1, world, seq, collective):
    peak, peak_kind = measured_peak()
    line = {"metric": METRIC, "value": round(r["value"], 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["ms_per_step"], 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "%s fp32 %dx%d row-sharded over %d GPU(s), column partials "
                                   "reduced %s" % (seq, r["m"], r["n"], world,
                                                   "in-kernel over NVLink peer memory"
                                                   if collective == "fused" else "by NCCL all-reduce"),
                       "rows_per_rank": r["rows_per_rank"], "kernels": r["kernels"],
                       "collectives_per_step": r["collectives_per_step"],
                       "parallelism": "row-sharded x%d" % world,
                       "l2": "inputs (%d GiB) >> L2; no flush" % (r["step_bytes"] // (1 << 30)),
                       "data": "synthetic, device-side counter-based U(-1,1) generator at global indices"},
            "roofline": {"bound": "hbm", "achieved": round(r["value"] / world, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(r["value"] / world / peak, 4),
                         "traffic": None, "peak_source": peak_kind + " (per GPU)",
                         "kernel": r["kernels"][0]},
            "clocks": r["clocks"], "gpu_launches": r["launches"]}
    if "parity" in r:
        line["parity"] = r["parity"]
    if t1 is not None:
        line["strong_scaling"] = {"t1_ms": round(t1["t1_ms"], 4), "tN_ms": round(r["ms_per_step"], 4),
                                  "n": world, "t1_value": round(t1["t1_value"], 1),
                                  "efficiency": round(t1["t1_ms"] / (world * r["ms_per_step"]), 4),
                                  "t1_how": "rank 0 alone on its GPU, whole problem, before the shards"}
    if "e2e" in r:
        line["e2e"] = r["e2e"]
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mapfuse", choices=["mapfuse", "reference"])
    ap.add_argument("--n", "--elements", dest="n", type=int, default=N_DEFAULT)
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sharded", action="store_true",
                    help="N = 1: skip the BiCGK 131072^2 sharding-layer leg")
    ap.add_argument("--no-fused-child", action="store_true",
                    help="N > 1: skip the in-kernel (NVLink peer memory) variant of the sharded line")
    ap.add_argument("--no-t1", action="store_true", help="sharded workloads: skip the T(1) run")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--workload", default="auto",
                    choices=["auto", "blas1", "bicgk-sharded", "atax-sharded", "gemver-sharded"],
                    help="auto: blas1 at N = 1, bicgk-sharded (strong scaling) at N > 1")
    ap.add_argument("--n-matrix", type=int, default=0,
                    help="sharded workloads: matrix size (0: 131072, gemver 65536)")
    ap.add_argument("--mode", default="fused", choices=["fused", "b200"],
                    help="planner mode of the sharded workloads (b200: row-resident ATAX)")
    ap.add_argument("--collective", default="nccl", choices=["fused", "nccl"],
                    help="sharded workloads: NCCL all-reduce (default) or in-kernel peer-memory reduction")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, local, world = env_rank()
    workload = args.workload
    if workload == "auto":
        workload = "blas1" if world == 1 else "bicgk-sharded"
    config = {"workload": WORKLOAD, "n": args.n, "dtype": "fp32", "parallelism": "dp%d" % world,
              "global_elements": args.n * world, "l2": "inputs (7 GiB/step) >> 126 MB L2; no flush",
              "data": "synthetic, device-side counter-based U(-1,1) generator"}

    if args.impl == "reference":
        if rank != 0:
            return
        threads = os.cpu_count() or 1
        if workload != "blas1":
            # the sharded line's workload: row panels of the n x n matrix
            seq = SHARDED_SEQ[workload]
            n = args.n_matrix or SHARDED_N[seq]
            rows = max(1, (32 << 20) // (4 * n))  # ~32 MiB of A per thread per step
            r = cpu_reference_matrix(seq, n, threads, rows, args.steps, args.warmup)
            cfg = {"workload": "%s fp32 %dx%d (reference_execute on %d-row panels, one per host thread)"
                               % (seq, n, n, rows), "n": n, "rows_sampled": r["rows"],
                   "parallelism": "host threads x%d" % threads, "data": "synthetic (make_problem)"}
            line = {"impl": "reference", "metric": METRIC, "value": round(r["value"], 3), "unit": "GB/s",
                    "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": round(r["sec_per_step"] * 1e3, 3), "higher_is_better": True,
                    "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                    "config": cfg,
                    "cpu_baseline": {"value": round(r["value"], 3), "unit": "GB/s", "cores": r["cores"],
                                     "kind": "reference", "sample": r["sample"], "host": r["host"]},
                    "e2e": {"value": round(r["value"], 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
            return
        # the stated n: every step is the whole 2^28-element workload, split
        # into one independent slice per host thread
        r = cpu_reference(args.n, threads, args.steps, args.warmup)
        line = {"impl": "reference", "metric": METRIC, "value": round(r["value"], 3),
                "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(r["sec_per_step"] * 1e3, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(config, n=r["elements"], global_elements=r["elements"],
                               note="the reference arm always runs the N = 1 BLAS-1 workload on "
                                    "the host cores"),
                "cpu_baseline": {"value": round(r["value"], 3), "unit": "GB/s",
                                 "cores": r["cores"], "kind": "reference", "sample": r["sample"],
                                 "host": r["host"]},
                "e2e": {"value": round(r["value"], 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1305_1183_b200 as mf
    mf.lib()

    if workload != "blas1":
        seq = SHARDED_SEQ[workload]
        t1 = None if args.no_t1 else run_t1(args, torch, mf, rank, world, seq)
        r = run_sharded(args, torch, mf, rank, world, seq, collective=args.collective,
                        e2e_steps=args.e2e_steps if world > 1 else 0)
        fused = None
        if (world > 1 and args.collective == "nccl" and not args.no_fused_child and not SHARED_GPU
                and args.workload == "auto"):
            # the same line with the column reduction fused into the kernel over
            # NVLink peer memory (CUDA IPC, no NCCL on the data path), in child
            # processes with their own rendezvous: a failure there cannot take
            # this line down
            torch.cuda.empty_cache()
            fused = run_fused_child(args, rank, world, args.steps, seq)
        if rank == 0:
            line = sharded_line(args, r, t1, world, seq, args.collective)
            if fused is not None:
                line["fused_collective"] = fused
            print(json.dumps(line), flush=True)
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    res = run_workload(args, torch, mf, rank, world)
    ms_per_step = res["total_ms"] / args.steps
    value = res["step_bytes"] * world * args.steps / (res["total_ms"] / 1e3) / 1e9
    # dominant kernel: fused VADD
    key = [k for k in res["per"] if k[0] == "VADD"][0]
    kms = statistics.mean(res["per"][key])
    vadd_bytes = 16 * args.n
    peak, peak_kind = measured_peak()
    achieved = vadd_bytes / (kms / 1e3) / 1e9
    traffic, traffic_src = traffic_entry("stream_kernel<3, 1, 0,")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "frac_of_nominal_8000": round(achieved / 8000.0, 4),
                "traffic": traffic, "traffic_source": traffic_src,
                "kernel": key[2], "peak_source": peak_kind,
                "algorithmic_bytes_per_launch": vadd_bytes,
                "avg_launch_us": round(kms * 1e3, 1)}
    per_kernel = {"%s/%s" % (k[0], k[2]): round(statistics.mean(v) * 1e3, 1)
                  for k, v in res["per"].items()}

    line = {"metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config, "roofline": roofline,
            "clocks": res["clocks"], "gpu_launches": res["launches"],
            "kernel_us": per_kernel,
            "speedup_vs_unfused": round(res["unfused_ms_per_step"] / ms_per_step, 3),
            "bytes_saved_ratio": round(res["bytes_saved_ratio"], 4)}
    e2e = run_e2e(args, torch, mf, args.e2e_steps, world)
    torch.cuda.empty_cache()
    sharded = None
    if not args.no_sharded and world == 1:
        # BASELINE configs[4] through the sharding layer on this one GPU: the
        # T(1) of the strong-scaling line bench.py prints at N > 1, with the
        # sampled fp64 parity check
        import copy
        sa = copy.copy(args)
        sa.mode = "fused"
        sa.steps, sa.warmup = max(5, min(args.steps, 20)), 3
        try:
            r = run_sharded(sa, torch, mf, rank, world, "BICGK")
            sharded = {"workload": "BiCGK fp32 %dx%d through the sharding layer on 1 GPU (T(1) of the "
                                   "N > 1 strong-scaling line)" % (r["m"], r["n"]),
                       "value": round(r["value"], 1), "unit": "GB/s",
                       "ms_per_step": round(r["ms_per_step"], 4), "steps": sa.steps, "scaling": "strong",
                       "rows_per_rank": r["rows_per_rank"], "frac_per_gpu": round(r["value"] / peak, 4),
                       "collectives_per_step": r["collectives_per_step"], "parity": r["parity"]}
        except Exception as ex:  # report, keep the main line
            sharded = {"error": str(ex)[:300]}
        torch.cuda.empty_cache()
        # the same config's ATAX in planner mode b200: the row-resident chain
        # over CTA clusters reads A once (BASELINE configs[4]), sampled parity
        try:
            sb = copy.copy(sa)
            sb.mode = "b200"
            r = run_sharded(sb, torch, mf, rank, world, "ATAX")
            atax = {"workload": "ATAX fp32 %dx%d, planner mode b200 (row-resident chain over CTA clusters, "
                                "one read of A) on 1 GPU" % (r["m"], r["n"]),
                    "value": round(r["value"], 1), "unit": "GB/s", "ms_per_step": round(r["ms_per_step"], 4),
                    "steps": sb.steps, "frac_per_gpu": round(r["value"] / peak, 4), "kernels": r["kernels"],
                    "parity": r["parity"]}
        except Exception as ex:
            atax = {"error": str(ex)[:300]}
        torch.cuda.empty_cache()
    if rank == 0:
        line["e2e"] = e2e
        if sharded is not None:
            line["sharded"] = sharded
            line["atax_b200"] = atax
        if world == 1 and not args.no_suite:
            line["suite"] = run_suite(args, torch, mf)
        if world == 1 and not args.no_cpu:
            try:
                cores = os.cpu_count() or 1
                # the stated workload (the reference arm's n), ~10 s of host
                # work, and the serial code as written on a 2^24 sample
                many = cpu_reference(args.n, cores, 10, 1)
                one = cpu_reference(1 << 24, 1, 5, 1)
                line["cpu_baseline"] = {k: v for k, v in many.items() if k in
                                        ("value", "unit", "cores", "kind", "sample")}
                line["cpu_baseline"]["single_core"] = {
                    "value": one["value"], "unit": "GB/s", "cores": 1,
                    "sample": one["sample"] + " -- the serial reference as written"}
            except Exception as e:  # oracle/_ref absent: say so
                line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": 0,
                                        "kind": "reference", "sample": "unavailable: %s" % e}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
