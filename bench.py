#!/usr/bin/env python
"""bench.py -- fused-sequence effective GB/s on B200 (BASELINE.json metric).

Default workload (BASELINE.json configs[1]): the BLAS-1 chains at
n = 2^28 fp32 -- VADD (x = w + y + z) and WAXPBY (w = alpha x + beta y) --
each compiled by the planner into ONE fused sm_100a kernel.  A step is one
pass of both fused sequences over resident synthetic inputs (device-side
counter-based generator; inputs 4 GiB and 3 GiB, far larger than the 126 MB
L2, so no flush is needed between steps).

  value            algorithmic bytes of the step (every input read once, every
                   output written once) / device time  [GB/s, whole job]
  e2e              same metric through the C-ABI host entry point
                   (mf_launch_host): pinned host inputs copied H2D, kernels,
                   outputs copied D2H, every step inside the timed region
  roofline         dominant kernel (fused VADD): achieved GB/s vs the measured
                   HBM copy bandwidth in MEASURED_PEAKS.json
  cpu_baseline     the reference's own CPU oracle (oracle/_ref, compiled from
                   /root/reference/proj/src) on a bounded sample, all host cores
  speedup_vs_unfused  same step as one kernel per elementary call
  suite            the other BASELINE configs (AXPYDOT 2^24, BiCGK/ATAX 16384^2,
                   GEMVER/GESUMMV 32768^2), fused vs unfused, for context
  sharded          BASELINE configs[4]: BiCGK 131072^2 row-sharded over the N
                   ranks (strong scaling, NCCL all-reduce of A^T r); at N = 1
                   it is T(1) for the efficiency T(1)/(N T(N)); at N > 1 also
                   `fused_collective`: the same leg with A^T r reduced inside
                   the kernel over NVLink peer memory (child processes)

Multi-GPU (torchrun): every rank runs the workload on its own GPU on its own
slice (element-wise sequences shard with no exchange; "scaling": "weak");
time = max over ranks of the device-timed region.

--impl reference: rank 0 times the reference's CPU implementation
(reference_execute from oracle/_ref) on the same workload and metric.
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


def ncu_traffic(kernel_key: str):
    """DRAM bytes per launch of the kernel whose template name contains
    kernel_key, from the committed ncu capture (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    for k, v in d.items():
        if kernel_key in k:
            return v.get("dram_bytes_per_launch") if isinstance(v, dict) else v
    return None


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

def cpu_reference(n_total: int, threads: int, reps: int, warmup: int):
    from oracle import RefOracle
    ref = RefOracle()
    per = max(32, (n_total // threads) // 32 * 32)
    probs = []
    for t in range(threads):
        probs.append((ref.problem("VADD", 1, per, 1 + t), ref.problem("WAXPBY", 1, per, 101 + t)))

    def one(pair):
        pair[0].L.mfr_execute(pair[0].h)
        pair[1].L.mfr_execute(pair[1].h)

    def step():
        ths = [threading.Thread(target=one, args=(p,)) for p in probs]
        for th in ths:
            th.start()
        for th in ths:
            th.join()

    for _ in range(warmup):
        step()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    nbytes = 28 * per * threads  # VADD 16n + WAXPBY 12n
    sec = statistics.median(times)
    return {"value": nbytes / sec / 1e9, "unit": "GB/s", "cores": threads, "kind": "reference",
            "host": host_info(),
            "sample": "reference_execute (oracle/_ref) VADD+WAXPBY on %d x %d-element slices "
                      "(%d threads), make_problem excluded" % (threads, per, threads),
            "sec_per_step": sec, "elements": per * threads}


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
        first = e
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


def run_workload(args, torch, mf, rank, world):
    n = args.n
    sc = {"alpha": 0.5, "beta": 0.75}
    fused = [mf.Plan.sequence(s, 1, n, "fused") for s in ("VADD", "WAXPBY")]
    plans = []
    for i, p in enumerate(fused):
        bufs, d = make_buffers(torch, mf, p, seed=1 + rank * 17 + i)
        plans.append((p, bufs, sc))
    step_bytes = sum(p.describe()["bytes_loaded"] + p.describe()["bytes_stored"] for p in fused)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    gpu_index = env_rank()[1]
    with ClockSampler(gpu_index) as clk:
        total_ms, per = time_kernels(torch, plans, args.steps, args.warmup)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    res = {"total_ms": total_ms, "step_bytes": step_bytes, "per": per, "clocks": clk.summary(),
           "launches": args.steps * sum(p.num_kernels for p in fused)}
    # unfused chain (speedup context), same data
    unf = []
    for (p, bufs, _), s in zip(plans, ("VADD", "WAXPBY")):
        up = mf.Plan.sequence(s, 1, n, "unfused")
        unf.append((up, bufs, sc))
    u_ms, _ = time_kernels(torch, unf, max(2, args.steps // 2), 1)
    res["unfused_ms_per_step"] = u_ms / max(2, args.steps // 2)
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
    out = []
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


def run_sharded(args, torch, mf, rank, world, seq):
    """BiCGK / ATAX at 131072^2 row-sharded over the ranks (BASELINE configs[4]).
    Each rank generates its row panel on the device (counter-based, global
    row offset), runs the planner's fused kernels on it, and all-reduces the
    column partials (NCCL) after the kernel that produced them."""
    from paper_1305_1183_b200.sharding import ShardedPlan
    m = n = args.n_matrix
    sp = ShardedPlan(seq, m, n, args.mode, collective=args.collective)
    d = sp.desc
    bufs = {}
    for i, b in enumerate(d["buffers"]):
        if b["role"] == "intermediate":
            continue
        shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
        t = torch.empty(shp, device="cuda", dtype=torch.float32)
        if b["role"] == "input":
            sl = sp.local_slice(b["name"])
            if b["rows"] > 1:  # tile row panel: global element index (r0 + i) * n + j
                mf.generate(t, seed=11 + i, row0=sp.r0, ncols_global=n)
            elif sl is not None:  # row-indexed vector slice
                mf.runtime._check(mf.lib().mf_generate(mf.runtime.C.c_void_p(t.data_ptr()),
                                                       t.numel(), 1, 1, 11 + i, sp.r0, 1, None))
            else:
                mf.generate(t, seed=11 + i)
        bufs[b["name"]] = t
    local_bytes = d["bytes_loaded"] + d["bytes_stored"]
    for _ in range(args.warmup):
        sp.launch(bufs, {})
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    gpu_index = env_rank()[1]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_index) as clk:
        start.record()
        for _ in range(args.steps):
            sp.launch(bufs, {})
        end.record()
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        tb = torch.tensor([local_bytes], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tb)
        total_bytes = float(tb.item())
    else:
        total_bytes = float(local_bytes)
    return {"ms_per_step": ms / args.steps, "value": total_bytes * args.steps / (ms / 1e3) / 1e9,
            "clocks": clk.summary(), "launches": args.steps * sp.plan.num_kernels,
            "kernels": [k["name"] for k in d["kernels"]], "rows_per_rank": sp.r1 - sp.r0,
            "collectives_per_step": sum(len(c) for c in sp.collective_after)}


def run_fused_child(args, rank, world, steps):
    """Every rank starts `bench.py --workload bicgk-sharded --collective fused`
    with its own RANK / WORLD_SIZE on another rendezvous port; rank 0 returns
    the child's JSON summary (or the error)."""
    import torch
    env = dict(os.environ)
    env["MASTER_PORT"] = str(int(env.get("MASTER_PORT", "29500")) + 17)
    cmd = [sys.executable, os.path.abspath(__file__), "--workload", "bicgk-sharded",
           "--collective", "fused", "--steps", str(steps), "--warmup", "3", "--gpus", str(world)]
    torch.distributed.barrier()
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=150)
        out = r.stdout.strip().splitlines()
        if rank != 0:
            return None
        if r.returncode != 0 or not out:
            return {"error": ("rc=%d " % r.returncode) + (r.stderr or "")[-300:]}
        d = json.loads(out[-1])
        return {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"],
                "frac_per_gpu": d["roofline"]["frac"], "workload": d["config"]["workload"]}
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
                    help="skip the BiCGK 131072^2 row-sharded leg of the default workload")
    ap.add_argument("--no-fused-child", action="store_true",
                    help="N > 1: skip the in-kernel (NVLink peer memory) variant of the sharded leg")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--workload", default="blas1", choices=["blas1", "bicgk-sharded", "atax-sharded"])
    ap.add_argument("--n-matrix", type=int, default=131072)
    ap.add_argument("--mode", default="fused", choices=["fused", "b200"],
                    help="planner mode of the sharded workloads (b200: row-resident ATAX)")
    ap.add_argument("--collective", default="fused", choices=["fused", "nccl"],
                    help="sharded workloads: in-kernel peer-memory reduction or NCCL all-reduce")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, local, world = env_rank()
    config = {"workload": WORKLOAD, "n": args.n, "dtype": "fp32", "parallelism": "dp%d" % world,
              "global_elements": args.n * world, "l2": "inputs (7 GiB/step) >> 126 MB L2; no flush",
              "data": "synthetic, device-side counter-based U(-1,1) generator"}

    if args.impl == "reference":
        if rank != 0:
            return
        threads = os.cpu_count() or 1
        sample = 1 << 24
        r = cpu_reference(sample, threads, args.steps, args.warmup)
        line = {"impl": "reference", "metric": METRIC, "value": round(r["value"], 3),
                "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(r["sec_per_step"] * 1e3, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config,
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

    if args.workload != "blas1":
        seq = "BICGK" if args.workload.startswith("bicgk") else "ATAX"
        r = run_sharded(args, torch, mf, rank, world, seq)
        peak, peak_kind = measured_peak()
        if rank == 0:
            line = {"metric": METRIC, "value": round(r["value"], 1), "unit": "GB/s", "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": round(r["ms_per_step"], 4), "higher_is_better": True,
                    "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                    "config": {"workload": "%s fp32 %dx%d row-sharded over %d GPU(s), column partials "
                                           "reduced %s" % (seq, args.n_matrix, args.n_matrix, world,
                                                           "in-kernel over NVLink peer memory"
                                                           if args.collective == "fused" else
                                                           "by NCCL all-reduce"),
                               "rows_per_rank": r["rows_per_rank"], "kernels": r["kernels"],
                               "collectives_per_step": r["collectives_per_step"],
                               "l2": "inputs (64 GiB) >> L2; no flush"},
                    "roofline": {"bound": "hbm", "achieved": round(r["value"] / world, 1), "peak": peak,
                                 "unit": "GB/s", "frac": round(r["value"] / world / peak, 4),
                                 "traffic": None, "peak_source": peak_kind + " (per GPU)"},
                    "clocks": r["clocks"], "gpu_launches": r["launches"]}
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
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "frac_of_nominal_8000": round(achieved / 8000.0, 4),
                "traffic": ncu_traffic("stream_kernel<3, 1, 0,"),
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
            "bytes_saved_ratio": round((24 + 20) / 28, 3)}
    e2e = run_e2e(args, torch, mf, args.e2e_steps, world)
    torch.cuda.empty_cache()
    sharded = None
    if not args.no_sharded:
        # BASELINE configs[4]: BiCGK 131072^2 row-sharded over the N ranks
        # (strong scaling; T(1) at N = 1), column partials all-reduced by NCCL
        import copy
        sa = copy.copy(args)
        sa.collective, sa.mode = "nccl", "fused"  # n_matrix: 131072 unless --n-matrix
        sa.steps, sa.warmup = max(5, min(args.steps, 20)), 3
        try:
            r = run_sharded(sa, torch, mf, rank, world, "BICGK")
            peak, _ = measured_peak()
            sharded = {"workload": "BiCGK fp32 131072x131072 row-sharded over %d GPU(s), column "
                                   "partials all-reduced by NCCL after the fused kernel" % world,
                       "value": round(r["value"], 1), "unit": "GB/s", "ms_per_step": round(r["ms_per_step"], 4),
                       "steps": sa.steps, "scaling": "strong", "rows_per_rank": r["rows_per_rank"],
                       "frac_per_gpu": round(r["value"] / world / peak, 4),
                       "collectives_per_step": r["collectives_per_step"]}
        except Exception as ex:  # report, keep the main line
            sharded = {"error": str(ex)[:300]}
        torch.cuda.empty_cache()
        if world > 1 and not args.no_fused_child and not SHARED_GPU:
            # the same leg with the column reduction fused into the kernel over
            # NVLink peer memory (CUDA IPC, no NCCL on the data path) -- in
            # child processes with their own rendezvous, so a failure there
            # cannot take this line down
            fused = run_fused_child(args, rank, world, sa.steps)
            if sharded is not None and fused is not None:
                sharded["fused_collective"] = fused
    if rank == 0:
        line["e2e"] = e2e
        if sharded is not None:
            line["sharded"] = sharded
        if world == 1 and not args.no_suite:
            line["suite"] = run_suite(args, torch, mf)
        if world == 1 and not args.no_cpu:
            try:
                line["cpu_baseline"] = {k: v for k, v in cpu_reference(
                    1 << 24, os.cpu_count() or 1, 3, 1).items() if k in
                    ("value", "unit", "cores", "kind", "sample")}
            except Exception as e:  # oracle/_ref absent: say so
                line["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": 0,
                                        "kind": "reference", "sample": "unavailable: %s" % e}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
