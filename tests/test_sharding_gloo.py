"""Multi-rank host logic on CPU: world_size 2 (and 3) gloo process groups.

Each rank holds only its shard (row panel of every tile, its slice of
row-indexed vectors, full copies of column-indexed vectors), runs the plan's
kernels (CPU emulator standing in for the sm_100a kernels), and the
ShardedPlan inserts exactly the all-reduces the plan reports.  Gathered
results must match the pinned CPU oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_util import all_goldens
from gpu_util import check_output, scale_bound


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seq, m, n, seed, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from plan_emulator import run_kernel
    from paper_1305_1183_b200.sharding import ShardedPlan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = ShardedPlan(seq, m, n, "fused", executor=run_kernel)
        rng = np.random.default_rng(seed)
        gd = sp.global_desc
        full = {}
        for b in gd["buffers"]:
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            full[b["name"]] = (rng.uniform(-1, 1, shp).astype(np.float32) if b["role"] == "input"
                               else np.zeros(shp, np.float32))
        scalars = {s: float(np.float32(0.25 + 0.5 * rng.random())) for s in gd["scalars"]}
        local = {}
        for name, a in full.items():
            sl = sp.local_slice(name)
            if sl is None:
                local[name] = torch.from_numpy(a.copy())
            elif sl[0] == 0:
                local[name] = torch.from_numpy(a[sl[1]:sl[2]].copy())
            else:
                local[name] = torch.from_numpy(a.reshape(-1)[sl[1]:sl[2]].copy())
        info = sp.launch(local, scalars)
        # gather outputs on rank 0
        outs = {}
        for b in gd["buffers"]:
            if b["role"] != "output":
                continue
            t = local[b["name"]]
            sl = sp.local_slice(b["name"])
            if sl is None:
                outs[b["name"]] = t.numpy()
                continue
            lens = [None] * world
            dist.all_gather_object(lens, (sl, t.numpy()))
            if sl[0] == 0:
                outs[b["name"]] = np.concatenate([x[1] for x in lens], axis=0)
            else:
                outs[b["name"]] = np.concatenate([x[1].reshape(-1) for x in lens])
        if rank == 0:
            inputs = {k: v for k, v in full.items()}
            inputs.update(scalars)
            q.put((outs, inputs, info))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seq,m,n,world", [
    ("BICGK", 256, 192, 2), ("ATAX", 192, 256, 2), ("GEMVER", 256, 160, 2), ("GESUMMV", 128, 96, 2),
    ("SGEMVT", 160, 160, 2), ("AXPYDOT", 1, 4096, 2), ("VADD", 1, 4096, 2), ("BICGK", 320, 96, 3),
])
def test_row_sharded_plan_matches_oracle(seq, m, n, world):
    from oracle import COracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seq, m, n, 99, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs, inputs, info = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    co = COracle()
    mp_, np_ = (m + 31) // 32 * 32, (n + 31) // 32 * 32
    want = co.execute(seq, mp_, np_, inputs)
    S = scale_bound(co, seq, mp_, np_, inputs)
    for name, w in want.items():
        check_output(seq, name, outs[name], w, S[name], exact=False)
    expected_collectives = {"BICGK": 1, "ATAX": 1, "GEMVER": 1, "GESUMMV": 0, "SGEMVT": 1,
                            "AXPYDOT": 1, "VADD": 0}[seq]
    assert info["collectives"] == expected_collectives


def test_split_covers_exactly():
    from paper_1305_1183_b200.sharding import split
    for total in (32, 96, 131072, 4096 + 32):
        for parts in (1, 2, 3, 4, 8):
            blocks = [split(total, parts, r) for r in range(parts)]
            assert blocks[0][0] == 0 and blocks[-1][1] == total
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c and a <= b
            assert all(b % 32 == 0 or b == total for _, b in blocks)


def _worker_script(rank, world, port, text, m, n, seed, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from plan_emulator import run_kernel
    from paper_1305_1183_b200.sharding import ShardedPlan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = ShardedPlan(script=text, rows=m, cols=n, mode="fused", executor=run_kernel)
        rng = np.random.default_rng(seed)
        gd = sp.global_desc
        full = {}
        for b in gd["buffers"]:
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            full[b["name"]] = (rng.uniform(-1, 1, shp).astype(np.float32) if b["role"] == "input"
                               else np.zeros(shp, np.float32))
        local = {}
        for name, a in full.items():
            sl = sp.local_slice(name)
            local[name] = torch.from_numpy((a if sl is None else a[sl[1]:sl[2]]).copy())
        for b in sp.desc["buffers"]:  # intermediates the local plan adds
            if b["name"] not in local:
                shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
                local[b["name"]] = torch.zeros(shp)
        sp.launch(local, {"k": 0.625})
        outs = {}
        for b in gd["buffers"]:
            if b["role"] != "output":
                continue
            sl = sp.local_slice(b["name"])
            parts = [None] * world
            dist.all_gather_object(parts, local[b["name"]].numpy())
            outs[b["name"]] = parts[0] if sl is None else np.concatenate(parts, axis=0)
            if sl is None:  # replicated: every rank holds the same value
                assert all(np.array_equal(parts[0], p) for p in parts), b["name"]
        if rank == 0:
            q.put((outs, {k: v for k, v in full.items() if gd and k in
                          {x["name"] for x in gd["buffers"] if x["role"] == "input"}},
                   [k["calls"] for k in sp.desc["kernels"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("seed", range(int(os.environ.get("MF_GLOO_RANDOM_SEEDS", "3"))))
def test_random_scripts_row_sharded_gloo(seed, world):
    """Random planner outputs sharded over real gloo process groups: every
    rank must pick the same kernel partition, the layer must all-reduce
    exactly the rank partials (no dot over replicated vectors), and the
    gathered outputs must match the per-call fp64 oracle chain."""
    import paper_1305_1183_b200 as mf
    from oracle import COracle
    from test_gpu_random_scripts import abs_chain, make_script, reference_chain
    from gpu_util import TAU
    rng = np.random.default_rng(50000 + seed)
    text, calls, returns = make_script(rng, 3 + seed % 5)
    m, n = 192 + 32 * (seed % 3), 128 + 64 * (seed % 4)
    if any(k["kind"] == "generic" for k in mf.Plan.compile(text, m, n, "fused").describe()["kernels"]):
        pytest.skip("the CPU kernel emulator covers the hand-written families only")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_script, args=(r, world, port, text, m, n, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs, inputs, _ = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    co = COracle()
    env = dict(inputs)
    env["k"] = 0.625
    want = reference_chain(co, calls, dict(env), m, n)
    S = abs_chain(co, calls, dict(env), m, n)
    for name in returns:
        got = np.asarray(outs[name], np.float64).ravel()
        w = np.asarray(want[name], np.float64).ravel()
        s = np.asarray(S[name], np.float64).ravel()
        lim = 4 * TAU * s + 4 * np.spacing(np.abs(w).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(got - w) <= lim), (text, name)


def _worker_scatter(rank, world, port, seq, m, n, seed, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    from plan_emulator import run_kernel
    from paper_1305_1183_b200.sharding import ShardedPlan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = ShardedPlan(seq, m, n, "fused", executor=run_kernel, outputs="sharded")
        rng = np.random.default_rng(seed)
        gd = sp.global_desc
        full = {}
        for b in gd["buffers"]:
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            full[b["name"]] = (rng.uniform(-1, 1, shp).astype(np.float32) if b["role"] == "input"
                               else np.zeros(shp, np.float32))
        scalars = {s: float(np.float32(0.25 + 0.5 * rng.random())) for s in gd["scalars"]}
        local = {}
        for name, a in full.items():
            sl = sp.local_slice(name)
            local[name] = torch.from_numpy((a if sl is None else a[sl[1]:sl[2]]).copy())
        info = sp.launch(local, scalars)
        outs = {}
        for b in gd["buffers"]:
            if b["role"] != "output":
                continue
            name = b["name"]
            sl, cs = sp.local_slice(name), sp.column_slice(name)
            part = local[name].numpy()
            if cs is not None:  # only this rank's column slice is finished
                part = part[cs[0]:cs[1]]
            parts = [None] * world
            dist.all_gather_object(parts, part)
            outs[name] = parts[0] if (sl is None and cs is None) else np.concatenate(parts, axis=0)
        if rank == 0:
            inputs = dict(full)
            inputs.update(scalars)
            q.put((outs, inputs, info, [list(x) for x in sp.scatter_after]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seq,m,n,world,scattered", [
    ("ATAX", 192, 256, 2, ["y"]), ("BICGK", 256, 192, 2, ["s"]), ("SGEMVT", 160, 192, 2, []),
    ("GEMVER", 256, 160, 2, []), ("BICGK", 320, 96, 3, ["s"]), ("ATAX", 96, 160, 3, []),
])
def test_reduce_scatter_for_sharded_consumers(seq, m, n, world, scattered):
    """outputs="sharded": column outputs no later kernel reads are
    reduce-scattered (rank r finishes slice r of n), intermediates a later
    kernel reads (GEMVER's t) stay all-reduced, and so does an output whose
    length is not a multiple of the rank count (ATAX n = 160 over 3 ranks).
    The gathered slices match the oracle."""
    from oracle import COracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_scatter, args=(r, world, port, seq, m, n, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs, inputs, info, scatter_after = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(x for names in scatter_after for x in names) == scattered
    assert info["reduce_scatters"] == len(scattered)
    co = COracle()
    mp_, np_ = (m + 31) // 32 * 32, (n + 31) // 32 * 32
    want = co.execute(seq, mp_, np_, inputs)
    S = scale_bound(co, seq, mp_, np_, inputs)
    for name, w in want.items():
        check_output(seq, name, outs[name], w, S[name], exact=False)
