"""GPU: the in-kernel cross-rank column reduction (fused compute + collective).

This run has one GPU, so P "virtual ranks" share it: each rank is its own
plan (own workspace, own grid barrier) whose cooperative grid is sized for
148/P SMs, launched on its own stream so all ranks' kernels are co-resident;
peer pointers are the other ranks' group buffers (same code path as CUDA-IPC
mapped NVLink peers).  Every rank must end with the same, correct column
vector; row outputs stay local.
"""
import numpy as np
import pytest

from gpu_util import TAU
from oracle import COracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seq,m,n,P", [("BICGK", 2048, 4096, 2), ("BICGK", 4096, 2048, 4),
                                       ("ATAX", 1024, 3072, 2), ("GEMVER", 1024, 2048, 2),
                                       # full-width panels: every column chunk and a multi-band grid per rank
                                       ("BICGK", 32768, 16384, 4), ("GEMVER", 8192, 8192, 2),
                                       ("ATAX", 16384, 8192, 2)])
@pytest.mark.parametrize("tma", [0, 1])
def test_virtual_ranks_fused_column_reduction(seq, m, n, P, tma):
    import torch
    import paper_1305_1183_b200 as mf
    co = COracle()
    mf.set_option("max_sms", 148 // P)
    mf.set_option("tma", tma)
    try:
        rng = np.random.default_rng(m + n + P)
        full_plan = mf.Plan.sequence(seq, m, n, "fused")
        gd = full_plan.describe()
        vals = {}
        for b in gd["buffers"]:
            if b["role"] == "input":
                shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
                vals[b["name"]] = rng.uniform(-1, 1, shp).astype(np.float32)
        sc = {s: 0.5 + 0.25 * i for i, s in enumerate(gd["scalars"])}
        rows_of = {b["name"]: b for b in gd["buffers"]}
        mloc = m // P
        plans = [mf.Plan.sequence(seq, mloc, n, "fused") for _ in range(P)]
        groups = [mf.PeerGroup(P, r, n) for r in range(P)]
        for r in range(P):
            for q in range(P):
                if q != r:
                    groups[r].connect_local(q, groups[q])
        streams = [torch.cuda.Stream() for _ in range(P)]
        bufs = []
        for r in range(P):
            d = {}
            for b in plans[r].describe()["buffers"]:
                g = rows_of[b["name"]]
                shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
                if b["name"] in vals:
                    v = vals[b["name"]]
                    if g["rows"] > 1:
                        v = v[r * mloc:(r + 1) * mloc]
                    elif g["row_indexed"]:
                        v = v[r * mloc:(r + 1) * mloc]
                    d[b["name"]] = torch.from_numpy(np.ascontiguousarray(v)).cuda()
                else:
                    d[b["name"]] = torch.full(shp, float("nan"), device="cuda")
            bufs.append(d)
        # size every rank's workspace (one per stream) first: allocation can
        # synchronize the whole device -- with virtual ranks sharing one GPU
        # that would serialize ranks that must be co-resident
        for r in range(P):
            plans[r].launch(bufs[r], sc, stream=streams[r])
        torch.cuda.synchronize()
        for k in range(plans[0].num_kernels):
            kind = plans[0].describe()["kernels"][k]["kind"]
            for r in range(P):
                with torch.cuda.stream(streams[r]):
                    if kind == "matrix":
                        plans[r].launch_kernel_peers(k, groups[r], bufs[r], sc, streams[r])
                    else:
                        plans[r].launch_kernel(k, bufs[r], sc, streams[r])
            torch.cuda.synchronize()
        want = co.execute(seq, m, n, {**vals, **sc})
        absvals = {k: (np.abs(v) if isinstance(v, np.ndarray) else v) for k, v in vals.items()}
        S = co.execute(seq, m, n, {**absvals, **{k: abs(v) for k, v in sc.items()}})
        for name, w in want.items():
            g = rows_of[name]
            if g["rows"] > 1 or g["row_indexed"]:
                got = np.concatenate([bufs[r][name].cpu().numpy() for r in range(P)], axis=0)
            else:
                got = bufs[0][name].cpu().numpy()
                for r in range(1, P):  # replicated outputs: identical on every rank
                    assert np.array_equal(got, bufs[r][name].cpu().numpy()), name
            err = np.abs(got.astype(np.float64).ravel() - w.astype(np.float64).ravel())
            lim = TAU * S[name].astype(np.float64).ravel() + np.spacing(np.abs(w.ravel()))
            assert np.all(err <= lim), (name, float(np.max(err / lim)))
    finally:
        mf.set_option("max_sms", 0)
        mf.set_option("tma", -1)


@pytest.mark.parametrize("n", [8192, 32768])
def test_virtual_ranks_row_resident_chain(n):
    """Row-resident ATAX kernel (n = 32768: rows over a CTA cluster) +
    in-kernel cross-rank column reduction."""
    import torch
    import paper_1305_1183_b200 as mf
    co = COracle()
    P, m = 2, 2048
    mf.set_option("max_sms", 148 // P)
    try:
        rng = np.random.default_rng(5)
        A = rng.uniform(-1, 1, (m, n)).astype(np.float32)
        x = rng.uniform(-1, 1, n).astype(np.float32)
        mloc = m // P
        plans = [mf.Plan.sequence("ATAX", mloc, n, "b200") for _ in range(P)]
        assert plans[0].describe()["kernels"][0]["shape"]["chain"] == 1
        groups = [mf.PeerGroup(P, r, n) for r in range(P)]
        for r in range(P):
            for q in range(P):
                if q != r:
                    groups[r].connect_local(q, groups[q])
        bufs = [{"A": torch.from_numpy(A[r * mloc:(r + 1) * mloc].copy()).cuda(),
                 "x": torch.from_numpy(x).cuda(), "y": torch.zeros(n, device="cuda")}
                for r in range(P)]
        streams = [torch.cuda.Stream() for _ in range(P)]
        for r in range(P):  # size each stream's workspace first
            plans[r].launch(bufs[r], stream=streams[r])
        torch.cuda.synchronize()
        for r in range(P):
            plans[r].launch_kernel_peers(0, groups[r], bufs[r], {}, streams[r])
        torch.cuda.synchronize()
        want = co.execute("ATAX", m, n, {"A": A, "x": x})["y"]
        S = co.execute("ATAX", m, n, {"A": np.abs(A), "x": np.abs(x)})["y"]
        for r in range(P):
            got = bufs[r]["y"].cpu().numpy().astype(np.float64)
            assert np.all(np.abs(got - want) <= TAU * S + np.spacing(np.abs(want)))
        assert np.array_equal(bufs[0]["y"].cpu().numpy(), bufs[1]["y"].cpu().numpy())
    finally:
        mf.set_option("max_sms", 0)


@pytest.mark.parametrize("seq,m,n", [("BICGK", 2048, 4096), ("GEMVER", 1024, 2048),
                                     ("ATAX", 1536, 1024), ("AXPYDOT", 1, 1 << 20)])
def test_two_processes_ipc_fused_column_reduction(seq, m, n):
    """The real one-process-per-rank path: two OS processes (both on cuda:0),
    CUDA-IPC handles exchanged over gloo, in-kernel reduction across them
    (tools/ipc_two_process.py checks against the oracle)."""
    import os
    import random
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = str(29500 + random.randint(100, 900))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", port,
                        os.path.join(root, "tools", "ipc_two_process.py"), "--seq", seq,
                        "--rows", str(m), "--cols", str(n)],
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "ipc ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("P", [2, 4])
def test_virtual_ranks_fused_dot(P):
    """AXPYDOT element-sharded over P virtual ranks: each rank's stream kernel
    finishes the dot across ranks in-kernel (fp64 partials over peer memory,
    fixed rank order) -- every rank ends with the same r, within tolerance of
    the oracle; z stays local."""
    import torch
    import paper_1305_1183_b200 as mf
    co = COracle()
    n = 1 << 20
    rng = np.random.default_rng(P)
    w, v, u = (rng.uniform(-1, 1, n).astype(np.float32) for _ in range(3))
    alpha = 0.375
    nloc = n // P
    plans = [mf.Plan.sequence("AXPYDOT", 1, nloc, "fused") for _ in range(P)]
    groups = [mf.PeerGroup(P, r, nloc) for r in range(P)]
    for r in range(P):
        for q in range(P):
            if q != r:
                groups[r].connect_local(q, groups[q])
    streams = [torch.cuda.Stream() for _ in range(P)]
    bufs = []
    for r in range(P):
        sl = slice(r * nloc, (r + 1) * nloc)
        bufs.append({"w": torch.from_numpy(w[sl].copy()).cuda(), "v": torch.from_numpy(v[sl].copy()).cuda(),
                     "u": torch.from_numpy(u[sl].copy()).cuda(),
                     "z": torch.empty(nloc, device="cuda"), "r": torch.full((1,), float("nan"), device="cuda")})
    for r in range(P):  # size each stream's workspace first (allocation can sync the device)
        plans[r].launch(bufs[r], {"alpha": alpha}, stream=streams[r])
    torch.cuda.synchronize()
    for rep in range(3):
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                plans[r].launch_kernel_peers(0, groups[r], bufs[r], {"alpha": alpha}, streams[r])
        torch.cuda.synchronize()
    want = co.execute("AXPYDOT", 1, n, {"w": w, "v": v, "u": u, "alpha": alpha})
    S = co.execute("AXPYDOT", 1, n, {"w": np.abs(w), "v": np.abs(v), "u": np.abs(u), "alpha": -alpha})
    rs = [float(bufs[r]["r"].cpu()[0]) for r in range(P)]
    assert all(x == rs[0] for x in rs), rs  # identical on every rank
    assert abs(rs[0] - float(want["r"][0])) <= TAU * float(S["r"][0]) + abs(float(want["r"][0])) * 2 ** -23
    z = np.concatenate([bufs[r]["z"].cpu().numpy() for r in range(P)])
    assert np.array_equal(z, want["z"])


@pytest.mark.parametrize("seq", ["GEMVER", "BICGK", "AXPYDOT"])
def test_virtual_ranks_launch_peers_whole_plan(seq):
    """mf_launch_peers: a whole plan per rank with every cross-rank reduction
    in-kernel (C-ABI sharded launch, no NCCL), two virtual ranks on one GPU."""
    import torch
    import paper_1305_1183_b200 as mf
    from paper_1305_1183_b200.sharding import split
    co = COracle()
    P = 2
    m, n = (1, 1 << 18) if seq == "AXPYDOT" else (2048, 2048)
    mf.set_option("max_sms", 148 // P)
    try:
        rng = np.random.default_rng(11)
        full = mf.Plan.sequence(seq, m, n, "fused")
        gd = full.describe()
        vals = {}
        for b in gd["buffers"]:
            if b["role"] == "input":
                shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
                vals[b["name"]] = rng.uniform(-1, 1, shp).astype(np.float32)
        sc = {s: 0.5 + 0.25 * i for i, s in enumerate(gd["scalars"])}
        spec = {b["name"]: b for b in gd["buffers"]}
        depth1 = seq == "AXPYDOT"
        parts = [split(n if depth1 else m, P, r) for r in range(P)]
        plans = [mf.Plan.sequence(seq, 1 if depth1 else hi - lo, hi - lo if depth1 else n, "fused")
                 for lo, hi in parts]
        groups = [mf.PeerGroup(P, r, n) for r in range(P)]
        for r in range(P):
            for q in range(P):
                if q != r:
                    groups[r].connect_local(q, groups[q])
        bufs = []
        for r, (lo, hi) in enumerate(parts):
            d = {}
            for b in plans[r].describe()["buffers"]:
                shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
                g = spec[b["name"]]
                if b["name"] in vals:
                    v = vals[b["name"]]
                    if depth1 or g["rows"] > 1 or g["row_indexed"]:
                        v = v[lo:hi]
                    d[b["name"]] = torch.from_numpy(np.ascontiguousarray(v)).cuda()
                else:
                    d[b["name"]] = torch.full(shp, float("nan"), device="cuda")
            bufs.append(d)
        streams = [torch.cuda.Stream() for _ in range(P)]
        for r in range(P):  # size each stream's workspace (allocation can sync the device)
            plans[r].launch(bufs[r], sc, stream=streams[r])
        torch.cuda.synchronize()
        for r in range(P):
            plans[r].launch_peers(groups[r], bufs[r], sc, streams[r])
        torch.cuda.synchronize()
        want = co.execute(seq, m, n, {**vals, **sc})
        from gpu_util import scale_bound
        S = scale_bound(co, seq, m, n, {**vals, **sc})
        for name in want:
            g = spec[name]
            sharded = depth1 and not g["scalar"] or (not depth1 and (g["rows"] > 1 or g["row_indexed"]))
            if sharded:
                got = np.concatenate([bufs[r][name].cpu().numpy() for r in range(P)], axis=0)
            else:
                got = bufs[0][name].cpu().numpy()
                assert all(np.array_equal(got, bufs[r][name].cpu().numpy()) for r in range(P)), name
            w, s = np.asarray(want[name]).ravel(), np.asarray(S[name]).ravel()
            err = np.abs(got.ravel().astype(np.float64) - w)
            assert np.all(err <= TAU * s + np.spacing(np.abs(w).astype(np.float32))), name
    finally:
        mf.set_option("max_sms", 0)


_TIMEOUT_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1305_1183_b200 as mf
P, n = 2, 1 << 16
plan = mf.Plan.sequence("AXPYDOT", 1, n, "fused")
groups = [mf.PeerGroup(P, r, n) for r in range(P)]
groups[0].connect_local(1, groups[1]); groups[1].connect_local(0, groups[0])
b = {k: torch.rand(n, device="cuda") for k in ("w", "v", "u")}
b.update(z=torch.empty(n, device="cuda"), r=torch.empty(1, device="cuda"))
plan.launch(b, {"alpha": 0.5})           # size the workspace
torch.cuda.synchronize()
plan.launch_kernel_peers(0, groups[0], b, {"alpha": 0.5})   # rank 1 never launches
try:
    groups[0].check()
    print("NO-ERROR")
except mf.VmFault as e:
    print("FAULT:", e)
plan.launch(b, {"alpha": 0.5})           # the context is still usable
torch.cuda.synchronize()
print("USABLE")
"""


def test_peer_barrier_times_out_with_clear_error():
    """A rank whose peer never arrives gives up after MF_PEER_TIMEOUT_MS,
    flags the group and finishes; mf_peer_group_check reports it and the
    CUDA context stays usable (no trap, no hung GPU)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MF_PEER_TIMEOUT_MS="300")
    r = subprocess.run([sys.executable, "-c", _TIMEOUT_CHILD, root], env=env, capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "FAULT:" in r.stdout and "timed out" in r.stdout, r.stdout
    assert "USABLE" in r.stdout
