"""GPU: random scripts through the row-sharding layer (sharding.ShardedPlan)
on virtual ranks sharing one B200.

Every rank gets its row panel of the global problem (ShardedPlan.local_slice)
and its own plan; kernel k runs on every rank, then the names the layer
reduces after kernel k (collective_after) are summed over the ranks -- what
the NCCL all-reduce does on a real multi-GPU run.  The gathered outputs must
match the per-call fp64 oracle chain of the unsharded problem (tau*S bound),
and replicated outputs must be identical on every rank.
"""
import os

import numpy as np
import pytest

from gpu_util import TAU
from oracle import COracle
from test_gpu_random_scripts import abs_chain, make_script, reference_chain

pytestmark = pytest.mark.gpu
SEEDS = range(int(os.environ.get("MF_RANDOM_SHARDED_SEEDS", "24")))


@pytest.mark.parametrize("mode", ["fused", "b200"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("seed", SEEDS)
def test_random_script_row_sharded(seed, P, mode):
    import torch
    import paper_1305_1183_b200 as mf
    from paper_1305_1183_b200.sharding import ShardedPlan
    co = COracle()
    rng = np.random.default_rng(1000 + seed)
    text, calls, returns = make_script(rng, 3 + seed % 5)
    m, n = 192 + 32 * (seed % 3), 128 + 64 * (seed % 4)
    sps = [ShardedPlan(script=text, rows=m, cols=n, mode=mode, world=P, rank=r, collective="nccl")
           for r in range(P)]
    gd = sps[0].global_desc
    env = {"k": 0.625}
    for b in gd["buffers"]:
        if b["role"] == "input":
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            env[b["name"]] = rng.uniform(-1, 1, shp).astype(np.float32)
    bufs = []
    for sp in sps:
        d = {}
        for b in sp.desc["buffers"]:
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            v = env.get(b["name"])
            if isinstance(v, np.ndarray):
                sl = sp.local_slice(b["name"])
                if sl is not None:
                    v = v[sl[1]:sl[2]] if sl[0] == 0 or v.ndim == 1 else v[:, sl[1]:sl[2]]
                d[b["name"]] = torch.from_numpy(np.ascontiguousarray(v)).cuda()
            else:
                d[b["name"]] = torch.full(shp, float("nan"), device="cuda")
        bufs.append(d)
    for k in range(sps[0].plan.num_kernels):
        for r, sp in enumerate(sps):
            sp.plan.launch_kernel(k, bufs[r], {"k": env["k"]})
        torch.cuda.synchronize()
        for name in sps[0].collective_after[k]:  # the all-reduce
            total = sum(bufs[r][name] for r in range(P))
            for r in range(P):
                bufs[r][name].copy_(total)
    torch.cuda.synchronize()
    want = reference_chain(co, calls, dict(env), m, n)
    S = abs_chain(co, calls, dict(env), m, n)
    for name in returns:
        sl = sps[0].local_slice(name)
        if sl is None:
            got = bufs[0][name].cpu().numpy()
            # hand-written kernels are deterministic: replicas are bit-identical;
            # generic kernels accumulate with float atomics (the paper's
            # semantics), so their replicas only agree within the bound below
            kind = next(k["kind"] for k in sps[0].desc["kernels"] if name in k["outputs"])
            for r in range(1, P):
                if kind != "generic":
                    assert np.array_equal(bufs[r][name].cpu().numpy(), got), (text, name, "ranks differ")
        else:
            parts = [bufs[r][name].cpu().numpy() for r in range(P)]
            got = np.concatenate(parts, axis=0)
        got = got.astype(np.float64).ravel()
        w = np.asarray(want[name], np.float64).ravel()
        s = np.asarray(S[name], np.float64).ravel()
        lim = 4 * TAU * s + 4 * np.spacing(np.abs(w).astype(np.float32)).astype(np.float64)
        err = np.abs(got - w)
        assert np.all(err <= lim), (text, name, float(np.max(err / np.maximum(lim, 1e-300))))


@pytest.mark.parametrize("mode", ["fused", "b200"])
@pytest.mark.parametrize("seed", SEEDS)
def test_random_script_peers_in_kernel(seed, mode):
    """The same random scripts through mf_launch_peers: two virtual ranks on
    their own streams, every cross-rank sum done inside the kernels over the
    peer buffers (the CUDA-IPC / NVLink code path).  Plans whose generic
    kernels leave rank partials need a host collective and are skipped."""
    import torch
    import paper_1305_1183_b200 as mf
    from paper_1305_1183_b200.sharding import ShardedPlan
    co = COracle()
    P = 2
    rng = np.random.default_rng(5000 + seed)
    text, calls, returns = make_script(rng, 3 + seed % 5)
    m, n = 192 + 64 * (seed % 3), 128 + 64 * (seed % 4)
    sps = [ShardedPlan(script=text, rows=m, cols=n, mode=mode, world=P, rank=r, collective="nccl")
           for r in range(P)]
    for k, kd in enumerate(sps[0].desc["kernels"]):
        if kd["kind"] == "generic" and sps[0].collective_after[k]:
            pytest.skip("generic kernel with rank partials: host collective only")
    gd = sps[0].global_desc
    env = {"k": 0.625}
    for b in gd["buffers"]:
        if b["role"] == "input":
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            env[b["name"]] = rng.uniform(-1, 1, shp).astype(np.float32)
    bufs = []
    for sp in sps:
        d = {}
        for b in sp.desc["buffers"]:
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            v = env.get(b["name"])
            if isinstance(v, np.ndarray):
                sl = sp.local_slice(b["name"])
                if sl is not None:
                    v = v[sl[1]:sl[2]]
                d[b["name"]] = torch.from_numpy(np.ascontiguousarray(v)).cuda()
            else:
                d[b["name"]] = torch.full(shp, float("nan"), device="cuda")
        bufs.append(d)
    mf.set_option("max_sms", 148 // P)
    try:
        groups = [mf.PeerGroup(P, r, max(m, n)) for r in range(P)]
        for r in range(P):
            for q in range(P):
                if q != r:
                    groups[r].connect_local(q, groups[q])
        streams = [torch.cuda.Stream() for _ in range(P)]
        for r in range(P):  # size each stream's workspace first (allocation can sync the device)
            sps[r].plan.launch(bufs[r], {"k": env["k"]}, stream=streams[r])
        torch.cuda.synchronize()
        for r in range(P):
            sps[r].plan.launch_peers(groups[r], bufs[r], {"k": env["k"]}, streams[r])
        torch.cuda.synchronize()
    finally:
        mf.set_option("max_sms", 0)
    want = reference_chain(co, calls, dict(env), m, n)
    S = abs_chain(co, calls, dict(env), m, n)
    for name in returns:
        sl = sps[0].local_slice(name)
        if sl is None:
            got = bufs[0][name].cpu().numpy()
            kind = next(k["kind"] for k in sps[0].desc["kernels"] if name in k["outputs"])
            if kind != "generic":
                assert np.array_equal(bufs[1][name].cpu().numpy(), got), (text, name, "ranks differ")
        else:
            got = np.concatenate([bufs[r][name].cpu().numpy() for r in range(P)], axis=0)
        got = got.astype(np.float64).ravel()
        w = np.asarray(want[name], np.float64).ravel()
        s = np.asarray(S[name], np.float64).ravel()
        lim = 4 * TAU * s + 4 * np.spacing(np.abs(w).astype(np.float32)).astype(np.float64)
        err = np.abs(got - w)
        assert np.all(err <= lim), (text, name, float(np.max(err / np.maximum(lim, 1e-300))))
