"""Two OS processes, one GPU: the REAL multi-process path of the fused
compute + collective (CUDA-IPC handle export, exchange over the process
group, cudaIpcOpenMemHandle, system-scope peer barriers, in-kernel column
reduction) -- the path one-process-per-GPU ranks take on an 8-GPU box.
Virtual ranks in one process (tests/test_gpu_fused_collective.py) cannot
exercise the IPC calls; this can.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 tools/ipc_two_process.py [--seq BICGK --rows 2048 --cols 4096]

Both ranks use cuda:0 (their contexts time-slice the GPU; the kernels'
peer barriers wait across slices).  The exchange uses gloo.  Rank 0 checks
the gathered result against the CPU oracle and prints "ipc ok".
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", default="BICGK")
    ap.add_argument("--rows", type=int, default=2048)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--collective", default="fused")
    a = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    import paper_1305_1183_b200 as mf
    from paper_1305_1183_b200.sharding import ShardedPlan
    from oracle import COracle
    sp = ShardedPlan(a.seq, a.rows, a.cols, "fused", collective=a.collective)
    if a.collective == "fused":
        assert sp.peers is not None, "peer group not connected"
    gd = sp.global_desc
    rng = np.random.default_rng(5)
    vals = {}
    for b in gd["buffers"]:
        if b["role"] == "input":
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            vals[b["name"]] = rng.uniform(-1, 1, shp).astype(np.float32)
    sc = {s: 0.5 + 0.25 * i for i, s in enumerate(gd["scalars"])}
    bufs = {}
    for b in sp.desc["buffers"]:
        sl = sp.local_slice(b["name"])
        if b["name"] in vals:
            v = vals[b["name"]]
            if sl is not None:
                v = v[sl[1]:sl[2]] if sl[0] == 0 or v.ndim == 1 else v[:, sl[1]:sl[2]]
            bufs[b["name"]] = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        else:
            bufs[b["name"]] = torch.full(sp.local_shape(b["name"]), float("nan"), device="cuda")
    for rep in range(3):  # repeated launches: epochs of the peer barriers advance
        st = sp.launch(bufs, sc)
        torch.cuda.synchronize()
    outs = {}
    for b in gd["buffers"]:
        if b["role"] != "output":
            continue
        t = bufs[b["name"]].cpu()
        parts = [None] * world
        dist.all_gather_object(parts, (sp.local_slice(b["name"]), t.numpy()))
        outs[b["name"]] = parts
    if rank == 0:
        from gpu_util import scale_bound  # |.|-formula bound (signs handled per sequence)
        co = COracle()
        want = co.execute(a.seq, a.rows, a.cols, {**vals, **sc})
        S = scale_bound(co, a.seq, a.rows, a.cols, {**vals, **sc})
        for name, parts in outs.items():
            sl0 = parts[0][0]
            if sl0 is None:  # replicated (column reduction): every rank holds all of it
                for _, p in parts:
                    got = p.ravel()
                    err = np.abs(got.astype(np.float64) - want[name].ravel())
                    lim = 2.0 ** -17 * S[name].ravel() + np.spacing(np.abs(want[name].ravel()))
                    assert np.all(err <= lim), (name, float(np.max(err / lim)))
                assert all(np.array_equal(parts[0][1], p) for _, p in parts), name
            else:
                got = np.concatenate([p for _, p in parts], axis=0 if parts[0][1].ndim == 2 else 0)
                err = np.abs(got.ravel().astype(np.float64) - want[name].ravel())
                lim = 2.0 ** -17 * S[name].ravel() + np.spacing(np.abs(want[name].ravel()))
                assert np.all(err <= lim), (name, float(np.max(err / lim)))
        print("ipc ok", a.seq, a.rows, a.cols, st, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
