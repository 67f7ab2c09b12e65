"""CPU stand-in for the sm_100a kernels, driven by a plan's kernel
description (describe()["kernels"][k]["op"]).  TEST INFRASTRUCTURE: used only
to exercise the host-side sharding orchestration with the gloo backend where
no GPU exists.  fp64 arithmetic, fp32 storage, like the kernels."""
import torch


def coef(terms, scalars):
    s = 0.0
    for c, syms in terms:
        v = float(c)
        for n in syms:
            v *= float(scalars[n])
        s += v
    return s


def run_kernel(kern, bufs, scalars):
    op = kern["op"]
    f64 = lambda n: bufs[n].to(torch.float64)
    if kern["kind"] == "stream":
        ins = [f64(n).reshape(-1) for n in op["inputs"]]
        for o in op["outs"]:
            acc = None
            for x, c in zip(ins, o["coef"]):
                t = coef(c, scalars) * x
                acc = t if acc is None else acc + t
            bufs[o["name"]].copy_(acc.reshape(bufs[o["name"]].shape).to(torch.float32))
        if "dot" in op:
            d = op["dot"]
            a = sum(coef(c, scalars) * x for x, c in zip(ins, d["a"]))
            b = sum(coef(c, scalars) * x for x, c in zip(ins, d["b"]))
            bufs[d["out"]].copy_((a * b).sum().reshape(bufs[d["out"]].shape).to(torch.float32))
        return
    mats = [f64(n) for n in op["mats"]]
    if op["rank"]:
        for u, v in op["rank"]:
            mats[0] = mats[0] + torch.outer(f64(u).reshape(-1), f64(v).reshape(-1))
        if op["store"]:
            bufs[op["store"]].copy_(mats[0].to(torch.float32))
    for r in op["rows"]:
        y = coef(r["coef"], scalars) * (mats[r["mat"]] @ f64(r["x"]).reshape(-1))
        bufs[r["y"]].copy_(y.reshape(bufs[r["y"]].shape).to(torch.float32))
    for c in op["cols"]:
        y = coef(c["coef"], scalars) * (mats[c["mat"]].T @ f64(c["x"]).reshape(-1))
        bufs[c["y"]].copy_(y.reshape(bufs[c["y"]].shape).to(torch.float32))
