"""Bound plans and CUDA-graph launches (mf_plan_bind / mf_bound_launch /
mf_bound_graph_launch): the same kernels with the host-side work done once.
Results must be bit-identical to Plan.launch (every kernel is deterministic),
across repeated launches (grid barriers and tickets reset themselves)."""
import numpy as np
import pytest

from generic_util import GENERIC_MF, USER_SCRIPTS

pytestmark = pytest.mark.gpu


def make(torch, mf, plan, seed):
    bufs = {}
    for i, b in enumerate(plan.describe()["buffers"]):
        t = torch.empty((b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],), device="cuda")
        if b["role"] == "input":
            mf.generate(t, seed=seed + i)
        else:
            t.fill_(float("nan"))
        bufs[b["name"]] = t
    return bufs


def outputs(plan, bufs):
    return {b["name"]: bufs[b["name"]].cpu().numpy().copy() for b in plan.describe()["buffers"]
            if b["role"] == "output"}


@pytest.mark.parametrize("seq,m,n,mode", [
    ("AXPYDOT", 1, 1 << 20, "fused"), ("VADD", 1, 1 << 20, "fused"), ("WAXPBY", 1, 4096, "fused"),
    ("BICGK", 2048, 4096, "fused"), ("ATAX", 1024, 2048, "fused"), ("ATAX", 1024, 2048, "b200"),
    ("GEMVER", 1024, 1536, "fused"), ("GESUMMV", 512, 2048, "fused"), ("SGEMVT", 512, 768, "unfused")])
def test_bound_and_graph_match_plan_launch(seq, m, n, mode):
    import torch
    import paper_1305_1183_b200 as mf
    plan = mf.Plan.sequence(seq, m, n, mode)
    sc = {"alpha": 0.5, "beta": 0.75}
    bufs = make(torch, mf, plan, 3)
    plan.launch(bufs, sc)
    torch.cuda.synchronize()
    want = outputs(plan, bufs)
    bound = plan.bind(bufs, sc)
    for k in want:
        bufs[k].fill_(float("nan"))
    for _ in range(3):
        bound.launch()
    torch.cuda.synchronize()
    got = outputs(plan, bufs)
    for k in want:
        assert np.array_equal(got[k], want[k], equal_nan=True), k
    s = torch.cuda.Stream()
    for k in want:
        bufs[k].fill_(float("nan"))
    torch.cuda.synchronize()
    for _ in range(4):
        bound.graph_launch(s)
    s.synchronize()
    got = outputs(plan, bufs)
    for k in want:
        assert np.array_equal(got[k], want[k], equal_nan=True), k


def test_generic_plan_graph():
    import torch
    import paper_1305_1183_b200 as mf
    s_, m, n = USER_SCRIPTS["rscale_sgemv"]
    plan = mf.Plan.compile(s_, m, n, "fused", manifest=open(GENERIC_MF).read())
    bufs = make(torch, mf, plan, 9)
    plan.launch(bufs, {})
    torch.cuda.synchronize()
    want = outputs(plan, bufs)
    bound = plan.bind(bufs, {})
    st = torch.cuda.Stream()
    for _ in range(3):
        bound.graph_launch(st)
    st.synchronize()
    got = outputs(plan, bufs)
    assert np.array_equal(got["B"], want["B"])  # map: exact
    assert np.max(np.abs(got["y"] - want["y"])) <= 1e-5 * np.max(np.abs(want["y"]))  # atomics


def test_graph_needs_a_stream():
    import torch
    import paper_1305_1183_b200 as mf
    plan = mf.Plan.sequence("VADD", 1, 4096, "fused")
    bufs = make(torch, mf, plan, 1)
    bound = plan.bind(bufs, {})
    with pytest.raises(mf.ParseError, match="non-default stream"):
        bound.graph_launch(None)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("MF_RANDOM_BOUND_SEEDS", "16"))))
def test_random_scripts_bound_and_graph(seed):
    """Random planner outputs (tests/test_gpu_random_scripts.py) replayed as
    bound plans and CUDA graphs: bit-identical to Plan.launch where every
    kernel is hand-written (generic kernels accumulate with atomics)."""
    import torch
    import paper_1305_1183_b200 as mf
    from test_gpu_random_scripts import make_script
    rng = np.random.default_rng(7000 + seed)
    text, _, _ = make_script(rng, 3 + seed % 5)
    m, n = 1024 + 96 * (seed % 3), 2048 + 160 * (seed % 4)
    plan = mf.Plan.compile(text, m, n, ("fused", "unfused", "b200")[seed % 3])
    if any(k["kind"] == "generic" for k in plan.describe()["kernels"]):
        pytest.skip("generic kernels are not bit-reproducible (float atomics)")
    sc = {"k": 0.625}
    bufs = make(torch, mf, plan, seed)
    plan.launch(bufs, sc)
    torch.cuda.synchronize()
    want = outputs(plan, bufs)
    bound = plan.bind(bufs, sc)
    s = torch.cuda.Stream()
    for k in want:
        bufs[k].fill_(float("nan"))
    torch.cuda.synchronize()
    for _ in range(3):
        bound.graph_launch(s)
    s.synchronize()
    got = outputs(plan, bufs)
    for k in want:
        assert np.array_equal(got[k], want[k], equal_nan=True), (text, k)


def test_bound_plan_survives_workspace_growth():
    """Paper-mode ATAX with n > 2048: sgemv records a small row-partial
    scratch, then sgemtv needs a larger column-partial one.  The first
    recorded launch must keep a live buffer (the workspace retires outgrown
    scratch instead of freeing it), and later cudaMalloc users must not be
    written through it."""
    import torch
    import paper_1305_1183_b200 as mf
    plan = mf.Plan.sequence("ATAX", 2048, 8192, "fused")
    assert plan.num_kernels == 2
    bufs = make(torch, mf, plan, 11)
    plan.launch(bufs)
    torch.cuda.synchronize()
    want = outputs(plan, bufs)
    bound = plan.bind(bufs, {})
    canary = torch.full((1 << 22,), 7.0, device="cuda")  # allocated after the bind
    for k in want:
        bufs[k].fill_(float("nan"))
    for _ in range(3):
        bound.launch()
    torch.cuda.synchronize()
    got = outputs(plan, bufs)
    for k in want:
        assert np.array_equal(got[k], want[k]), k
    assert bool(torch.all(canary == 7.0))


@pytest.mark.parametrize("seq,m,n", [("BICGK", 4096, 8192), ("AXPYDOT", 1, 1 << 22),
                                     ("GEMVER", 2048, 4096)])
def test_one_plan_concurrent_streams(seq, m, n):
    """One plan launched on two streams at once with different inputs: each
    stream has its own workspace (barrier counters, dot ticket, partials), so
    both results equal the serial launches bit for bit."""
    import torch
    import paper_1305_1183_b200 as mf
    plan = mf.Plan.sequence(seq, m, n, "fused")
    sc = {"alpha": 0.5, "beta": 0.75}
    b1, b2 = make(torch, mf, plan, 21), make(torch, mf, plan, 57)
    plan.launch(b1, sc)
    plan.launch(b2, sc)
    torch.cuda.synchronize()
    w1, w2 = outputs(plan, b1), outputs(plan, b2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(5):
        for k in w1:
            b1[k].fill_(float("nan"))
            b2[k].fill_(float("nan"))
        torch.cuda.synchronize()
        plan.launch(b1, sc, stream=s1)
        plan.launch(b2, sc, stream=s2)
        torch.cuda.synchronize()
        g1, g2 = outputs(plan, b1), outputs(plan, b2)
        for k in w1:
            assert np.array_equal(g1[k], w1[k]), (k, 1)
            assert np.array_equal(g2[k], w2[k]), (k, 2)


def test_matrix_dims_must_be_padded_to_32():
    """The matrix families reject shapes the reference never produces (every
    buffer is padded to 32, proj/include/mapfuse/blas.hpp:29-30) instead of
    running the cross-CTA finalize on a ragged column group."""
    import torch
    import paper_1305_1183_b200 as mf
    plan = mf.Plan.sequence("BICGK", 64, 64, "fused")
    A = torch.zeros(64, 52, device="cuda")
    with pytest.raises(mf.VmFault, match="multiples of 32"):
        plan.launch({"A": A, "p": torch.zeros(52, device="cuda"), "r": torch.zeros(64, device="cuda"),
                     "q": torch.zeros(64, device="cuda"), "s": torch.zeros(52, device="cuda")})
