"""Generic path on the B200: NVRTC-compiled kernels emitted
from KernelIR by host/cudagen.cpp, checked against the reference's own
virtual SIMT device (oracle/_ref: vm::launch, proj/src/vm.cpp:450-479).

Per kernel, on identical inputs (the GPU's own upstream values):
  * outputs the kernel stores without global atomics are BIT-EXACT against
    the VM (same IEEE fp32 operations in the same order, no contraction);
  * outputs accumulated with global atomics (the paper's finalisation
    option (iii)) sum in hardware order: normwise <= 1e-5 against the VM.
End to end, every output meets the oracle tolerance of SURVEY.md 8(c).
"""
import os

import numpy as np
import pytest

from generic_util import GENERIC_MF, USER_SCRIPTS, accumulated, host_buffers, vm_kernel
from golden_util import all_goldens
from gpu_util import check_output, scale_bound
from oracle import COracle, RefOracle

pytestmark = pytest.mark.gpu
GOLDENS = all_goldens()


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_1305_1183_b200 as mf
    mf.lib()
    assert RefOracle.available(), "oracle/_ref must travel with the repo"
    return torch, mf, RefOracle(), COracle()


@pytest.fixture
def generic(env):
    env[1].set_option("generic", 1)
    yield env
    env[1].set_option("generic", 0)


def run_per_kernel(torch, ref, plan, host, scalars, acc_floor=1e-30):
    """Kernel by kernel: GPU generic kernel vs the VM on the same inputs."""
    dev = {k: torch.from_numpy(v.copy()).cuda() for k, v in host.items()}
    d = plan.describe()
    for k in range(plan.num_kernels):
        assert d["kernels"][k]["kind"] == "generic"
        text = plan.kernel_text(k)
        vm_in = {n: dev[n].cpu().numpy().copy() for n in dev}
        vm_kernel(ref, plan, k, vm_in, scalars)
        plan.launch_kernel(k, dev, scalars)
        plan.check()
        acc = set(accumulated(text))
        for name in d["kernels"][k]["outputs"]:
            got = dev[name].cpu().numpy()
            want = vm_in[name]
            if name in acc:
                err = np.max(np.abs(got.astype(np.float64) - want))
                assert err <= 1e-5 * max(np.max(np.abs(want)), acc_floor), (name, err)
            else:
                bad = np.count_nonzero(got != want)
                assert bad == 0, "%s: %d elements differ from the reference VM" % (name, bad)
    return {k: v.cpu().numpy() for k, v in dev.items()}


@pytest.mark.parametrize("mode", ["fused", "unfused"])
@pytest.mark.parametrize("g", GOLDENS, ids=lambda g: g.name)
def test_generic_vs_reference_vm(generic, g, mode):
    torch, mf, ref, co = generic
    plan = mf.Plan.sequence(g.seq, g.meta["requested"][0], g.meta["requested"][1], mode)
    host = host_buffers(plan, g.inputs)
    got = run_per_kernel(torch, ref, plan, host, g.scalars)
    S = scale_bound(co, g.seq, g.m, g.n, g.values())
    for name in g.out:
        check_output(g.seq, name, got[name], g.out[name], S[name], exact=False)


@pytest.mark.parametrize("seq,m,n", [("BICGK", 1024, 2016), ("GEMVER", 512, 768),
                                     ("AXPYDOT", 1, 100032), ("GESUMMV", 256, 1024),
                                     ("ATAX", 640, 384), ("BICGK", 4096, 4096),
                                     # the sizes the generic sweeps time: 8 serial iterations,
                                     # late prefetch, 32x2 blocks, every default rewrite
                                     ("BICGK", 16384, 16384), ("GEMVER", 8192, 8192),
                                     ("ATAX", 8192, 8192), ("GESUMMV", 8192, 8192)])
def test_generic_larger_vs_oracle(generic, seq, m, n):
    """Grids of thousands of CTAs, serial iterations chosen per size, whole-plan
    launch.  Buffers are padded to 32 as the VM requires (vm.cpp:31-39)."""
    torch, mf, ref, co = generic
    from test_gpu_parity import out_shapes, rand_inputs, run_plan
    vals = rand_inputs(seq, m, n, 77)
    plan = mf.Plan.sequence(seq, m, n, "fused")
    got = run_plan(torch, plan, vals, out_shapes(plan))
    want = co.execute(seq, m, n, vals)
    S = scale_bound(co, seq, m, n, vals)
    for name in want:
        check_output(seq, name, got[name], want[name], S[name], exact=False)


@pytest.mark.parametrize("d", [1, 2, 4])
@pytest.mark.parametrize("seq,m,n", [("AXPYDOT", 1, 1 << 20), ("VADD", 1, 1 << 20),
                                     ("BICGK", 1024, 1024), ("GEMVER", 512, 512)])
def test_prefetch_distance_vs_oracle(generic, seq, m, n, d):
    """Loads issued 1, 2 or 4 iterations ahead give the same results."""
    torch, mf, ref, co = generic
    from test_gpu_parity import out_shapes, rand_inputs, run_plan
    mf.set_option("generic_prefetch", d)
    mf.set_option("generic_iterations", 8)
    try:
        vals = rand_inputs(seq, m, n, 5)
        plan = mf.Plan.sequence(seq, m, n, "fused")
        assert "float mfj_pf0[%d][" % d in plan.kernel_source(0)
        got = run_plan(torch, plan, vals, out_shapes(plan))
    finally:
        mf.set_option("generic_prefetch", 0)
        mf.set_option("generic_iterations", 0)
    want = co.execute(seq, m, n, vals)
    S = scale_bound(co, seq, m, n, vals)
    for name in want:
        check_output(seq, name, got[name], want[name], S[name], exact=False)


@pytest.mark.parametrize("mask", [0, 1, 3, 23, 31, 55, 119, 127])
@pytest.mark.parametrize("seq,m,n", [("BICGK", 1024, 2016), ("ATAX", 640, 384), ("GEMVER", 512, 768),
                                     ("GESUMMV", 256, 1024), ("AXPYDOT", 1, 4096)])
def test_rewrite_masks_vs_reference_vm(generic, seq, m, n, mask):
    """Each combination of the uninstrumented rewrites (host/cudagen.cpp:
    1 warp row reduction, 2 deferred on-chip accumulators, 4 prologue vectors
    from global, 8 row-reduction stores folded, 16 barrier pruning; 0 the
    literal tile algorithm), kernel by kernel against the reference VM."""
    torch, mf, ref, co = generic
    mf.set_option("generic_rewrite", mask)
    try:
        plan = mf.Plan.sequence(seq, m, n, "fused")
        host = host_buffers(plan, {}, np.random.default_rng(mask + 3))
        sc = {s: 0.5 for s in plan.describe()["scalars"]}
        # accumulated outputs: 1e-5 x max(|y|, 1), as the VM-exact tests --
        # a cancelling dot keeps the absolute error of its unit-scale summands
        run_per_kernel(torch, ref, plan, host, sc, acc_floor=1.0)
    finally:
        mf.set_option("generic_rewrite", 55)


@pytest.mark.parametrize("mask", [0, 23, 31, 55, 119])
@pytest.mark.parametrize("seq,m,n", [("AXPYDOT", 1, 100032), ("BICGK", 4096, 4096), ("GEMVER", 2048, 2048)])
def test_rewrite_masks_vs_oracle(generic, seq, m, n, mask):
    """Larger problems per rewrite mask, whole plan against the C oracle
    with the S-scaled tolerance (a 10^5-term dot's fp32 rounding depends on
    the summation order, which the rewrites change)."""
    torch, mf, ref, co = generic
    from test_gpu_parity import out_shapes, rand_inputs, run_plan
    mf.set_option("generic_rewrite", mask)
    try:
        vals = rand_inputs(seq, m, n, 21 + mask)
        plan = mf.Plan.sequence(seq, m, n, "fused")
        got = run_plan(torch, plan, vals, out_shapes(plan))
    finally:
        mf.set_option("generic_rewrite", 55)
    want = co.execute(seq, m, n, vals)
    S = scale_bound(co, seq, m, n, vals)
    for name in want:
        check_output(seq, name, got[name], want[name], S[name], exact=False)


@pytest.mark.parametrize("script", sorted(USER_SCRIPTS))
@pytest.mark.parametrize("mode", ["fused", "unfused"])
def test_user_functions_vs_reference_vm(env, script, mode):
    torch, mf, ref, co = env
    s, m, n = USER_SCRIPTS[script]
    plan = mf.Plan.compile(s, m, n, mode, manifest=open(GENERIC_MF).read())
    host = host_buffers(plan, {}, np.random.default_rng(11))
    dev = {k: torch.from_numpy(v.copy()).cuda() for k, v in host.items()}
    vm_in = {k: v.copy() for k, v in host.items()}
    for k in range(plan.num_kernels):
        vm_kernel(ref, plan, k, vm_in, {})
    plan.launch(dev, {})
    plan.check()
    for b in plan.describe()["buffers"]:
        if b["role"] != "output":
            continue
        got, want = dev[b["name"]].cpu().numpy(), vm_in[b["name"]]
        if b["name"] == "y":  # atomically accumulated row sums
            assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))
        else:  # maps; the hand-written add (fp64, rounded once) equals the fp32 add
            assert np.array_equal(got, want), b["name"]


def test_vm_fault_out_of_bounds(env):
    """A KernelIR reading past its buffer faults like the VM (vm.cpp:101-109)."""
    torch, mf, ref, co = env
    text = """kernel oob {
  depth 1
  block 32 1
  instances 1
  iterations 1
  iterate x
  domain a
  shared 0
  loop {
    call f.compute id=0 kind=compute shape=32x1 remap=flat {
      global o[ex*32 + tx] = global a[ex*32 + tx + 1]
    }
  }
}
"""
    p = mf.Plan.from_kernel_text(text, 1, 64)
    assert p.describe()["kernels"][0]["kind"] == "generic"
    a = np.ones(64, np.float32)
    o = np.zeros(64, np.float32)
    with pytest.raises(mf.VmFault, match="out of bounds"):
        p.launch_host({"a": a, "o": o})
    with pytest.raises(RuntimeError, match="out of bounds"):
        ref.vm_launch(text, {"a": a.reshape(1, -1).copy(), "o": o.reshape(1, -1).copy()})
    # the fault is reported once, then the plan is usable again
    text_ok = text.replace("tx + 1]", "tx]")
    p2 = mf.Plan.from_kernel_text(text_ok, 1, 64)
    p2.launch_host({"a": a, "o": o})
    assert np.array_equal(o, a)


def test_vm_fault_poisoned_read(env):
    """Reading an on-chip word never written faults when poisoning is on
    (vm.cpp:184-185), exactly as the VM with poison_onchip."""
    torch, mf, ref, co = env
    text = """kernel poison {
  depth 1
  block 32 1
  instances 1
  iterations 1
  iterate x
  domain a
  shared 32
  shared t @ 0 words 32
  loop {
    call f.compute id=0 kind=compute shape=32x1 remap=flat {
      global o[ex*32 + tx] = onchip t[tx]
    }
  }
}
"""
    a = np.ones(64, np.float32)
    o = np.zeros(64, np.float32)
    with pytest.raises(RuntimeError, match="uninitialized"):
        ref.vm_launch(text, {"a": a.reshape(1, -1).copy(), "o": o.reshape(1, -1).copy()})
    mf.set_option("generic_poison", 1)
    try:
        p = mf.Plan.from_kernel_text(text, 1, 64)
        with pytest.raises(mf.VmFault, match="uninitialized"):
            p.launch_host({"a": a, "o": o})
    finally:
        mf.set_option("generic_poison", 0)


def test_generic_deterministic_maps_and_repeatable(generic):
    torch, mf, ref, co = generic
    from test_gpu_parity import out_shapes, rand_inputs, run_plan
    vals = rand_inputs("GEMVER", 256, 384, 5)
    plan = mf.Plan.sequence("GEMVER", 256, 384, "fused")
    a = run_plan(torch, plan, vals, out_shapes(plan))
    b = run_plan(torch, plan, vals, out_shapes(plan))
    assert np.array_equal(a["B"], b["B"])  # the rank-2 map has no atomics


@pytest.mark.parametrize("seq,m,n", [("BICGK", 256, 256), ("GEMVER", 256, 256), ("AXPYDOT", 1, 8192),
                                     ("ATAX", 256, 256), ("GESUMMV", 128, 256)])
def test_implementations_on_gpu_vs_reference_vm(generic, seq, m, n):
    """Implementations from the implementation generator (routine orders,
    block shapes, instances, serial iterations, overlapping memory plans) as
    generic kernels on the B200, each checked against the reference VM on
    identical inputs: maps bit-exact, atomic accumulations within 1e-5."""
    torch, mf, ref, co = generic
    p = mf.Plan.sequence(seq, m, n, "fused")
    for k in range(p.num_kernels):
        cnt = p.implementations(k)
        for i in sorted({0, cnt - 1} | set(range(0, cnt, max(1, cnt // 8)))):
            q = mf.Plan.sequence(seq, m, n, "fused")
            q.set_implementation(k, i)
            assert q.describe()["kernels"][k]["kind"] == "generic"
            host = host_buffers(q, {}, np.random.default_rng(i))
            sc = {s: 0.5 for s in q.describe()["scalars"]}
            run_per_kernel(torch, ref, q, host, sc)


@pytest.mark.parametrize("seed", range(int(os.environ.get("MF_GENERIC_RANDOM_SEEDS", "24"))))
def test_random_scripts_generic_random_implementations(generic, seed):
    """Random scripts (planner paths the Table-1 suite does not cover), every
    kernel on the generic path with a random implementation (order, block
    shape, instances, serial iterations, memory plan), on the B200 against the
    per-call oracle chain."""
    import torch
    torch_, mf, ref, co = generic
    from test_gpu_random_scripts import abs_chain, make_script, reference_chain
    from gpu_util import TAU
    rng = np.random.default_rng(2000 + seed)
    text, calls, returns = make_script(rng, 3 + seed % 5)
    m, n = 96 + 32 * (seed % 3), 128 + 64 * (seed % 4)
    plan = mf.Plan.compile(text, m, n, "fused")
    for k in range(plan.num_kernels):
        plan.set_implementation(k, int(rng.integers(plan.implementations(k))))
    d = plan.describe()
    env = {"k": 0.625}
    for b in d["buffers"]:
        if b["role"] == "input":
            shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
            env[b["name"]] = rng.uniform(-1, 1, shp).astype(np.float32)
    bufs = {}
    for b in d["buffers"]:
        shp = (b["rows"], b["cols"]) if b["rows"] > 1 else (b["cols"],)
        v = env.get(b["name"])
        bufs[b["name"]] = (torch.from_numpy(v).cuda() if isinstance(v, np.ndarray)
                           else torch.full(shp, float("nan"), device="cuda"))
    plan.launch(bufs, {"k": env["k"]})
    plan.check()
    want = reference_chain(co, calls, dict(env), m, n)
    S = abs_chain(co, calls, dict(env), m, n)
    for name in returns:
        got = bufs[name].cpu().numpy().astype(np.float64).ravel()
        w = np.asarray(want[name], np.float64).ravel()
        s = np.asarray(S[name], np.float64).ravel()
        lim = 4 * TAU * s + 4 * np.spacing(np.abs(w).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(got - w) <= lim), (text, name)
