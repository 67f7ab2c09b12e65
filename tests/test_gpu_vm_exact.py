"""vm::launch with the reference VM's own bookkeeping, on the B200.

The generic kernel emitted from a KernelIR can carry the VM's counters and
access trace (host/cudagen.cpp MFJ_STATS / MFJ_TRACE).  Run on identical
inputs, vm::launch must then report EXACTLY what the reference's virtual SIMT
device reports (proj/src/vm.cpp): per-buffer global words, shared accesses,
atomics, barriers, arithmetic ops, modeled block cycles and cycles, launch
shape, occupancy, latency factor, trace length and race count -- and
vm::measure_routine (the paper's cost-DB micro-benchmark, vm.cpp:523-608)
the same cycles for every routine of the shipped library.
"""
import numpy as np
import pytest

from generic_util import GENERIC_MF, USER_SCRIPTS, accumulated, host_buffers
from golden_util import all_goldens
from oracle import RefOracle

pytestmark = pytest.mark.gpu
GOLDENS = all_goldens()
EXACT_KEYS = ["global_words_loaded", "global_words_stored", "per_buffer", "shared_accesses",
              "atomics", "barriers", "arith_ops", "block_cycles_sum", "cycles", "blocks",
              "threads_per_block", "shared_bytes", "occupancy", "latency_factor", "trace_records",
              "hazards"]


@pytest.fixture(scope="module")
def env():
    import paper_1305_1183_b200 as mf
    mf.lib()
    return mf, RefOracle()


def compare_kernel(mf, ref, text, host, scalars, trace=True):
    acc = accumulated(text)
    a = {k: v.copy() for k, v in host.items()}
    b = {k: v.copy() for k, v in host.items()}
    for name in acc:  # the VM contract: the caller zeroes reduce outputs
        a[name][...] = 0
        b[name][...] = 0
    want = ref.vm_launch(text, a, scalars, poison=True, trace=trace)["stats"]
    got = mf.vm_launch(text, b, scalars, trace=trace)
    assert got["vm_exact"] and got["native_kernel"] == "generic"
    keys = EXACT_KEYS if trace else [k for k in EXACT_KEYS if k not in ("trace_records", "hazards")]
    diff = {k: (got[k], want[k]) for k in keys if got[k] != want[k]}
    assert not diff, diff
    for name in a:  # maps bit-exact; atomically accumulated outputs within 1e-5 normwise
        if name in acc:
            # float atomics add in a different order than the VM; a dot that
            # cancels to a small value keeps an absolute error of the size of
            # its unit-scale summands, hence the floor of 1
            err = np.max(np.abs(a[name].astype(np.float64) - b[name]))
            assert err <= 1e-5 * max(np.max(np.abs(a[name])), 1.0), name
        else:
            assert np.array_equal(a[name], b[name]), name
    return a


@pytest.mark.parametrize("mode", ["fused", "unfused"])
@pytest.mark.parametrize("g", GOLDENS[::2], ids=lambda g: g.name)
def test_stats_and_trace_match_reference_vm(env, g, mode):
    mf, ref = env
    plan = mf.Plan.sequence(g.seq, g.meta["requested"][0], g.meta["requested"][1], mode)
    host = host_buffers(plan, g.inputs)
    for k in range(plan.num_kernels):
        host = compare_kernel(mf, ref, plan.kernel_text(k), host, g.scalars)


def test_iterations_and_instances_match(env):
    """Serial iterations (hoisted loads, epilogue stores) and 4-instance blocks."""
    mf, ref = env
    mf.set_option("generic", 1)
    mf.set_option("generic_iterations", 4)
    try:
        for seq, m, n in [("BICGK", 256, 128), ("GEMVER", 128, 96), ("AXPYDOT", 1, 8192),
                          ("GESUMMV", 128, 64)]:
            plan = mf.Plan.sequence(seq, m, n, "fused")
            assert "iterations 4" in plan.kernel_text(0)
            host = host_buffers(plan, {}, np.random.default_rng(1))
            sc = {s: 0.5 for s in plan.describe()["scalars"]}
            for k in range(plan.num_kernels):
                host = compare_kernel(mf, ref, plan.kernel_text(k), host, sc)
    finally:
        mf.set_option("generic_iterations", 0)
        mf.set_option("generic", 0)


def test_races_of_the_barrier_mutation_match(env):
    """the barrier-suppressed BiCGK kernel has the same number of
    hazards on the GPU trace as in the reference VM's trace."""
    mf, ref = env
    mf.set_option("codegen_barriers", 0)
    try:
        plan = mf.Plan.sequence("BICGK", 128, 128, "fused")
    finally:
        mf.set_option("codegen_barriers", 1)
    host = host_buffers(plan, {}, np.random.default_rng(0))
    text = plan.kernel_text(0)
    want = ref.vm_launch(text, {k: v.copy() for k, v in host.items()}, {}, trace=True)["stats"]
    got = mf.vm_launch(text, {k: v.copy() for k, v in host.items()}, {}, trace=True)
    assert want["hazards"] > 0
    assert got["hazards"] == want["hazards"]
    assert got["trace_records"] == want["trace_records"]


def test_user_function_without_trace_reports_vm_stats(env):
    mf, ref = env
    s, m, n = USER_SCRIPTS["rscale_sgemv"]
    plan = mf.Plan.compile(s, m, n, "fused", manifest=open(GENERIC_MF).read())
    host = host_buffers(plan, {}, np.random.default_rng(4))
    compare_kernel(mf, ref, plan.kernel_text(0), host, {}, trace=False)


def test_hand_written_path_reports_shape(env):
    """A lowerable kernel runs the hand-written family (fast path): the launch
    shape matches the VM, traffic is algorithmic."""
    mf, ref = env
    plan = mf.Plan.sequence("BICGK", 128, 192, "fused")
    host = host_buffers(plan, {}, np.random.default_rng(2))
    got = mf.vm_launch(plan.kernel_text(0), {k: v.copy() for k, v in host.items()})
    want = ref.vm_launch(plan.kernel_text(0), {k: v.copy() for k, v in host.items()})["stats"]
    assert got["native_kernel"] == "matrix" and not got["vm_exact"]
    for k in ("blocks", "threads_per_block", "shared_bytes", "occupancy", "latency_factor"):
        assert got[k] == want[k], k
    assert got["per_buffer"]["A"] == [128 * 192, 0]  # A read once


def test_measure_routine_matches_reference(env):
    mf, ref = env
    lib = ref.L.mfr_manifest().decode()
    fns = [l.split()[1] for l in lib.splitlines() if l.startswith("function ")]
    checked = 0
    for fn in fns:
        routines = []
        cur = None
        for l in lib.splitlines():
            if l.startswith("function "):
                cur = l.split()[1]
            elif cur == fn and l.strip().startswith("routine "):
                parts = l.split()
                routines.append(parts[1] + ("_" + parts[2] if parts[2] != "{" else ""))
        for r in routines:
            for inst, it, extra in [(1, 1, 0), (4, 1, 0), (2, 3, 0), (1, 2, 16384)]:
                want = ref.measure_routine(fn, r, inst, it, extra)
                got = mf.measure_routine(fn, r, inst, it, extra)
                assert got == want, (fn, r, inst, it, extra, got, want)
                checked += 1
    assert checked >= 100


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("MF_RANDOM_VM_SEEDS", "12"))))
def test_random_scripts_stats_match_reference_vm(env, seed):
    """Every kernel of a random planner output (tests/test_gpu_random_scripts.py)
    through vm::launch on the GPU against the reference VM: the same
    ExecutionStats field by field, maps bit-exact."""
    mf, ref = env
    from test_gpu_random_scripts import make_script
    rng = np.random.default_rng(9000 + seed)
    text, _, _ = make_script(rng, 3 + seed % 5)
    m, n = 64 + 32 * (seed % 2), 96 + 32 * (seed % 3)
    plan = mf.Plan.compile(text, m, n, ("fused", "unfused")[seed % 2])
    host = host_buffers(plan, {}, rng)
    mf.set_option("vm_exact", 1)  # hand-written-covered kernels count like the VM too
    try:
        for k in range(plan.num_kernels):
            host = compare_kernel(mf, ref, plan.kernel_text(k), host, {"k": 0.625}, trace=seed % 3 == 0)
    finally:
        mf.set_option("vm_exact", 0)
