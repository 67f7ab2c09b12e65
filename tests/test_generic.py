"""Generic path, CPU side.

* host/cudagen.cpp emits CUDA C++ for every kernel the planner can produce
  (all 11 Table-1 sequences, fused and unfused, forced onto the generic path)
  and NVRTC compiles each one for sm_100a -- no GPU needed.
* The code generator's KernelIRs execute race-free on the reference's own
  virtual SIMT device and reproduce the reference oracle within the
  tolerance of SURVEY.md 8(c): the semantics the generic kernels reproduce
  on the GPU (tests/test_gpu_generic.py) are the reference's.
* User functions outside the hand-written algebra plan onto generic kernels.
"""
import numpy as np
import pytest

from generic_util import GENERIC_MF, USER_SCRIPTS, host_buffers, vm_plan
from golden_util import all_goldens
from gpu_util import TAU, check_output, scale_bound
from oracle import COracle, RefOracle

SEQS = ["AXPYDOT", "VADD", "WAXPBY", "SSCAL", "MADD", "BICGK", "ATAX", "SGEMV", "SGEMVT",
        "GEMVER", "GESUMMV"]
GOLDENS = all_goldens()


@pytest.fixture(scope="module")
def mf():
    import paper_1305_1183_b200 as mf
    mf.lib()
    return mf


@pytest.fixture
def generic(mf):
    mf.set_option("generic", 1)
    yield mf
    mf.set_option("generic", 0)


@pytest.mark.parametrize("mode", ["fused", "unfused"])
@pytest.mark.parametrize("seq", SEQS)
def test_every_sequence_emits_and_compiles(generic, seq, mode):
    mf = generic
    m, n = (1, 4096) if seq in ("AXPYDOT", "VADD", "WAXPBY", "SSCAL") else (96, 160)
    plan = mf.Plan.sequence(seq, m, n, mode)
    d = plan.describe()
    assert all(k["kind"] == "generic" for k in d["kernels"])
    for k in range(plan.num_kernels):
        src = plan.kernel_source(k)
        assert 'extern "C" __global__' in src and "mfj_kernel" in src
    plan.prepare()  # NVRTC -> sm_100a cubin for every kernel; raises on a compile error


@pytest.mark.parametrize("d", [0, 1, 2, 4])
def test_prefetch_distance_emits_and_compiles(generic, d):
    """Loads issued d iterations ahead: one register slot per distance, the
    loop unrolled by the distance (auto: 4 for depth 1, 1 for depth 2)."""
    mf = generic
    mf.set_option("generic_prefetch", d)
    mf.set_option("generic_iterations", 8)
    try:
        for seq, m, n, auto in [("AXPYDOT", 1, 1 << 20, 4), ("BICGK", 1024, 1024, 1)]:
            plan = mf.Plan.sequence(seq, m, n, "fused")
            src = plan.kernel_source(0)
            want = d if d else auto
            assert "float mfj_pf0[%d][" % want in src, (seq, d)
            assert ("it0 += %d" % want in src) == (want > 1)
            plan.prepare()
    finally:
        mf.set_option("generic_prefetch", 0)
        mf.set_option("generic_iterations", 0)


def test_hand_written_kernels_have_no_source(mf):
    plan = mf.Plan.sequence("BICGK", 128, 128, "fused")
    assert plan.describe()["kernels"][0]["kind"] == "matrix"
    assert plan.kernel_source(0) == ""


def test_generic_traffic_matches_hand_written(mf):
    """Algorithmic bytes are a property of the plan, not of the kernel family."""
    for seq, m, n in [("BICGK", 128, 192), ("GEMVER", 96, 160), ("AXPYDOT", 1, 4096),
                      ("GESUMMV", 64, 96)]:
        a = mf.Plan.sequence(seq, m, n, "fused").describe()
        mf.set_option("generic", 1)
        try:
            b = mf.Plan.sequence(seq, m, n, "fused").describe()
        finally:
            mf.set_option("generic", 0)
        assert (a["bytes_loaded"], a["bytes_stored"]) == (b["bytes_loaded"], b["bytes_stored"]), seq


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("mode", ["fused", "unfused"])
@pytest.mark.parametrize("g", GOLDENS, ids=lambda g: g.name)
def test_codegen_kernels_on_reference_vm(mf, g, mode):
    """The planner's KernelIRs, run by the reference's vm::launch, are
    race-free (vm.cpp:481-521) and match the reference oracle."""
    ref, co = RefOracle(), COracle()
    plan = mf.Plan.sequence(g.seq, g.meta["requested"][0], g.meta["requested"][1], mode)
    host = host_buffers(plan, g.inputs)
    vm_plan(ref, plan, host, g.scalars)
    want = g.out
    S = scale_bound(co, g.seq, g.m, g.n, g.values())
    for name in want:
        check_output(g.seq, name, host[name], want[name], S[name], exact=False)


def test_user_functions_plan_onto_generic_kernels(mf):
    lib = open(GENERIC_MF).read()
    s, m, n = USER_SCRIPTS["mul_add"]
    fused = mf.Plan.compile(s, m, n, "fused", manifest=lib).describe()
    assert [k["kind"] for k in fused["kernels"]] == ["generic"]
    unf = mf.Plan.compile(s, m, n, "unfused", manifest=lib).describe()
    assert [k["kind"] for k in unf["kernels"]] == ["generic", "stream"]  # add is hand-written
    assert fused["bytes_loaded"] + fused["bytes_stored"] == 16 * 4096
    s, m, n = USER_SCRIPTS["rscale_sgemv"]
    fused = mf.Plan.compile(s, m, n, "fused", manifest=lib)
    d = fused.describe()
    assert [k["kind"] for k in d["kernels"]] == ["generic"]
    assert d["kernels"][0]["op"]["accumulated"] == ["y"]
    assert d["kernels"][0]["column_outputs"] == []  # y is row-indexed: row-local under sharding
    fused.prepare()


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
def test_user_functions_on_reference_vm(mf):
    ref = RefOracle()
    lib = open(GENERIC_MF).read()
    s, m, n = USER_SCRIPTS["rscale_sgemv"]
    plan = mf.Plan.compile(s, m, n, "fused", manifest=lib)
    host = host_buffers(plan, {}, np.random.default_rng(3))
    vm_plan(ref, plan, host, {})
    A, d, e, x = (host[k].astype(np.float64) for k in ("A", "d", "e", "x"))
    B = (d.reshape(-1, 1) * A) * e.reshape(1, -1)
    assert np.allclose(host["B"], B, rtol=1e-6, atol=1e-7)
    y = B @ x.ravel()
    assert np.max(np.abs(host["y"].ravel() - y)) <= 1e-5 * np.max(np.abs(y))


def test_kernel_text_boundary_falls_back_to_generic(mf):
    """mf_plan_create accepts any KernelIR text the VM accepts."""
    lib = open(GENERIC_MF).read()
    s, m, n = USER_SCRIPTS["mul_add"]
    text = mf.Plan.compile(s, m, n, "fused", manifest=lib).kernel_text(0)
    p = mf.Plan.from_kernel_text(text, 1, 4096)
    d = p.describe()
    assert d["kernels"][0]["kind"] == "generic"
    assert {b["name"]: b["role"] for b in d["buffers"]} == {
        "a": "input", "b": "input", "c": "input", "o": "output"}
    p.prepare()


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
def test_barrier_mutation_is_a_race(mf):
    """SPEC.md:723 mutation check: with codegen's barriers suppressed the fused
    BiCGK kernel has shared-memory hazards the reference VM's race detector
    reports (vm.cpp:481-521); with them it has none.  (On the GPU the same
    mutated generic kernel is what compute-sanitizer racecheck flags,
    profiles/r01_sanitizer_generic.txt.)"""
    ref = RefOracle()
    counts = {}
    for barriers in (1, 0):
        mf.set_option("codegen_barriers", barriers)
        try:
            plan = mf.Plan.sequence("BICGK", 128, 128, "fused")
        finally:
            mf.set_option("codegen_barriers", 1)
        host = host_buffers(plan, {}, np.random.default_rng(0))
        counts[barriers] = ref.vm_launch(plan.kernel_text(0), host, {}, trace=True)["hazards"]
        assert ("barrier" in plan.kernel_text(0)) == bool(barriers)
    assert counts[1] == 0 and counts[0] > 0, counts


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("iterations", [1, 2, 4])
def test_codegen_race_free_with_serial_iterations(mf, iterations):
    """Barrier soundness: every kernel the code generator emits,
    for every sequence and mode, with serial iterations 1/2/4, has zero
    hazards in the reference VM's race detector -- including the loop-carried
    write-after-read of condition 2 (a load of x in iteration i+1 while other
    threads still read x in iteration i)."""
    ref = RefOracle()
    mf.set_option("generic", 1)
    mf.set_option("generic_iterations", iterations)
    try:
        for seq in SEQS:
            for mode in ("fused", "unfused"):
                m, n = (1, 8192) if seq in ("AXPYDOT", "VADD", "WAXPBY", "SSCAL") else (256, 128)
                plan = mf.Plan.sequence(seq, m, n, mode)
                host = host_buffers(plan, {}, np.random.default_rng(1))
                sc = {s: 0.5 for s in plan.describe()["scalars"]}
                for k in range(plan.num_kernels):
                    text = plan.kernel_text(k)
                    info = ref.vm_launch(text, {a: v.copy() for a, v in host.items()}, sc, trace=True)
                    assert info["hazards"] == 0, (seq, mode, k, iterations, info["hazards"])
    finally:
        mf.set_option("generic_iterations", 0)
        mf.set_option("generic", 0)


IMPL_CASES = [("BICGK", 128, 128), ("AXPYDOT", 1, 4096), ("GEMVER", 128, 128), ("GESUMMV", 128, 128),
              ("ATAX", 128, 128), ("SGEMVT", 128, 128), ("WAXPBY", 1, 2048)]


def test_implementation_generator_counts(mf):
    """Orderings x block shapes x instances x iterations x memory plans,
    deduplicated and pruned."""
    for seq, m, n in IMPL_CASES:
        p = mf.Plan.sequence(seq, m, n, "fused")
        for k in range(p.num_kernels):
            cnt = p.implementations(k)
            assert cnt >= 2, (seq, k)
            descs = [p.implementation(k, i) for i in range(cnt)]
            keys = {(tuple(d["block"]), d["instances"], d["iterations"]) for d in descs}
            # pruning: within one shape / iteration count, no implementation uses
            # more shared memory than the smallest one
            for key in keys:
                sizes = {d["shared_bytes"] for d in descs
                         if (tuple(d["block"]), d["instances"], d["iterations"]) == key}
                assert len(sizes) == 1, (seq, key, sizes)
    p = mf.Plan.sequence("BICGK", 256, 256, "fused")
    orders = {tuple(p.implementation(0, i)["order"]) for i in range(p.implementations(0))}
    assert len(orders) >= 2  # Algorithm 3's order and the script order are both generated


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", IMPL_CASES, ids=lambda c: c[0])
def test_every_implementation_on_reference_vm(mf, case):
    """every generated implementation executes on the VM with
    results equal to the reference executor within tolerance -- race-free
    (overlapping memory plans and reordered routines included).  A spread of
    about 12 implementations per kernel here; tools/check_implementations.py runs all (1091 over
    the 11 sequences at 256^2, all clean)."""
    seq, m, n = case
    ref, co = RefOracle(), COracle()
    mf.set_option("generic", 1)
    try:
        p = mf.Plan.sequence(seq, m, n, "fused")
        d = p.describe()
        rng = np.random.default_rng(5)
        vals = {b["name"]: rng.uniform(-1, 1, (b["rows"], b["cols"])).astype(np.float32)
                for b in d["buffers"] if b["role"] == "input"}
        sc = {s: 0.5 + 0.25 * i for i, s in enumerate(d["scalars"])}
        flat = {**{k: v.ravel() for k, v in vals.items()}, **sc}
        want = co.execute(seq, m, n, flat)
        S = scale_bound(co, seq, m, n, flat)
        for k in range(p.num_kernels):
            cnt = p.implementations(k)
            for i in sorted({0, cnt - 1} | set(range(0, cnt, max(1, cnt // 10)))):
                q = mf.Plan.sequence(seq, m, n, "fused")
                q.set_implementation(k, i)
                host = host_buffers(q, vals)
                vm_plan(ref, q, host, sc)  # asserts zero hazards per kernel
                for name in want:
                    check_output(seq, name, host[name].ravel(), want[name], S[name], exact=False)
    finally:
        mf.set_option("generic", 0)


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(24))
def test_random_scripts_random_implementations_on_reference_vm(mf, seed):
    """Random straight-line scripts (tests/test_gpu_random_scripts.py) through
    planner + implementation generator (a random implementation per kernel) +
    codegen, executed by the reference's VM: race-free, and equal to the
    per-call oracle chain within the tolerance."""
    from test_gpu_random_scripts import abs_chain, make_script, reference_chain
    ref, co = RefOracle(), COracle()
    rng = np.random.default_rng(1000 + seed)
    text, calls, returns = make_script(rng, 3 + seed % 5)
    m, n = 64 + 32 * (seed % 3), 96 + 32 * (seed % 4)
    plan = mf.Plan.compile(text, m, n, "fused")
    for k in range(plan.num_kernels):
        cnt = plan.implementations(k)
        plan.set_implementation(k, int(rng.integers(cnt)))
    d = plan.describe()
    env = {"k": 0.625}
    for b in d["buffers"]:
        if b["role"] == "input":
            env[b["name"]] = rng.uniform(-1, 1, (b["rows"], b["cols"])).astype(np.float32)
    host = host_buffers(plan, env)
    vm_plan(ref, plan, host, {"k": env["k"]})
    flat = {k: (v.ravel() if isinstance(v, np.ndarray) and v.shape[0] == 1 else v) for k, v in env.items()}
    want = reference_chain(co, calls, dict(flat), m, n)
    S = abs_chain(co, calls, dict(flat), m, n)
    for name in returns:
        got = host[name].astype(np.float64).ravel()
        w = np.asarray(want[name], np.float64).ravel()
        s = np.asarray(S[name], np.float64).ravel()
        lim = 4 * TAU * s + 4 * np.spacing(np.abs(w).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(got - w) <= lim), (text, name)


def test_implementation_space_counts(mf):
    """SPEC.md acceptance 6 (directional): covers x implementation choices --
    GEMVER's space is the largest of the Table-1 sequences, GESUMMV's next."""
    counts = {}
    for s in ("GEMVER", "GESUMMV", "SGEMV", "BICGK", "SSCAL"):
        txt = mf.runtime.sequence_script(s)
        m, n = (1, 8192) if s == "SSCAL" else (256, 256)
        counts[s] = mf.Plan.count_implementation_space(txt, m, n)
        assert counts[s] >= mf.Plan.count_combinations(txt, m, n)
    assert counts["GEMVER"] > counts["GESUMMV"] > max(counts["SGEMV"], counts["BICGK"]) >= 2
    assert counts["SSCAL"] < counts["BICGK"]


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
def test_acceptance_traffic_and_hoisting_on_reference_vm(mf):
    """SPEC.md acceptance 3 and 7, counted by the reference VM's own per-buffer
    counters (vm.cpp:164-173) on the code generator's kernels: fused BiCGK
    loads A exactly m*n words (2*m*n unfused); fused VADD moves 4n words
    (6n unfused); the hoisted p of fused BiCGK is loaded once per block for
    every serial iteration count."""
    ref = RefOracle()
    m = n = 256

    def words(seq, mm, nn, mode, it=None):
        if it:
            mf.set_option("generic_iterations", it)
        mf.set_option("generic", 1)
        try:
            p = mf.Plan.sequence(seq, mm, nn, mode)
        finally:
            mf.set_option("generic", 0)
            mf.set_option("generic_iterations", 0)
        host = host_buffers(p, {}, np.random.default_rng(0))
        tot = {}
        for k in range(p.num_kernels):
            st = ref.vm_launch(p.kernel_text(k), {a: v.copy() for a, v in host.items()},
                               {s: 0.5 for s in p.describe()["scalars"]})["stats"]
            for b, (ld, sd) in st["per_buffer"].items():
                t = tot.setdefault(b, [0, 0])
                t[0] += ld
                t[1] += sd
            tot.setdefault("__blocks", [0, 0])[0] += st["blocks"]
        return tot

    assert words("BICGK", m, n, "fused")["A"][0] == m * n
    assert words("BICGK", m, n, "unfused")["A"][0] == 2 * m * n
    f, u = words("VADD", 1, 8192, "fused"), words("VADD", 1, 8192, "unfused")
    tf = sum(l + s for b, (l, s) in f.items() if not b.startswith("__"))
    tu = sum(l + s for b, (l, s) in u.items() if not b.startswith("__"))
    assert (tf, tu) == (4 * 8192, 6 * 8192)
    for it in (1, 2, 4, 8):
        w = words("BICGK", m, n, "fused", it)
        assert w["p"][0] == 32 * w["__blocks"][0], it  # one 32-word p slice per block
        assert w["A"][0] == m * n


REWRITES = {"rowreduce": 1, "defer": 2, "global": 4, "store": 8, "prune": 16}


def _rewrite_markers(src):
    return {"rowreduce": "warp row reduction" in src,
            "defer": "deferred on-chip atomics" in src,
            "store": "mfj_atg(a, " in src and "warp row reduction" in src,
            "pruned": src.count("MFJ_CHECKED) __syncthreads();")}


@pytest.mark.parametrize("seq,m,n,want", [
    ("BICGK", 16384, 16384, {"rowreduce", "defer"}),
    ("ATAX", 8192, 8192, {"rowreduce", "defer"}),
    ("GESUMMV", 8192, 8192, {"rowreduce"}),
    ("GEMVER", 8192, 8192, {"rowreduce", "defer"}),
    ("AXPYDOT", 1, 1 << 24, {"defer"}),
])
def test_uninstrumented_rewrites_fire(generic, seq, m, n, want):
    """The default Table-1 generic kernels take the rewrites of the literal
    tile algorithm (host/cudagen.cpp: warp row reduction, deferred on-chip
    accumulators, barrier pruning), every one guarded so the instrumented
    variants (MFJ_STATS / TRACE / POISON / CHECKED) keep the literal
    algorithm; option generic_rewrite=0 emits the literal algorithm alone."""
    mf = generic
    plan = mf.Plan.sequence(seq, m, n, "fused")
    got, pruned = set(), 0
    for k in range(plan.num_kernels):
        src = plan.kernel_source(k)
        mk = _rewrite_markers(src)
        got |= {r for r in ("rowreduce", "defer") if mk[r]}
        pruned += mk["pruned"]
        assert not mk["store"], "store folding is off by default (measured slower)"
        # a pruned barrier is compiled out of the uninstrumented variant only:
        # every unconditional barrier of the literal kernel is still there
        # for the instrumented ones
        literal = len([l for l in src.splitlines() if l.strip() == "__syncthreads();"])
        assert literal + mk["pruned"] > 0
    assert want <= got, (seq, got)
    assert pruned > 0 or seq == "AXPYDOT"
    mf.set_option("generic_rewrite", 0)
    try:
        plan = mf.Plan.sequence(seq, m, n, "fused")
        for k in range(plan.num_kernels):
            mk = _rewrite_markers(plan.kernel_source(k))
            assert not mk["rowreduce"] and not mk["defer"] and mk["pruned"] == 0
    finally:
        mf.set_option("generic_rewrite", 55)


@pytest.mark.parametrize("mask", [0, 1, 2, 4, 8 + 1, 16, 31, 55, 63, 119, 127])
@pytest.mark.parametrize("seq", ["BICGK", "ATAX", "GEMVER", "GESUMMV", "AXPYDOT"])
def test_rewrite_masks_emit_and_compile(generic, seq, mask):
    mf = generic
    mf.set_option("generic_rewrite", mask)
    try:
        assert mf.get_option("generic_rewrite") == mask
        m, n = (1, 1 << 16) if seq == "AXPYDOT" else (2048, 2048)
        plan = mf.Plan.sequence(seq, m, n, "fused")
        for k in range(plan.num_kernels):
            mk = _rewrite_markers(plan.kernel_source(k))
            if not mask & 1:
                assert not mk["rowreduce"]
            if not mask & 2:
                assert not mk["defer"]
            if not mask & 16:
                assert mk["pruned"] == 0
        plan.prepare()
    finally:
        mf.set_option("generic_rewrite", 55)
