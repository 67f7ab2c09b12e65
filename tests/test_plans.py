"""CPU tests of the compile pipeline through the C-ABI (no GPU needed).

* every Table-1 sequence compiles (fused and unfused) to exactly the plan
  SURVEY.md Appendix A derives (cross-checked against the hand-derived
  builtin plans: same kernels, calls, fusion shapes, algorithmic bytes,
  buffer roles);
* each emitted KernelIR text re-enters through mf_plan_create (the
  vm::launch boundary) and lowers to the same kernel;
* the shared library exports every entry point include/mapfuse_b200.h declares;
* errors map to the reference's exception classes.
"""
import os
import re

import pytest

import paper_1305_1183_b200 as mf
from paper_1305_1183_b200 import runtime

SEQS = ["AXPYDOT", "VADD", "WAXPBY", "BICGK", "ATAX", "GEMVER", "GESUMMV", "SGEMV", "SGEMVT",
        "SSCAL", "MADD"]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def summary(d):
    ks = [(tuple(k["calls"]), k["kind"], tuple(sorted(k["shape"].items())), tuple(k["inputs"]),
           tuple(k["outputs"])) for k in d["kernels"]]
    bufs = sorted((b["name"], b["rows"], b["cols"], b["role"]) for b in d["buffers"])
    return ks, bufs, d["bytes_loaded"], d["bytes_stored"]


@pytest.mark.parametrize("mode", ["fused", "unfused"])
@pytest.mark.parametrize("seq", SEQS)
def test_pipeline_matches_appendix_a(seq, mode):
    m, n = (1, 4096) if seq in ("AXPYDOT", "VADD", "WAXPBY", "SSCAL") else (256, 256)
    got = mf.Plan.sequence(seq, m, n, mode).describe()
    want = mf.Plan.sequence(seq, m, n, "builtin_" + mode).describe()
    gk, gb, gl, gs = summary(got)
    wk, wb, wl, ws = summary(want)
    assert [k[:3] for k in gk] == [k[:3] for k in wk]
    assert (gl, gs) == (wl, ws)
    assert [(b[0], b[3]) for b in gb] == [(b[0], b[3]) for b in wb]


@pytest.mark.parametrize("seq", SEQS)
def test_kernel_text_boundary_round_trip(seq):
    p = mf.Plan.sequence(seq, 128, 128, "fused")
    d = p.describe()
    for k in range(p.num_kernels):
        text = p.kernel_text(k)
        assert text.startswith("kernel ")
        q = mf.Plan.from_kernel_text(text, 128, 128)
        qd = q.describe()["kernels"][0]
        assert qd["kind"] == d["kernels"][k]["kind"]
        assert qd["shape"] == d["kernels"][k]["shape"]
        assert qd["inputs"] == d["kernels"][k]["inputs"]
        assert qd["outputs"] == d["kernels"][k]["outputs"]


def test_fusion_bytes_saved_ratios():
    # bytes-saved ratios of the BASELINE configs
    def ratio(seq, m, n):
        f = mf.Plan.sequence(seq, m, n, "fused").describe()
        u = mf.Plan.sequence(seq, m, n, "unfused").describe()
        return (u["bytes_loaded"] + u["bytes_stored"]) / (f["bytes_loaded"] + f["bytes_stored"])
    assert abs(ratio("AXPYDOT", 1, 1 << 24) - 1.25) < 1e-6
    assert ratio("VADD", 1, 1 << 20) == 1.5
    assert abs(ratio("WAXPBY", 1, 1 << 20) - 5 / 3) < 1e-9
    assert abs(ratio("BICGK", 16384, 16384) - 2.147745792 / 1.074003968) < 1e-9
    assert abs(ratio("GEMVER", 32768, 32768) - 17181310976 / 12886343680) < 1e-9
    assert ratio("ATAX", 1024, 1024) == 1.0


def test_c_abi_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "mapfuse_b200.h")).read()
    declared = sorted(set(re.findall(r"\b(mf_[a-z_]+)\s*\(", hdr)))
    assert len(declared) >= 16
    L = mf.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert set(runtime.EXPORTS) <= set(declared)


def test_errors_map_to_reference_classes():
    with pytest.raises(mf.ParseError, match="'t'"):
        mf.Plan.compile("subvector32 x;\ninput x;\nreturn t;\n", 1, 64)
    with pytest.raises(mf.ParseError, match="type-mismatch"):
        mf.Plan.compile("subvector32 A, x, y;\ninput A, x;\ny = sgemv(A, x);\nreturn y;\n", 64, 64)
    with pytest.raises(mf.ParseError, match="kind-violation"):
        mf.Plan.compile("subvector32 x, y;\ninput x;\ny = f(x);\nreturn y;\n", 1, 64,
                        manifest="function f {\n kind map\n depth 1\n parallelism 32 1\n"
                                 " max_instances 1\n arg a subvector32 varies x\n"
                                 " out b subvector32 varies x\n routine load a {\n"
                                 "  map a: tx = w, ty = 0\n  body {\n"
                                 "   onchip a[tx] = global a[ex*32 + tx]\n  }\n }\n"
                                 " routine compute {\n  map a: tx = w, ty = 0\n"
                                 "  map b: tx = w, ty = 0\n  body {\n"
                                 "   onchip b[tx] = global a[ex*32 + tx]\n  }\n }\n"
                                 " routine store b {\n  map b: tx = w, ty = 0\n  body {\n"
                                 "   global b[ex*32 + tx] = onchip b[tx]\n  }\n }\n}\n")
    with pytest.raises(mf.ParseError):
        mf.Plan.from_kernel_text("kernel x {\n  bogus 1\n}\n", 64, 64)


def test_user_manifest_function_gets_a_kernel():
    # a new elementary function written only in the routine IR (not one of the
    # shipped ten) is understood from its compute body and lowered
    text = open(os.path.join(ROOT, "tests", "golden", "axpby3.mf")).read()
    p = mf.Plan.compile("subvector32 a, b, c, o;\nfloat k;\ninput a, b, c, k;\n"
                        "o = axpby3(k, a, b, c);\nreturn o;\n", 1, 4096, manifest=text)
    k = p.describe()["kernels"][0]
    assert k["kind"] == "stream" and k["shape"]["inputs"] == 3


# -- empirical-search support and plan files -------------
def test_ranked_combinations_and_counts():
    text = mf.runtime.sequence_script("GEMVER")
    assert mf.Plan.count_combinations(text, 256, 256) == 2
    best = mf.Plan.compile_ranked(text, 256, 256, 0)
    second = mf.Plan.compile_ranked(text, 256, 256, 1)
    assert best.num_kernels == 3 and second.num_kernels == 4
    assert best.predicted_us <= second.predicted_us
    with pytest.raises(mf.ParseError, match="out of range"):
        mf.Plan.compile_ranked(text, 256, 256, 2)
    assert mf.Plan.count_combinations(mf.runtime.sequence_script("ATAX"), 256, 256) == 1
    assert mf.Plan.count_combinations(mf.runtime.sequence_script("BICGK"), 256, 256) == 2


@pytest.mark.parametrize("seq", SEQS)
def test_plan_file_round_trip(seq):
    p = mf.Plan.sequence(seq, 96, 160, "fused")
    text = p.save()
    assert text.startswith("mapfuse-plan 1\n")
    q = mf.Plan.load(text)
    assert q.describe() == p.describe()
    assert q.save() == text


def test_plan_file_errors():
    with pytest.raises(mf.ParseError, match="not a mapfuse plan file"):
        mf.Plan.load("hello\n")
    good = mf.Plan.sequence("VADD", 1, 64).save()
    with pytest.raises(mf.ParseError, match="not terminated"):
        mf.Plan.load(good.replace("\nend\n", "\n"))


def test_cli_compile_and_usage_errors(tmp_path):
    from paper_1305_1183_b200 import cli
    out = tmp_path / "bicgk.mfp"
    assert cli.main(["compile", "--sequence", "BICGK", "--rows", "512", "--cols", "512",
                     "-o", str(out), "--emit-source", str(tmp_path / "src")]) == 0
    assert mf.Plan.load(out.read_text()).num_kernels == 1
    assert (tmp_path / "src" / "kernel0.kir").read_text().startswith("kernel ")
    assert cli.main(["compile", "--sequence", "NOPE", "-o", str(out)]) == 2
    bad = tmp_path / "bad.mfs"
    bad.write_text("subvector32 x;\ninput x;\nreturn q;\n")
    assert cli.main(["compile", "--script", str(bad), "-o", str(out)]) == 2


def test_random_scripts_always_compile():
    """Every random mixed-depth script compiles (dead calls eliminated, every
    live call lowerable onto a template) -- the GPU side runs them in
    tests/test_gpu_random_scripts.py."""
    import numpy as np
    from test_gpu_random_scripts import make_script
    for seed in range(300):
        rng = np.random.default_rng(seed)
        text, calls, ret = make_script(rng, 3 + seed % 5)
        p = mf.Plan.compile(text, 96 + 32 * (seed % 3), 128 + 64 * (seed % 4))
        assert p.num_kernels >= 1


def test_b200_mode_row_resident_plans():
    """Mode "b200" fuses ATAX's sgemv -> sgemtv through t when a row fits a
    CTA (n <= 16384) or a CTA cluster (n <= 131072), keeps the paper's plan
    otherwise and elsewhere."""
    d = mf.Plan.sequence("ATAX", 16384, 16384, "b200").describe()
    assert [k["calls"] for k in d["kernels"]] == [[0, 1]]
    assert d["kernels"][0]["op"]["chain"] is True
    assert d["bytes_loaded"] + d["bytes_stored"] == 4 * (16384 * 16384 + 2 * 16384)
    assert len(mf.Plan.sequence("ATAX", 16384, 32768, "b200").describe()["kernels"]) == 1
    assert len(mf.Plan.sequence("ATAX", 1024, 131072, "b200").describe()["kernels"]) == 1
    assert len(mf.Plan.sequence("ATAX", 1024, 131104, "b200").describe()["kernels"]) == 2
    for seq in ("BICGK", "GEMVER", "GESUMMV", "SGEMVT", "VADD", "AXPYDOT"):
        a = mf.Plan.sequence(seq, 2048, 2048, "b200").describe()
        b = mf.Plan.sequence(seq, 2048, 2048, "fused").describe()
        assert [k["calls"] for k in a["kernels"]] == [k["calls"] for k in b["kernels"]], seq
    # the chain kernel survives the KernelIR text boundary
    p = mf.Plan.sequence("ATAX", 1024, 1024, "b200")
    q = mf.Plan.from_kernel_text(p.kernel_text(0), 1024, 1024)
    assert q.describe()["kernels"][0]["op"]["chain"] is True


def test_identical_rank_updates_stored_twice_are_not_merged():
    """Two ger2 calls with the same operands and different results: the
    matrix kernel has one store, so the fusion must not lower onto it (found
    by the 1000-seed random-script sweep, profiles/r01_random_scripts.txt)."""
    text = ("TILE32x32 A, v1, v2;\nsubvector32 xa, v0;\ninput A, xa, v0;\n"
            "v1 = ger2(A, v0, xa, v0, xa);\nv2 = ger2(A, v0, xa, v0, xa);\nreturn v1, v2;\n")
    d = mf.Plan.compile(text, 128, 320, "fused").describe()
    for k in d["kernels"]:
        if k["kind"] == "matrix":
            assert k["shape"]["store"] <= 1 and "+" not in k["name"], k
    outs = {b["name"] for b in d["buffers"] if b["role"] == "output"}
    assert outs == {"v1", "v2"}


def test_b200_mode_chains_only_on_the_native_kernel():
    """Planner mode b200 fuses a row reduction into a column reduction only
    where the row-resident kernel runs it: a chain with extra members must not
    become a generic kernel (the paper's per-tile semantics would read a
    partial row sum)."""
    import numpy as np
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_random_scripts import make_script
    for seed in (48, 49, 61, 94, 99, 103, 107, 111, 118, 119):
        rng = np.random.default_rng(seed)
        text, calls, _ = make_script(rng, 3 + seed % 5)
        m, n = 96 + 32 * (seed % 3), 128 + 64 * (seed % 4)
        p = mf.Plan.compile(text, m, n, "b200")
        stmts = re.findall(r"^(\w+) = (\w+)\(([^)]*)\);$", text, re.M)  # call id = statement order
        for kd in p.describe()["kernels"]:
            if kd["kind"] != "generic":
                continue
            for a in kd["calls"]:
                for b in kd["calls"]:
                    out, fn, _ = stmts[a]
                    args = [x.strip() for x in stmts[b][2].split(",")]
                    assert not (fn in ("sgemv", "sgemvs", "sgemtv", "dot") and out in args), (seed, kd["name"])


def test_rank_reductions_skip_dots_over_replicated_vectors():
    """Under row sharding a matrix plan replicates column-indexed vectors, so
    a dot over them is whole on every rank and must not be summed again; a
    dot over row-indexed (split) vectors and every column reduction are
    partial (found by tests/test_gpu_random_sharded.py)."""
    text = ("TILE32x32 A;\nsubvector32 xa, xb, ra, v0, v1;\nfloat s0, s1;\ninput A, xa, xb, ra;\n"
            "v0 = sgemv(A, xa);\nv1 = sgemtv(A, ra);\ns0 = dot(xa, xb);\ns1 = dot(v0, ra);\n"
            "return v1, s0, s1;\n")
    p = mf.Plan.compile(text, 256, 192, "unfused")
    d = p.describe()
    red = {}
    for k, kd in enumerate(d["kernels"]):
        for name in kd["outputs"]:
            red[name] = name in p.column_outputs(k)
    assert red["v1"] and red["s1"] and not red["s0"] and not red["v0"], red
    # depth-1 plans split every vector: their dots are partial
    q = mf.Plan.sequence("AXPYDOT", 1, 4096, "fused")
    assert q.column_outputs(0) == ["r"]


def test_sharded_ranks_share_one_kernel_partition():
    """Row panels of different heights may rank fusion partitions differently;
    every rank must still run the global plan's partition so the collectives
    after each kernel line up (found by tests/test_gpu_random_sharded.py)."""
    from paper_1305_1183_b200.sharding import ShardedPlan
    text = ("TILE32x32 A;\nsubvector32 xa, xb, ra, v0, v1, v3;\nfloat k, s3;\n"
            "input A, xa, xb, ra, k;\nv0 = sgemv(A, xb);\nv1 = sgemvs(k, A, xa);\n"
            "s3 = dot(xb, xa);\nv3 = sgemtv(A, v0);\nreturn v1, s3, v3;\n")
    parts = []
    for r in range(2):
        sp = ShardedPlan(script=text, rows=224, cols=128, mode="fused", world=2, rank=r)
        parts.append(([k["calls"] for k in sp.desc["kernels"]], sp.collective_after))
    glob = [k["calls"] for k in mf.Plan.compile(text, 224, 128, "fused").describe()["kernels"]]
    assert parts[0] == parts[1] and parts[0][0] == glob, parts


@pytest.mark.parametrize("mode", ["fused", "unfused", "b200"])
def test_random_scripts_plan_file_round_trip(mode):
    """Plan files (mf_plan_save / mf_plan_load) reproduce random planner
    outputs exactly: same kernels, shapes, buffers and kernel IR."""
    import json
    import sys

    import numpy as np
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_random_scripts import make_script
    for seed in range(60):
        rng = np.random.default_rng(30000 + seed)
        text, _, _ = make_script(rng, 3 + seed % 5)
        m, n = 96 + 32 * (seed % 3), 128 + 64 * (seed % 4)
        p = mf.Plan.compile(text, m, n, mode)
        q = mf.Plan.load(p.save())
        a, b = p.describe(), q.describe()
        for d in (a, b):
            d.pop("predicted_us", None)
            for k in d["kernels"]:
                k.get("op", {}).pop("source_bytes", None)
        assert json.dumps(a, sort_keys=True) == json.dumps(b, sort_keys=True), (seed, text)
        for k in range(p.num_kernels):
            assert p.kernel_text(k) == q.kernel_text(k), (seed, k)


def test_random_kernels_text_boundary_round_trip():
    """mf_plan_create(kernel_ir_text): every kernel of random planner outputs,
    re-created from its KernelIR text alone, lowers to the same family, shape
    and bindings (the vm::launch boundary)."""
    import sys

    import numpy as np
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_random_scripts import make_script
    for seed in range(80):
        rng = np.random.default_rng(40000 + seed)
        text, _, _ = make_script(rng, 3 + seed % 5)
        m, n = 96 + 32 * (seed % 3), 128 + 64 * (seed % 4)
        p = mf.Plan.compile(text, m, n, ("fused", "unfused", "b200")[seed % 3])
        d = p.describe()
        for k in range(p.num_kernels):
            qd = mf.Plan.from_kernel_text(p.kernel_text(k), m, n).describe()["kernels"][0]
            for key in ("kind", "shape", "inputs", "outputs"):
                assert qd.get(key) == d["kernels"][k].get(key), (seed, k, key, text)


@pytest.mark.parametrize("key,good,bad", [
    ("matrix_waves", [1, 2, 16], [0, 17]),
    ("matrix_dynamic", [0, 1], [2, -1]),
    ("generic_rewrite", [0, 23, 55, 127], [-1, 128]),
    ("matrix_tile_finalize", [0, 1, 2], [3]),
])
def test_engine_option_ranges(key, good, bad):
    """Engine options round-trip through mf_set_option / mf_get_option and
    out-of-range values are rejected with MF_ERR_INVALID (the previous value
    stays)."""
    before = mf.get_option(key)
    try:
        for v in good:
            mf.set_option(key, v)
            assert mf.get_option(key) == v
        last = mf.get_option(key)
        for v in bad:
            with pytest.raises(Exception, match=key):
                mf.set_option(key, v)
            assert mf.get_option(key) == last
    finally:
        mf.set_option(key, before)


def test_plan_create_with_device_description():
    """mf_plan_create_desc: the KernelIR is checked against
    the DeviceConfig's static limits as vm::launch checks them
    (proj/src/vm.cpp:457-460) -- VmFault over the limit, ParseError for a
    malformed config -- and the SM budget is kept with the plan."""
    text = mf.Plan.sequence("BICGK", 1024, 1024, "fused").kernel_text(0)
    p = mf.Plan.from_kernel_text(text, 1024, 1024, sm_count=74)
    assert p.num_kernels == 1
    q = mf.Plan.from_kernel_text(text, 1024, 1024, device_config="warp_size 32\nmax_threads_per_block 1024\n"
                                 "shared_bytes_per_block 232448\nsm_count 148\n")
    assert q.describe()["kernels"][0]["name"] == p.describe()["kernels"][0]["name"]
    threads = 1
    for line in text.splitlines():
        if line.strip().startswith("block "):
            bx, by = line.split()[1:3]
            threads = int(bx) * int(by)
    with pytest.raises(mf.VmFault, match="threads exceeds device"):
        mf.Plan.from_kernel_text(text, 1024, 1024,
                                 device_config="max_threads_per_block %d\n" % max(32, threads // 2))
    gen = "".join(l + "\n" for l in text.splitlines())
    mf.set_option("generic", 1)
    try:  # a generic kernel with a shared tile: over a 1 KB shared limit
        gtext = mf.Plan.sequence("BICGK", 1024, 1024, "fused").kernel_text(0)
    finally:
        mf.set_option("generic", 0)
    if "shared A" in gtext:
        with pytest.raises(mf.VmFault, match="shared allocation"):
            mf.Plan.from_kernel_text(gtext, 1024, 1024, device_config="shared_bytes_per_block 1024\n")
    with pytest.raises(mf.ParseError):
        mf.Plan.from_kernel_text(gen, 1024, 1024, device_config="bogus_key 3\n")
