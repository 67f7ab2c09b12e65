"""GPU parity at BASELINE sizes through size-independent checks.

Full-size problems exceed what the CPU oracle evaluates in seconds, so the
matrices are generated on the device by the counter-based generator that
oracle/mf_oracle.c restates bit for bit, and sampled rows / columns are
re-derived in fp64 on the CPU.
"""
import numpy as np
import pytest

from gpu_util import NORMWISE, TAU
from oracle import COracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_1305_1183_b200 as mf
    mf.lib()
    return torch, mf, COracle()


# sampled rows / columns per full-size output (~256 + 256)
NSAMPLE = 256


def _check(got, ref, absref, what):
    """|got - ref| <= tau * S + ulp(ref) per element, and the normwise bound
    max|got - ref| / max|ref| <= 1e-5 over the sample."""
    err = np.abs(got.astype(np.float64) - ref)
    lim = TAU * absref + np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    assert np.all(err <= lim), (what, float(np.max(err / lim)))
    nw = float(np.max(err) / max(float(np.max(np.abs(ref))), 1e-30))
    assert nw <= NORMWISE, (what, "normwise", nw)
    return nw


@pytest.mark.parametrize("m,n", [(16384, 16384), (4096, 131072), (131072, 131072)])
def test_bicgk_sampled_rows_and_columns(env, m, n):
    torch, mf, co = env
    plan = mf.Plan.sequence("BICGK", m, n, "fused")
    A = torch.empty(m, n, device="cuda")
    mf.generate(A, seed=7)
    p = torch.empty(n, device="cuda")
    r = torch.empty(m, device="cuda")
    mf.generate(p, seed=8)
    mf.generate(r, seed=9)
    q = torch.empty(m, device="cuda")
    s = torch.empty(n, device="cuda")
    plan.launch({"A": A, "p": p, "r": r, "q": q, "s": s})
    torch.cuda.synchronize()
    rng = np.random.default_rng(m + n)
    rows = np.sort(rng.choice(m, NSAMPLE, replace=False))
    cols = np.sort(rng.choice(n, NSAMPLE, replace=False))
    pc, rc = p.cpu().numpy(), r.cpu().numpy()
    qr, qa = co.hash_rows(7, n, rows, pc)
    _check(q.cpu().numpy()[rows], qr, qa, "q")
    sr, sa = co.hash_cols(7, n, 0, m, cols, rc)
    _check(s.cpu().numpy()[cols], sr, sa, "s")
    del A
    torch.cuda.empty_cache()


def test_gemver_full_size_properties(env):
    """GEMVER 32768^2: B is exact (fp64 rank update rounded once); x and w
    checked on sampled entries against fp64 recomputation from B."""
    torch, mf, co = env
    m = n = 32768
    plan = mf.Plan.sequence("GEMVER", m, n, "fused")
    d = {}
    for i, name in enumerate(["A", "u1", "v1", "u2", "v2", "y", "z"]):
        shp = (m, n) if name == "A" else ((m,) if name in ("u1", "u2", "y") else (n,))
        d[name] = torch.empty(shp, device="cuda")
        mf.generate(d[name], seed=20 + i)
    d["B"] = torch.empty(m, n, device="cuda")
    d["x"] = torch.empty(n, device="cuda")
    d["w"] = torch.empty(m, device="cuda")
    al, be = 0.625, 0.375
    plan.launch(d, {"alpha": al, "beta": be})
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    rows = np.sort(rng.choice(m, NSAMPLE, replace=False))
    cols = np.sort(rng.choice(n, NSAMPLE, replace=False))
    f64 = lambda t: t.cpu().numpy().astype(np.float64)
    u1, v1, u2, v2, y, z = (f64(d[k]) for k in ("u1", "v1", "u2", "v2", "y", "z"))
    A_rows = d["A"][torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64)
    B_rows = d["B"][torch.from_numpy(rows).cuda()].cpu().numpy()
    Bexp = (A_rows + u1[rows, None] * v1[None, :] + u2[rows, None] * v2[None, :]).astype(np.float32)
    assert np.array_equal(B_rows, Bexp)
    # x = beta * B^T y + z on sampled columns (B exact in float -> fp64 reference)
    Bc = d["B"][:, torch.from_numpy(cols).cuda()].cpu().numpy().astype(np.float64)
    Ac = d["A"][:, torch.from_numpy(cols).cuda()].cpu().numpy().astype(np.float64)
    B64c = Ac + u1[:, None] * v1[None, cols] + u2[:, None] * v2[None, cols]
    xref = be * (B64c.T @ y) + z[cols]
    xabs = abs(be) * (np.abs(B64c).T @ np.abs(y)) + np.abs(z[cols])
    _check(d["x"].cpu().numpy()[cols], xref, xabs, "x")
    # w = alpha * B x on sampled rows using the device's x
    x = f64(d["x"])
    wref = al * (B_rows.astype(np.float64) @ x)
    wabs = abs(al) * (np.abs(B_rows.astype(np.float64)) @ np.abs(x))
    _check(d["w"].cpu().numpy()[rows], wref, wabs, "w")


def test_gesummv_full_size_sampled_rows(env):
    """GESUMMV 32768^2 (BASELINE configs[3]; proj/data/scripts/gesummv.mfs:8-10,
    oracle proj/src/blas.cpp:243+): y = alpha A x + beta B x on sampled rows
    against fp64 sums over the same hash-generated A and B."""
    torch, mf, co = env
    m = n = 32768
    plan = mf.Plan.sequence("GESUMMV", m, n, "fused")
    A = torch.empty(m, n, device="cuda")
    B = torch.empty(m, n, device="cuda")
    mf.generate(A, seed=71)
    mf.generate(B, seed=72)
    x = torch.empty(n, device="cuda")
    mf.generate(x, seed=73)
    y = torch.full((m,), float("nan"), device="cuda")
    al, be = 0.625, 0.375
    plan.launch({"A": A, "B": B, "x": x, "y": y}, {"alpha": al, "beta": be})
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(11).choice(m, NSAMPLE, replace=False))
    xc = x.cpu().numpy()
    ta, taa = co.hash_rows(71, n, rows, xc)
    tb, tba = co.hash_rows(72, n, rows, xc)
    _check(y.cpu().numpy()[rows], al * ta + be * tb, abs(al) * taa + abs(be) * tba, "y")
    assert not torch.isnan(y).any()
    del A, B
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["fused", "b200"])
def test_atax_131072_sampled(env, mode):
    """ATAX 131072^2 (BASELINE configs[4]; proj/data/scripts/atax.mfs:7-8,
    oracle proj/src/blas.cpp:194-196 = matvec_t(matvec)): the paper's
    two-kernel plan and the row-resident cluster kernel (mode b200).  The CPU
    evaluates the whole intermediate t = A x in fp64 (multi-threaded hash
    oracle), then y = A^T t on sampled columns, with the |.|-formula
    S = |A|^T (|A||x|) as the tolerance scale; t is checked on sampled rows
    where the plan stores it."""
    torch, mf, co = env
    m = n = 131072
    plan = mf.Plan.sequence("ATAX", m, n, mode)
    d = plan.describe()
    if mode == "b200":
        assert plan.num_kernels == 1 and d["kernels"][0]["shape"]["chain"] == 1
    A = torch.empty(m, n, device="cuda")
    mf.generate(A, seed=81)
    x = torch.empty(n, device="cuda")
    mf.generate(x, seed=82)
    bufs = {"A": A, "x": x, "y": torch.full((n,), float("nan"), device="cuda")}
    if any(b["name"] == "t" for b in d["buffers"]):
        bufs["t"] = torch.full((m,), float("nan"), device="cuda")
    plan.launch(bufs)
    torch.cuda.synchronize()
    xc = x.cpu().numpy()
    t64, tabs = co.hash_matvec_all(81, m, n, xc)
    rng = np.random.default_rng(13)
    if "t" in bufs:
        rows = np.sort(rng.choice(m, NSAMPLE, replace=False))
        _check(bufs["t"].cpu().numpy()[rows], t64[rows], tabs[rows], "t")
    cols = np.sort(rng.choice(n, NSAMPLE, replace=False))
    yr, ya = co.hash_cols_f64(81, n, m, cols, t64, tabs)
    y = bufs["y"].cpu().numpy()
    assert not np.isnan(y).any()
    _check(y[cols], yr, ya, "y")
    del A, bufs
    torch.cuda.empty_cache()


def test_sharded_plan_single_rank_equals_plan(env):
    torch, mf, co = env
    from paper_1305_1183_b200.sharding import ShardedPlan
    sp = ShardedPlan("ATAX", 2048, 3072, "fused", world=1, rank=0)
    plan = mf.Plan.sequence("ATAX", 2048, 3072, "fused")
    A = torch.empty(2048, 3072, device="cuda")
    x = torch.empty(3072, device="cuda")
    mf.generate(A, seed=1)
    mf.generate(x, seed=2)
    y1 = torch.empty(3072, device="cuda")
    y2 = torch.empty(3072, device="cuda")
    info = sp.launch({"A": A, "x": x, "y": y1, "t": torch.empty(2048, device="cuda")})
    plan.launch({"A": A, "x": x, "y": y2})
    torch.cuda.synchronize()
    assert info["collectives"] == 1
    assert torch.equal(y1, y2)


def test_blas1_bench_size_exact(env):
    """The bench workload at its full size (n = 2^28): VADD x = w + y + z and
    WAXPBY w = alpha x + beta y through the fused stream kernels, inputs from
    the device generator.  Maps are bit-exact (fp64, rounded once), so whole
    slices are compared exactly -- the first and last 2^20 elements (the
    block-edge tail included) and a random interior slice."""
    torch, mf, co = env
    n = 1 << 28
    vadd = mf.Plan.sequence("VADD", 1, n, "fused")
    ins = {}
    for i, k in enumerate(("w", "y", "z")):
        ins[k] = torch.empty(n, device="cuda")
        mf.generate(ins[k], seed=40 + i)
    x = torch.empty(n, device="cuda")
    vadd.launch({**ins, "x": x})
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    mid = int(rng.integers(1 << 20, n - (2 << 20))) // 32 * 32
    for lo in (0, mid, n - (1 << 20)):
        sl = slice(lo, lo + (1 << 20))
        vals = {k: ins[k][sl].cpu().numpy() for k in ("w", "y", "z")}
        want = co.execute("VADD", 1, 1 << 20, vals)["x"]  # elementwise: a slice is a problem
        assert np.array_equal(x[sl].cpu().numpy(), want), lo
    del ins, x
    torch.cuda.empty_cache()
    wax = mf.Plan.sequence("WAXPBY", 1, n, "fused")
    xx, yy, ww = (torch.empty(n, device="cuda") for _ in range(3))
    mf.generate(xx, seed=50)
    mf.generate(yy, seed=51)
    al, be = 0.625, 0.375
    wax.launch({"x": xx, "y": yy, "w": ww}, {"alpha": al, "beta": be})
    torch.cuda.synchronize()
    for lo in (0, mid, n - (1 << 20)):
        sl = slice(lo, lo + (1 << 20))
        vals = {"x": xx[sl].cpu().numpy(), "y": yy[sl].cpu().numpy(), "alpha": al, "beta": be}
        want = co.execute("WAXPBY", 1, 1 << 20, vals)["w"]
        assert np.array_equal(ww[sl].cpu().numpy(), want), lo
    del xx, yy, ww
    torch.cuda.empty_cache()


def test_axpydot_full_size(env):
    """AXPYDOT at n = 2^24 (BASELINE configs[0]) against the C oracle on the
    same device-generated inputs: z bit-exact, r within tau * sum |z u|."""
    torch, mf, co = env
    n = 1 << 24
    plan = mf.Plan.sequence("AXPYDOT", 1, n, "fused")
    d = {}
    for i, k in enumerate(("w", "v", "u")):
        d[k] = torch.empty(n, device="cuda")
        mf.generate(d[k], seed=60 + i)
    d["z"] = torch.empty(n, device="cuda")
    d["r"] = torch.empty(1, device="cuda")
    al = 0.625
    plan.launch(d, {"alpha": al})
    torch.cuda.synchronize()
    vals = {k: d[k].cpu().numpy() for k in ("w", "v", "u")}
    want = co.execute("AXPYDOT", 1, n, {**vals, "alpha": al})
    assert np.array_equal(d["z"].cpu().numpy(), want["z"])
    zz = want["z"].astype(np.float64)
    S = float(np.sum(np.abs(zz * vals["u"].astype(np.float64))))
    _check(d["r"].cpu().numpy(), want["r"].astype(np.float64), np.array([S]), "r")
