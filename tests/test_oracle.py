"""The oracle is pinned before anything is checked against it.

CPU-only: the C restatement (oracle/mf_oracle.c) must reproduce, bit for
bit, the golden vectors the unmodified reference produced
(tests/golden/, oracle/gen_golden.py), and -- where oracle/_ref exists --
the reference itself on fresh seeds and larger sizes.
"""
import numpy as np
import pytest

from golden_util import CHAINS, all_goldens
from oracle import COracle, RefOracle

GOLDENS = all_goldens()


@pytest.fixture(scope="module")
def co():
    return COracle()


def test_goldens_present():
    assert len(GOLDENS) >= 30
    seqs = {g.seq for g in GOLDENS}
    assert seqs == set(CHAINS)


@pytest.mark.parametrize("g", GOLDENS, ids=lambda g: g.name)
def test_inputs_regenerate_bit_exact(co, g):
    plan = [(n, tuple(s) if s else None) for n, s in g.meta["inputs"]]
    ins = co.make_inputs(g.meta["seed"], plan)
    for name, a in g.inputs.items():
        assert np.array_equal(np.asarray(ins[name]).ravel(), a.ravel()), name
    for name, v in g.scalars.items():
        assert np.float32(ins[name]) == np.float32(v), name


@pytest.mark.parametrize("g", GOLDENS, ids=lambda g: g.name)
def test_reference_execute_bit_exact(co, g):
    got = co.execute(g.seq, g.m, g.n, g.values())
    for name, want in g.out.items():
        assert np.array_equal(got[name].ravel(), want.ravel()), name


def run_chain(co, g):
    env = g.values()
    for fn, args, res in CHAINS[g.seq]:
        vals = [float(a) if a[0].isdigit() else env[a] for a in args]
        env[res] = co.call(fn, g.m, g.n, vals)
    return env


@pytest.mark.parametrize("g", GOLDENS, ids=lambda g: g.name)
def test_reference_call_chain_bit_exact(co, g):
    env = run_chain(co, g)
    for name, want in g.call.items():
        assert np.array_equal(np.asarray(env[name]).ravel(), want.ravel()), name


def test_known_answers(co):
    # VADD with all-ones inputs gives 3 everywhere.
    one = np.ones(256, np.float32)
    assert np.all(co.execute("VADD", 1, 256, {"w": one, "y": one, "z": one})["x"] == 3.0)
    # SGEMV with A = I, beta = 0 gives z = alpha x.
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, 64).astype(np.float32)
    got = co.execute("SGEMV", 64, 64, {"A": np.eye(64, dtype=np.float32), "x": x,
                                         "y": x, "alpha": 0.75, "beta": 0.0})["z"]
    assert np.array_equal(got, (np.float64(0.75) * x.astype(np.float64)).astype(np.float32))


def test_hash_generator_exact_and_uniform(co):
    a = co.hash_fill(1, 0, 1 << 16)
    k = (a.astype(np.float64) + 1.0) * 8388608.0
    assert np.all(k == np.round(k)) and a.min() >= -1.0 and a.max() < 1.0
    assert abs(float(a.mean())) < 0.02
    assert co.hash_fill(1, 5, 3).tolist() == a[5:8].tolist()


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seq,rows,cols,seed", [
    ("BICGK", 256, 256, 3), ("GEMVER", 128, 192, 5), ("ATAX", 160, 96, 11),
    ("GESUMMV", 128, 128, 9), ("AXPYDOT", 1, 1 << 16, 13), ("VADD", 1, 4096, 2),
    ("WAXPBY", 1, 4096, 4), ("SGEMVT", 96, 96, 6), ("SGEMV", 64, 64, 8), ("MADD", 64, 128, 1),
])
def test_restatement_matches_reference_directly(co, seq, rows, cols, seed):
    ref = RefOracle()
    p = ref.problem(seq, rows, cols, seed)
    vals = {}
    for name in p.inputs:
        vals[name] = p.scalar(name) if name in p.scalars else p.buffer(name)
    plan = [(n, None if n in p.scalars else (vals[n].shape[0] if vals[n].ndim == 2 else 1,
                                             vals[n].shape[-1])) for n in p.inputs]
    regen = co.make_inputs(seed, plan)
    for n in p.inputs:
        assert np.array_equal(np.asarray(regen[n]).ravel(), np.asarray(vals[n]).ravel())
    want = p.execute()
    got = co.execute(seq, p.rows, p.cols, vals)
    for name, w in want.items():
        assert np.array_equal(got[name].ravel(), w.ravel()), name
