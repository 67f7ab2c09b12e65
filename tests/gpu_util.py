"""Shared helpers for the GPU parity tests (tolerances per SURVEY.md 8c)."""
import numpy as np

from oracle import COracle

# Element-wise bound: |y_hat - y_ref| <= TAU * S + ulp(y_ref), S = the same
# formula evaluated on absolute values.
TAU = 2.0 ** -17
NORMWISE = 1e-5

# outputs computed by a pure map chain: bit-exact against the fp64 oracle
EXACT = {
    "AXPYDOT": {"z"}, "VADD": {"x"}, "WAXPBY": {"w"}, "SSCAL": {"y"}, "MADD": {"C"},
    "GEMVER": {"B"},
}


def abs_inputs(seq, vals):
    """Inputs for evaluating the |.|-formula S with the same oracle."""
    out = {}
    for k, v in vals.items():
        out[k] = np.abs(v) if isinstance(v, np.ndarray) else abs(float(v))
    if seq.upper() == "AXPYDOT":  # z = w - alpha v  ->  |w| + |alpha||v|
        out["alpha"] = -abs(float(vals["alpha"]))
    return out


def scale_bound(co, seq, m, n, vals):
    return co.execute(seq, m, n, abs_inputs(seq, vals))


def check_output(seq, name, got, want, S, exact=None):
    got = np.asarray(got, np.float32).ravel()
    want = np.asarray(want, np.float32).ravel()
    assert got.shape == want.shape, (name, got.shape, want.shape)
    if exact is None:
        exact = name in EXACT.get(seq.upper(), set())
    if exact:
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, "%s.%s: %d/%d elements differ (first %s: %r vs %r)" % (
            seq, name, bad.size, got.size, bad[:3], got[bad[:3]], want[bad[:3]])
        return {"max_abs": 0.0}
    S = np.asarray(S, np.float64).ravel()
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    ulp = np.spacing(np.abs(want)).astype(np.float64)
    lim = TAU * S + ulp
    bad = np.nonzero(err > lim)[0]
    assert bad.size == 0, "%s.%s: %d elements exceed tau*S (worst ratio %.3g)" % (
        seq, name, bad.size, float(np.max(err / np.maximum(lim, 1e-300))))
    nw = float(np.max(err) / max(np.max(np.abs(want)), 1e-30))
    # normwise bound on vectors only: for a 1x1 output (a dot) it is the
    # relative error of one sum, which cancellation leaves unbounded in fp32
    # arithmetic of any order -- the elementwise tau*S bound above covers it
    assert got.size == 1 or nw <= NORMWISE, "%s.%s normwise %.3g" % (seq, name, nw)
    return {"max_scaled": float(np.max(err / np.maximum(S, 1e-30))), "normwise": nw}
