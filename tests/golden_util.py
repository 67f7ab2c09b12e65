"""Golden-fixture helpers shared by the CPU and GPU parity tests."""
import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# The Table-1 call chains (the reference scripts proj/data/scripts/*.mfs,
# restated): (function, [args...], result).  Literal scalars stay strings.
CHAINS = {
    "AXPYDOT": [("axpydot_stage", ["w", "alpha", "v"], "z"), ("dot", ["z", "u"], "r")],
    "VADD": [("add", ["w", "y"], "t"), ("add", ["t", "z"], "x")],
    "WAXPBY": [("scal", ["alpha", "x"], "t"), ("waxpby", ["1.0", "t", "beta", "y"], "w")],
    "SSCAL": [("scal", ["alpha", "x"], "y")],
    "MADD": [("madd", ["A", "B"], "C")],
    "BICGK": [("sgemv", ["A", "p"], "q"), ("sgemtv", ["A", "r"], "s")],
    "ATAX": [("sgemv", ["A", "x"], "t"), ("sgemtv", ["A", "t"], "y")],
    "SGEMV": [("sgemv", ["A", "x"], "t"), ("waxpby", ["alpha", "t", "beta", "y"], "z")],
    "SGEMVT": [("sgemtv", ["A", "y"], "t"), ("waxpby", ["beta", "t", "1.0", "z"], "x"),
               ("sgemv", ["A", "x"], "u"), ("scal", ["alpha", "u"], "w")],
    "GEMVER": [("ger2", ["A", "u1", "v1", "u2", "v2"], "B"), ("sgemtv", ["B", "y"], "t"),
               ("waxpby", ["beta", "t", "1.0", "z"], "x"), ("sgemvs", ["alpha", "B", "x"], "w")],
    "GESUMMV": [("sgemvs", ["alpha", "A", "x"], "t1"), ("sgemvs", ["beta", "B", "x"], "t2"),
                ("add", ["t1", "t2"], "y")],
}


class Golden:
    def __init__(self, path):
        z = np.load(path, allow_pickle=False)
        self.path = path
        self.meta = json.loads(str(z["meta"]))
        self.seq = self.meta["sequence"]
        self.m, self.n = self.meta["rows"], self.meta["cols"]
        self.inputs, self.scalars, self.out, self.call = {}, {}, {}, {}
        for k in z.files:
            if k.startswith("in__"):
                self.inputs[k[4:]] = z[k]
            elif k.startswith("sc__"):
                self.scalars[k[4:]] = float(z[k])
            elif k.startswith("out__"):
                self.out[k[5:]] = z[k]
            elif k.startswith("call__"):
                self.call[k[6:]] = z[k]

    @property
    def name(self):
        return os.path.basename(self.path)[:-4]

    def values(self):
        d = dict(self.inputs)
        d.update(self.scalars)
        return d


def all_goldens():
    return [Golden(p) for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))]
