"""Generates tests/golden/*.npz from the UNMODIFIED reference oracle.

TEST INFRASTRUCTURE.  Run here (where /root/reference exists and oracle/_ref
is built):  python oracle/gen_golden.py
Each fixture holds, for one (sequence, rows, cols, seed):
  in__<name>    the inputs blas::make_problem generated (proj/src/blas.cpp:107)
  sc__<name>    scalar inputs
  out__<name>   blas::reference_execute outputs (blas.cpp:178)
  call__<name>  blas::reference_run_script outputs, calls in script order
                (per-call narrowing, blas.cpp:344) -- the unfused-chain oracle
  meta          json: sequence, padded rows/cols, seed, input order + shapes
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from oracle import RefOracle  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

VECTOR_SEQS = ["AXPYDOT", "VADD", "WAXPBY", "SSCAL"]
MATRIX_SEQS = ["ATAX", "BICGK", "GEMVER", "GESUMMV", "MADD", "SGEMV", "SGEMVT"]

CASES = []
for s in VECTOR_SEQS + MATRIX_SEQS:
    for seed in (1, 42):
        CASES.append((s, 64, 64, seed))
for s in VECTOR_SEQS:
    CASES.append((s, 1, 1000, 1))      # pads to 1024 (padding is data)
for s in ("BICGK", "ATAX", "GEMVER"):
    CASES.append((s, 96, 160, 1))      # rectangular: shape inference is exact here
CASES.append(("BICGK", 33, 65, 7))     # odd sizes -> padded 64 x 96


def main():
    ref = RefOracle()
    os.makedirs(OUT, exist_ok=True)
    for seq, rows, cols, seed in CASES:
        p = ref.problem(seq, rows, cols, seed)
        arrays = {}
        order = []
        for name in p.inputs:
            if name in p.scalars:
                arrays["sc__" + name] = np.float32(p.scalar(name))
                order.append([name, None])
            else:
                a = p.buffer(name)
                arrays["in__" + name] = a
                order.append([name, [a.shape[0] if a.ndim == 2 else 1, a.shape[-1]]])
        for name, a in p.execute(per_call=False).items():
            arrays["out__" + name] = a
        for name, a in p.execute(per_call=True).items():
            arrays["call__" + name] = a
        meta = {"sequence": seq, "rows": p.rows, "cols": p.cols, "seed": seed,
                "requested": [rows, cols], "inputs": order, "outputs": p.outputs}
        arrays["meta"] = np.array(json.dumps(meta))
        fn = os.path.join(OUT, "%s_%dx%d_s%d.npz" % (seq.lower(), rows, cols, seed))
        np.savez_compressed(fn, **arrays)
        print(fn, os.path.getsize(fn))


if __name__ == "__main__":
    main()
