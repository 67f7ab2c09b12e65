"""CPU: bench.py's reference arm (the driver's `--impl reference` run) -- the
reference's own CPU path (reference_execute from oracle/_ref) on the host
cores, printing the contract's JSON line without touching a GPU."""
import json
import os
import subprocess
import sys

import pytest

from oracle import RefOracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference"] + list(args),
                       capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
def test_reference_arm_blas1_line():
    d = _line("--steps", "2", "--warmup", "1", "--n", str(1 << 20))
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["metric"] == "fused-sequence effective GB/s" and d["higher_is_better"] is True
    assert d["config"]["n"] == 1 << 20
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
def test_reference_arm_sharded_workload_line():
    d = _line("--steps", "1", "--warmup", "1", "--workload", "bicgk-sharded", "--n-matrix", "2048")
    assert d["impl"] == "reference" and d["value"] > 0 and d["scaling"] == "strong"
    assert "BICGK" in d["config"]["workload"].upper() and d["config"]["n"] == 2048
