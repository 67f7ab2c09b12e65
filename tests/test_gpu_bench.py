"""GPU: bench.py's contract at N = 1 and, on one GPU, its multi-rank code
path (MF_BENCH_SHARED_GPU=1: both ranks on cuda:0 over gloo) -- small sizes,
so this checks the JSON line's shape and the cross-rank plumbing, not speed."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--n", str(1 << 22),
                        "--n-matrix", "4096", "--no-suite", "--no-cpu"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "config", "roofline", "clocks", "gpu_launches", "e2e"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["gpu_launches"] == 10 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["sharded"]["value"] > 0 and d["sharded"]["rows_per_rank"] == 4096
    assert d["sharded"]["parity"]["ok"]
    assert d["atax_b200"]["value"] > 0 and d["atax_b200"]["parity"]["ok"], d["atax_b200"]


def test_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, MF_BENCH_SHARED_GPU="1")

    def torchrun(*args):
        return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(_port()),
                os.path.join(ROOT, "bench.py"), "--gpus", "2"] + list(args)

    cmd = torchrun("--steps", "5", "--elements", str(1 << 22), "--n-matrix", "4096")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    # N > 1 headline: BiCGK row-sharded strong scaling (bench.py workload "auto")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["rows_per_rank"] == 2048 and d["config"]["collectives_per_step"] == 1
    assert d["parity"]["ok"] and d["parity"]["checked"] == ["q", "s"]
    ss = d["strong_scaling"]
    assert ss["n"] == 2 and ss["t1_ms"] > 0 and ss["efficiency"] > 0
    assert "max over ranks" in d["e2e"]["path"] and d["e2e"]["h2d_bytes_per_step"] > 0
    ref = subprocess.run(torchrun("--impl", "reference", "--steps", "2"), capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert ref.returncode == 0, ref.stderr[-3000:]
    assert _line(ref.stdout)["impl"] == "reference"
