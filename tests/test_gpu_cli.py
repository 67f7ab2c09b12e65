"""GPU: the CLI's empirical search, verification and plan-file run."""
import json

import pytest

pytestmark = pytest.mark.gpu


def test_search_reports_measured_ranking(capsys):
    from paper_1305_1183_b200 import cli
    assert cli.main(["search", "--sequence", "BICGK", "--rows", "4096", "--cols", "4096",
                     "--top", "2", "--reps", "5"]) == 0
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert out["combinations"] == 2 and out["evaluated"] == 2
    # the fused single pass must be the measured winner (2x fewer bytes)
    assert out["best_measured_rank"] == 0
    assert out["results"][0]["measured_us"] < out["results"][1]["measured_us"]


def test_verify_every_combination(capsys):
    from paper_1305_1183_b200 import cli
    assert cli.main(["verify", "--size", "128", "--seed", "3"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert len(lines) >= 11 and all(l.endswith(": ok") for l in lines)


def test_run_plan_file(tmp_path, capsys):
    from paper_1305_1183_b200 import cli
    p = tmp_path / "gemver.mfp"
    assert cli.main(["compile", "--sequence", "GEMVER", "--rows", "2048", "--cols", "2048",
                     "-o", str(p)]) == 0
    capsys.readouterr()
    assert cli.main(["run", str(p), "--reps", "3"]) == 0
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert out["us"] > 0 and out["GBps"] > 0
