"""abft_cli (csrc/cli.cpp), the command-line front end over the C ABI -- the checks of the reference's CLI smoke test
(P:tests/cli_smoke.cmake:14-30) plus the eb-check exit status (P:tools/abft_cli.cpp:165)."""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
CLI = REPO / "paper_2103_00130_b200" / "abft_cli"
sys.path.insert(0, str(REPO / "tests"))


def run(*args, **kw):
    assert CLI.exists(), "abft_cli not built (python paper_2103_00130_b200/build.py)"
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=600, **kw)


def test_analyze_and_usage_errors():
    r = run("analyze", "--m", 1, "--n", 800, "--k", 3200, "--d", 64, "--pool", 100)
    assert r.returncode == 0 and "98.8281" in r.stdout  # the m = 1 bit-flip detection figure
    assert run("campaign", "/nonexistent/does_not_exist.cfg").returncode == 1
    assert run().returncode == 1 and run("frobnicate").returncode == 1
    assert run("analyze", "--m", 0, "--n", 1, "--k", 1).returncode == 1


@pytest.mark.gpu
def test_campaign_bench_and_eb_check(tmp_path):
    from campaign_configs import CAMPAIGNS
    cfg = tmp_path / "smoke.cfg"
    cfg.write_text(CAMPAIGNS["gemm_smoke"][0])
    r = run("campaign", cfg, "--out", tmp_path / "smoke.csv")
    assert r.returncode == 0 and (tmp_path / "smoke.csv").exists() and "intermediate_c" in r.stdout
    shapes = tmp_path / "shapes.txt"
    shapes.write_text("# smoke shapes\n1x256x256\n8x800x800\n")
    r = run("bench", "--shapes", shapes, "--reps", 5, "--eb-rows", 2000, "--out", tmp_path / "bench.csv")
    assert r.returncode == 0 and (tmp_path / "bench.csv").read_text().startswith("shape,baseline_ns")
    # eb-check: exit 0 on a clean table, 2 when a bag is flagged (stale row sum, validation skipped)
    from paper_2103_00130_b200 import embedding as E
    rng = np.random.default_rng(61)
    rows = rng.integers(-128, 128, (50, 8)).astype(np.int8)
    sums = rows.astype(np.int32).sum(axis=1)
    t = E.QuantEmbeddingTable(rows, np.full(50, 0.01, np.float32), np.full(50, 0.1, np.float32), row_sums=sums)
    E.save_table(t, str(tmp_path / "t.abeb"))
    (tmp_path / "bags.txt").write_text("0 1 2 3\n10 10 11\n4:0.5 5:1.5\n")
    r = run("eb-check", tmp_path / "t.abeb", tmp_path / "bags.txt")
    assert r.returncode == 0 and "0/3 bags flagged" in r.stdout
    sums[1] += 100
    t2 = E.QuantEmbeddingTable(rows, np.full(50, 0.01, np.float32), np.full(50, 0.1, np.float32), row_sums=sums)
    E.save_table(t2, str(tmp_path / "t2.abeb"))
    assert run("eb-check", tmp_path / "t2.abeb", tmp_path / "bags.txt").returncode == 1  # validation refuses
    r = run("eb-check", tmp_path / "t2.abeb", tmp_path / "bags.txt", "--skip-validation")
    assert r.returncode == 2 and "1/3 bags flagged" in r.stdout
