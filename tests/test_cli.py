"""CLI (row f3) and bench harness (row f4): real subprocesses, reference exit codes,
file formats; GPU legs reproduce the reference's tiny reconstruction bit for bit."""

import csv
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import load_golden

REPO = Path(__file__).resolve().parents[1]


def run_cli(*args, cwd=None):
    env = dict(os.environ)
    env["PYTHONPATH"] = str(REPO) + os.pathsep + env.get("PYTHONPATH", "")
    return subprocess.run([sys.executable, "-m", "paper_2104_13248_b200.cli", *map(str, args)], capture_output=True,
                          text=True, cwd=cwd, env=env, timeout=600)


def test_count_ops_output():
    r = run_cli("count-ops", "--variant", "baseline", "--nx", 8, "--ny", 8, "--nz", 8, "--np", 4)
    assert r.returncode == 0, r.stderr
    assert "dot_ops 6144" in r.stdout


def test_usage_errors_exit_2(tmp_path):
    r = run_cli("count-ops", "--variant", "symmetry", "--nx", 8, "--ny", 8, "--nz", 7, "--np", 4)
    assert r.returncode == 2 and "even nz" in r.stderr
    r = run_cli("backproject", "--in", tmp_path / "missing", "--variant", "baseline", "--out", tmp_path / "v.raw")
    assert r.returncode == 2 and "input file not found" in r.stderr
    r = run_cli("verify", "--a", tmp_path / "a.raw", "--b", tmp_path / "b.raw")
    assert r.returncode == 2


def test_verify_pass_and_fail(tmp_path):
    from paper_2104_13248_b200.tensors import Volume, save_volume

    a = np.zeros((4, 4, 4), np.float32)
    save_volume(tmp_path / "a.raw", Volume.from_array(a))
    save_volume(tmp_path / "b.raw", Volume.from_array(a + 1e-7))
    save_volume(tmp_path / "c.raw", Volume.from_array(a + 1.0))
    assert run_cli("verify", "--a", tmp_path / "a.raw", "--b", tmp_path / "b.raw").returncode == 0
    r = run_cli("verify", "--a", tmp_path / "a.raw", "--b", tmp_path / "c.raw")
    assert r.returncode == 1 and "FAIL" in r.stdout


@pytest.mark.gpu
def test_gen_data_backproject_pipeline_bitwise(tmp_path):
    from paper_2104_13248_b200.geometry import build_geometry, save_geometry
    from paper_2104_13248_b200.tensors import load_projections, load_volume

    save_geometry(tmp_path / "g.json", build_geometry(nx=12, ny=12, nz=12, nw=24, nh=24, np=8))
    r = run_cli("gen-data", "--geometry", tmp_path / "g.json", "--out", tmp_path / "data")
    assert r.returncode == 0, r.stderr
    g = load_golden("tiny")
    assert load_projections(tmp_path / "data" / "projections.raw").data.tobytes() == g["img"].tobytes()
    r = run_cli("backproject", "--in", tmp_path / "data", "--variant", "baseline", "--out", tmp_path / "base.raw")
    assert r.returncode == 0, r.stderr
    assert load_volume(tmp_path / "base.raw").data.tobytes() == g["baseline"].tobytes()
    r = run_cli("backproject", "--in", tmp_path / "data", "--variant", "subline_prefetch", "--nb", 2,
                "--out", tmp_path / "sp.raw")
    assert r.returncode == 0, r.stderr
    sp = g["subline_prefetch"].transpose(2, 1, 0)
    assert load_volume(tmp_path / "sp.raw").data.tobytes() == np.ascontiguousarray(sp).tobytes()
    assert run_cli("verify", "--a", tmp_path / "base.raw", "--b", tmp_path / "sp.raw").returncode == 0


@pytest.mark.gpu
def test_bench_harness_reports(tmp_path):
    r = run_cli("bench", "--problem", "D1", "--variants", "baseline,subline_prefetch", "--nb", 32, "--repeats", 2,
                "--out", tmp_path / "r.csv", "--json", tmp_path / "r.json", "--verify")
    assert r.returncode == 0, r.stdout + r.stderr
    rows = list(csv.DictReader(open(tmp_path / "r.csv")))
    assert [x["variant"] for x in rows] == ["baseline", "subline_prefetch"]
    assert all(float(x["gups"]) > 0 and x["gpus"] == "1" for x in rows)
    doc = json.loads((tmp_path / "r.json").read_text())
    assert doc[0]["schema_version"] == 1 and doc[0]["dot_ops"] == 3 * 64 ** 3 * 128
