"""The reference-compatible CLI verbs (cli.cpp:532-780): config parsing,
validation messages and exit codes on CPU; solve / compare / sweep / generate
/ decompose end to end on the GPU (outputs against the library API)."""
import csv
import json
import os
import subprocess
import sys

import pytest

from paper_2311_15393_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2311_15393_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_apply_key_and_config_file(tmp_path):
    cfg = cli.ExperimentConfig()
    f = tmp_path / "c.cfg"
    f.write_text("# comment\nn = 48\nnoise=0.02  # trailing\nsolver= fpcg\nsweep_values = 1, 2,3\n\n")
    cli.load_config_file(cfg, str(f))
    assert (cfg.n, cfg.noise, cfg.solver, cfg.sweep_values) == (48, 0.02, "fpcg", ["1", "2", "3"])
    cli.apply_key(cfg, "precond_lambda", "0.5")
    assert cfg.precond_lambda == 0.5
    with pytest.raises(cli.ConfigError, match='config key n: cannot parse "x" as an integer'):
        cli.apply_key(cfg, "n", "x")
    with pytest.raises(cli.ConfigError, match="unknown config key: bogus"):
        cli.apply_key(cfg, "bogus", "1")
    with pytest.raises(cli.ConfigError, match="a nonnegative integer"):
        cli.apply_key(cfg, "seed", "-1")
    with pytest.raises(cli.ConfigError, match="a finite number"):
        cli.apply_key(cfg, "tol", "inf")
    with pytest.raises(cli.ConfigError, match="empty item"):
        cli.apply_key(cfg, "sweep_values", "1,,2")
    bad = tmp_path / "bad.cfg"
    bad.write_text("n 3\n")
    with pytest.raises(cli.ConfigError, match="bad.cfg:1: expected key=value"):
        cli.load_config_file(cli.ExperimentConfig(), str(bad))


@pytest.mark.parametrize("key,value,msg", [
    ("solver", "gmres", "config key solver: unknown solver gmres"),
    ("param", "lcurve", "config key param: unknown method lcurve"),
    ("n", "1", "config key n: need n >= 2"),
    ("psf_size", "8", "config key psf_size: need a positive odd size"),
    ("psf_size", "65", "config key psf_size: PSF larger than the image"),
    ("maxit", "0", "config key maxit: must be >= 1"),
    ("tol", "0", "config key tol: must be > 0"),
    ("fmt", "fp8", "config key fmt"),
])
def test_validate_messages(key, value, msg):
    cfg = cli.ExperimentConfig()
    cli.apply_key(cfg, key, value)
    with pytest.raises(cli.ConfigError, match=msg):
        cli.validate(cfg)


def test_exit_codes_without_gpu(tmp_path):
    r = run_cli("solve", "--solver", "gmres", "--out", str(tmp_path / "o"))
    assert r.returncode == 2 and "config error: config key solver" in r.stderr
    r = run_cli("solve", "--config", str(tmp_path / "missing.cfg"))
    assert r.returncode == 3 and "io error: cannot read config file" in r.stderr
    r = run_cli("sweep", "--out", str(tmp_path / "s"))
    assert r.returncode == 2 and "sweep needs sweep_key" in r.stderr


@pytest.mark.gpu
def test_solve_and_compare_verbs(tmp_path):
    out = tmp_path / "solve"
    r = run_cli("solve", "--n", "64", "--param", "gcv", "--solver", "pcg", "--tol", "1e-6", "--out", str(out))
    assert r.returncode == 0, r.stderr
    s = json.load(open(out / "summary.json"))
    assert s["schema"] == "kronprec.summary/1" and s["selection"]["method"] == "gcv"
    # the same pipeline through the library API
    cfg = cli.ExperimentConfig()
    for k, v in (("n", "64"), ("param", "gcv"), ("tol", "1e-6")):
        cli.apply_key(cfg, k, v)
    oc = cli.run_single(cfg)
    assert s["selection"]["lambda"] == oc["selection"].lambda_
    assert s["solver"]["iterations"] == oc["result"].history.iterations_used
    assert s["solver"]["final_relative_error"] == oc["final_relative_error"]
    rows = list(csv.reader(open(out / "convergence.csv", newline="")))
    assert rows[0] == ["schema", "iteration", "relative_error", "residual_norm", "cumulative_work_units"]
    assert len(rows) == 1 + len(oc["result"].history.residual_norm)
    assert open(out / "reconstruction.pgm", "rb").read(2) == b"P5"
    assert f"iterations={oc['result'].history.iterations_used}" in r.stdout
    cmp_out = tmp_path / "cmp"
    r = run_cli("compare", "--n", "64", "--param", "discrepancy", "--eta", "1.01", "--include-fpcg",
                "--out", str(cmp_out))
    assert r.returncode == 0, r.stderr
    w = json.load(open(cmp_out / "work_report.json"))
    assert w["schema"] == "kronprec.work_report/1"
    assert {"baseline", "precond", "flexible", "m_baseline", "m_precond"} <= set(w)
    hdr = next(csv.reader(open(cmp_out / "comparison.csv", newline="")))
    assert hdr[-3:] == ["fpcg_relative_error", "fpcg_residual_norm", "fpcg_work_units"]


@pytest.mark.gpu
def test_sweep_generate_decompose_verbs(tmp_path):
    out = tmp_path / "sw"
    r = run_cli("sweep", "--n", "48", "--param", "fixed", "--lambda", "0.05", "--sweep-key", "noise",
                "--sweep-values", "0.001,0.01", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(open(out / "sweep.csv", newline="")))
    assert [row[1] for row in rows[1:]] == ["0.001", "0.01"] and all(row[5] == "ok" for row in rows[1:])
    assert (out / "run_1" / "summary.json").exists()
    g = tmp_path / "gen"
    r = run_cli("generate", "--n", "32", "--out", str(g))
    assert r.returncode == 0 and (g / "meta.json").exists() and (g / "b.pgm").exists()
    d = tmp_path / "dec"
    r = run_cli("decompose", "--n", "32", "--blur", "shake", "--out", str(d))
    assert r.returncode == 0, r.stderr
    j = json.load(open(d / "decompose.json"))
    assert j["schema"] == "kronprec.decompose/1" and j["terms"] >= 1
    assert 0.0 <= j["rel_error"] <= 1.0 and j["rel_error_rounded"] >= j["rel_error"] - 1e-3
