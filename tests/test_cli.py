"""CLI exit codes (SPEC.md External Interfaces: 0 converged, 1 usage/config, 2 stagnated, 3 breakdown)."""
import json
import subprocess
import sys
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2503_02134_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_usage_error_is_1():
    assert run("solve", "--policy", "fp16").returncode == 1
    assert run("nosuchcommand").returncode == 1


@pytest.mark.gpu
def test_converged_is_0():
    r = run("solve", "--nel", "4", "4", "4", "--p", "7", "--policy", "mixed")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["status"] == "converged" and rep["rel_res_final"] <= 1e-8


@pytest.mark.gpu
def test_bad_order_is_1():
    assert run("solve", "--nel", "2", "2", "2", "--p", "20").returncode == 1


@pytest.mark.gpu
def test_per_copy_fp32_failure_exit_codes():
    """fp32 with the per-copy GS order fails (the paper's stagnation); which of the two failure
    modes ends the run -- C-11 stagnation (exit 2) or the residual blowing up into a pap <= 0
    breakdown (exit 3) -- depends on rounding order.  The exit code must match the status."""
    r = run("solve", "--nel", "8", "8", "8", "--p", "7", "--policy", "fp32", "--gs-order", "per_copy",
            "--max-iter", "1200")
    st = json.loads(r.stdout)["status"]
    assert (r.returncode, st) in ((2, "stagnated"), (3, "breakdown")), r.stdout
    assert json.loads(r.stdout)["rel_res_min"] > 1e-8


@pytest.mark.gpu
def test_variants_and_slabs_from_cli():
    r = run("solve", "--nel", "6", "6", "6", "--p", "5", "--policy", "mixed", "--precond", "identity", "--x64",
            "--slabs", "3")
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    assert out["status"] == "converged" and out["slabs"] == 3 and out["precond"] == "identity"
    r1 = run("solve", "--nel", "6", "6", "6", "--p", "5", "--policy", "mixed", "--precond", "identity")
    assert abs(json.loads(r1.stdout)["iterations"] - out["iterations"]) <= 2


@pytest.mark.gpu
def test_slabs_need_consistent_order():
    r = run("solve", "--nel", "4", "4", "4", "--slabs", "2", "--gs-order", "per_copy")
    assert r.returncode == 1
