"""bench.py contract legs that run without a GPU: the reference arm (--impl reference: the CPU
oracle on bounded samples of the same workload) and --oracle-timing (per-config oracle timing)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout


def test_reference_arm_json_line():
    lines = [l for l in run("--impl", "reference", "--steps", "1", "--warmup", "3").splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_oracle_timing_small():
    d = json.loads(run("--oracle-timing", "--oracle-max-dof", "5000"))
    assert d["host"]["threads_used"] == 1 and d["host"]["nproc"] >= 1
    (c,) = d["cases"]
    assert c["config"] == "configs[0]" and c["n_local"] == 4096
    assert c["solve_fp64"]["iterations"] == 100 and c["solve_fp64"]["dof_iter_per_s"] > 0
