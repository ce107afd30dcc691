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


def test_gpus2_spawns_two_ranks_dry_run():
    """--gpus N without a torchrun environment relaunches itself with N ranks (127.0.0.1
    rendezvous); N > 1 defaults to the z-slab decomposition.  --dry-run: gloo plumbing only."""
    env_clean = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env_clean)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["mode"] == "slab" and "z-slabs over 2 GPUs" in d["parallelism"]


def test_survey_bytes_and_ae_mae():
    sys.path.insert(0, ROOT)
    import bench

    class Info:
        n_local, n_shared_copies, n_shared_global = 2097152, 1155960, 501705   # configs[1], SURVEY §8(a)

    got = [round(bench.survey_bytes(p, Info), 1) for p in (0, 2, 1)]
    assert got == [165.9, 92.5, 84.5]
    assert bench.impl_bytes(0) == 136 and bench.impl_bytes(2) == 72 and bench.impl_bytes(1) == 68
    d = bench.ae_mae([1.0, 0.5, 0.25, 0.1], [1.0, 0.5, 0.2, 0.1, 0.05])
    assert d["iterations_compared"] == 3 and abs(d["MAE"] - 0.05 / 3) < 1e-12 and abs(d["AE_max"] - 0.05) < 1e-12
