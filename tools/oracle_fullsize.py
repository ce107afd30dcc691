"""Full-size oracle goldens for configs[2] and configs[3] (CPU only; calls nothing but oracle/).

Runs the plain-C oracle (oracle/nb_oracle.c, single thread) to convergence on the full
BASELINE.json configurations and writes compact fixtures under tests/golden/ that the GPU
parity tests compare against (tests/test_gpu_fullsize.py):

  configs[2]: 32x32x32 elements, p = 9, deformed (amp 0.1, seed 0), uniform RHS seed 0, rtol 1e-8
  configs[3]: 64x32x32 elements, p = 11, manufactured RHS + 1e-3 noise (seed 0), rtol 1e-10

Each run stores: iterations, status, rtr0, final / minimum relative residual, the fp64 true
residual (C-14), the full relative-residual history, the first 64 iterations' scalar recurrence
(rho, alpha, beta), the c-norm of x and a strided sample of x (every STRIDE-th local DOF, STRIDE a
prime so the sample visits every in-element position).  The full x is kept under --scratch so a
final `--gaps` pass can compute the method floor ||x_a - x_b||_c / ||x_b||_c between policies
 over the whole vector.

Usage (one run per process; they are independent and can run side by side):
  python tools/oracle_fullsize.py --config 2 --policy fp64
  python tools/oracle_fullsize.py --config 2 --policy mixed
  python tools/oracle_fullsize.py --config 2 --policy mixed_x64
  python tools/oracle_fullsize.py --gaps --config 2
  python tools/oracle_fullsize.py --config 2 --policy sw_mixed      # Schwarz PCG (NEXT-4)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

CONFIGS = {
    2: dict(nel=(32, 32, 32), p=9, deform=0.1, rhs=oracle.RHS_UNIFORM, rtol=1e-8, stride=4001,
            desc="BASELINE.json configs[2]: 32^3 deformed, p=9, uniform RHS seed 0, rtol 1e-8"),
    3: dict(nel=(64, 32, 32), p=11, deform=0.0, rhs=oracle.RHS_MANUFACTURED, rtol=1e-10, stride=12007,
            desc="BASELINE.json configs[3]: 64x32x32, p=11, manufactured RHS + 1e-3 noise seed 0, rtol 1e-10"),
}
POLICIES = {"fp64": (oracle.FP64, False), "mixed": (oracle.MIXED, False), "mixed_x64": (oracle.MIXED, True),
            "sw_fp64": (oracle.FP64, False), "sw_mixed": (oracle.MIXED, False)}   # sw_*: NEXT-4 Schwarz PCG
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(HERE, "tests", "golden")


def golden_path(cfg: int, pol: str) -> str:
    return os.path.join(GOLDEN, f"fullsize_configs{cfg}_{pol}.json")


def run(cfg: int, pol: str, scratch: str, max_iter: int) -> None:
    c = CONFIGS[cfg]
    policy, x64 = POLICIES[pol]
    t0 = time.time()
    m = oracle.Mesh(*c["nel"], c["p"], c["deform"], 0)
    b = m.rhs(c["rhs"], 1e-3, 0)
    t1 = time.time()
    pc = oracle.PC_SCHWARZ if pol.startswith("sw_") else oracle.PC_JACOBI
    x, hist, rep, sc = m.cg(b, policy, max_iter=max_iter, rtol=c["rtol"], x64=x64, scalars=True, precond=pc)
    t2 = time.time()
    cw = m.geom()["c"]
    xnorm = float(np.sqrt(np.sum(cw * x * x)))
    os.makedirs(scratch, exist_ok=True)
    np.save(os.path.join(scratch, f"x_configs{cfg}_{pol}.npy"), x)
    idx = np.arange(0, m.n_local, c["stride"], dtype=np.int64)
    out = dict(
        source="tools/oracle_fullsize.py (oracle/ only; plain C, one thread, -O2 -ffp-contract=off)",
        config=c["desc"], nel=list(c["nel"]), p=c["p"], deform=c["deform"], rhs=c["rhs"], seed=0,
        rtol=c["rtol"], policy=pol, x_fp64=x64, precond="schwarz" if pc == oracle.PC_SCHWARZ else "jacobi",
        n_local=m.n_local,
        iterations=rep.iterations, status=rep.status, rtr0=rep.rtr0, rel_res_final=rep.rel_res_final,
        rel_res_min=rep.rel_res_min, true_res=rep.true_res,
        history=[float(v) for v in hist],
        scalars_first64=[[float(v) for v in row] for row in sc[:64]],
        x_cnorm=xnorm, sample_stride=c["stride"], sample_n=int(idx.size),
        x_sample=[float(v) for v in x[idx]],
        setup_s=t1 - t0, solve_s=t2 - t1, host_threads=1,
    )
    os.makedirs(GOLDEN, exist_ok=True)
    with open(golden_path(cfg, pol), "w") as f:
        json.dump(out, f, indent=0)
    print(json.dumps({k: out[k] for k in ("policy", "iterations", "status", "rel_res_final", "true_res",
                                          "x_cnorm", "solve_s")}))


def gaps(cfg: int, scratch: str) -> None:
    c = CONFIGS[cfg]
    m = oracle.Mesh(*c["nel"], c["p"], c["deform"], 0)
    cw = m.geom()["c"]
    xs = {}
    for pol in POLICIES:
        if pol.startswith("sw_"):
            continue
        f = os.path.join(scratch, f"x_configs{cfg}_{pol}.npy")
        if os.path.exists(f):
            xs[pol] = np.load(f)
    ref = xs["fp64"]
    den = float(np.sqrt(np.sum(cw * ref * ref)))
    res = {}
    for pol, x in xs.items():
        if pol == "fp64":
            continue
        d = x - ref
        res[f"{pol}_vs_fp64"] = float(np.sqrt(np.sum(cw * d * d))) / den
    path = os.path.join(GOLDEN, f"fullsize_configs{cfg}_gaps.json")
    with open(path, "w") as f:
        json.dump(dict(source="tools/oracle_fullsize.py --gaps (oracle/ only)", config=c["desc"],
                       norm="c-weighted L2 over all local DOF (= global L2 on unique nodes), SURVEY.md C-15",
                       method_floor=res), f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, choices=sorted(CONFIGS), required=True)
    ap.add_argument("--policy", choices=sorted(POLICIES))
    ap.add_argument("--gaps", action="store_true")
    ap.add_argument("--scratch", default="/tmp/nb_fullsize")
    ap.add_argument("--max-iter", type=int, default=8000)
    a = ap.parse_args()
    if a.gaps:
        gaps(a.config, a.scratch)
    else:
        run(a.config, a.policy, a.scratch, a.max_iter)
