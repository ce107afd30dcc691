#!/usr/bin/env python3
"""The paper's closest workload to this path: Neko's Poisson example, E = 16384
elements (32x32x16), N = 7, CG with the Jacobi and the identity preconditioners, fp64 vs mixed
(fp64 GS and dots), tolerance 1e-9.  Time to tolerance on one B200,
median of --reps solves after a warm-up; one JSON line per (preconditioner, policy).

    python tools/neko_shape.py [--reps 5] > profiles/r1_neko_shape.jsonl
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_02134_b200 as nb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--rtol", type=float, default=1e-9)
a = ap.parse_args()
m = nb.Mesh(32, 32, 16, 7)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for pc_name, pc in (("jacobi", nb.NB_PC_JACOBI), ("identity", nb.NB_PC_IDENTITY)):
    res = {}
    for pol_name, pol in (("fp64", nb.NB_FP64), ("mixed", nb.NB_MIXED), ("fp32", nb.NB_FP32)):
        b = m.rhs(pol, seed=0)
        m.cg(b, pol, max_iter=20000, rtol=a.rtol, precond=pc)
        runs = []
        for _ in range(a.reps):
            flush.zero_()
            _, r = m.cg(b, pol, max_iter=20000, rtol=a.rtol, precond=pc)
            runs.append(r)
        t = statistics.median(r.solve_ms for r in runs)
        res[pol_name] = {"iterations": runs[-1].iterations, "status": runs[-1].status, "time_ms": t,
                         "rel_res_min": runs[-1].rel_res_min}
        print(json.dumps({"workload": "Neko Poisson shape E=16384 (32x32x16), N=7, uniform RHS seed 0",
                          "precond": pc_name, "policy": pol_name, "rtol": a.rtol, **res[pol_name]}), flush=True)
    gain = (res["fp64"]["time_ms"] - res["mixed"]["time_ms"]) / res["fp64"]["time_ms"]
    print(json.dumps({"precond": pc_name, "gain_mixed_vs_fp64": gain,
                      "speedup_fp64_over_mixed": res["fp64"]["time_ms"] / res["mixed"]["time_ms"]}), flush=True)
m.close()
