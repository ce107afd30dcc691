#!/usr/bin/env python3
"""Time to tolerance, fp64 vs mixed (and fp32), for BASELINE.json configs[1..3] on one GPU:
median of --reps solves after a warm-up, 256 MiB L2 flush between solves.  One JSON line each.

    python tools/time_to_solution.py > profiles/r1_time_to_solution.jsonl
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_02134_b200 as nb  # noqa: E402

CASES = [("configs[1]", (16, 16, 16), 7, 0.0, nb.NB_RHS_UNIFORM, 1e-8, ("fp64", "fp32", "mixed")),
         ("configs[2]", (32, 32, 32), 9, 0.1, nb.NB_RHS_UNIFORM, 1e-8, ("fp64", "mixed")),
         ("configs[3]", (64, 32, 32), 11, 0.0, nb.NB_RHS_MANUFACTURED, 1e-10, ("fp64", "mixed"))]
POL = {"fp64": nb.NB_FP64, "fp32": nb.NB_FP32, "mixed": nb.NB_MIXED}

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for name, nel, p, d, kind, rtol, pols in CASES:
    m = nb.Mesh(*nel, p, deform=d, seed=0)
    for pol in pols:
        b = m.rhs(POL[pol], kind, noise=1e-3, seed=0)
        m.cg(b, POL[pol], max_iter=8000, rtol=rtol)
        runs = []
        for _ in range(a.reps):
            flush.zero_()
            _, r = m.cg(b, POL[pol], max_iter=8000, rtol=rtol)
            runs.append(r)
        t = statistics.median(r.solve_ms for r in runs)
        print(json.dumps({"config": name, "policy": pol, "rtol": rtol, "n_local": m.n_local,
                          "iterations": runs[-1].iterations, "status": runs[-1].status, "time_ms": t,
                          "dof_iter_per_s": m.n_local * runs[-1].iterations / (t * 1e-3)}), flush=True)
        del b
    m.close()
