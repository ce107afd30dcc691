#!/usr/bin/env python3
"""Jacobi vs two-level Schwarz PCG (NB_PC_SCHWARZ) to a tolerance:
iterations, time to solution, per-iteration time and its phases (A: p update + Ax, B: gather +
r update, S: solveM), per policy.  Median of --reps after one warm-up; L2 flushed between runs.

    python tools/schwarz_bench.py --cases 16x16x16p7 32x32x32p9d --policies fp64 mixed fp32
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_02134_b200 as nb  # noqa: E402

POL = {"fp64": nb.NB_FP64, "fp32": nb.NB_FP32, "mixed": nb.NB_MIXED, "fp32_dot2": nb.NB_FP32_DOT2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", nargs="+", default=["16x16x16p7"])
    ap.add_argument("--policies", nargs="+", default=["fp64", "mixed"])
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--apply", action="store_true", help="time solveM alone (nb_precond_apply), L2 flushed per call")
    a = ap.parse_args()
    if a.apply:
        return apply_only(a)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for c in a.cases:
        d = 0.1 if c.endswith("d") else 0.0
        dims, p = c.rstrip("d").split("p")
        m = nb.Mesh(*[int(v) for v in dims.split("x")], int(p), deform=d)
        for name in a.policies:
            pol = POL[name]
            b = m.rhs(pol, seed=0)
            for pc, pcn in ((nb.NB_PC_JACOBI, "jacobi"), (nb.NB_PC_SCHWARZ, "schwarz")):
                m.cg(b, pol, max_iter=20000, rtol=a.rtol, precond=pc)   # warm-up (+ table setup)
                runs = []
                for _ in range(a.reps):
                    flush.zero_()
                    _, r = m.cg(b, pol, max_iter=20000, rtol=a.rtol, precond=pc)
                    runs.append(r)
                r = sorted(runs, key=lambda t: t.solve_ms)[len(runs) // 2]
                it = max(r.iterations, 1)
                print(json.dumps({"case": c, "policy": name, "precond": pcn, "iterations": r.iterations,
                                  "status": r.status, "time_ms": r.solve_ms, "us_per_iter": 1e3 * r.solve_ms / it,
                                  "phaseA_us": 1e3 * r.k_ax_ms / it, "phaseB_us": 1e3 * r.k_upd_ms / it,
                                  "solveM_us": 1e3 * r.k_gs_ms / it, "rel_res": r.rel_res_final,
                                  "n_local": m.n_local}), flush=True)
        m.close()


def apply_only(a):
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for c in a.cases:
        d = 0.1 if c.endswith("d") else 0.0
        dims, p = c.rstrip("d").split("p")
        m = nb.Mesh(*[int(v) for v in dims.split("x")], int(p), deform=d)
        for name in a.policies:
            pol = POL[name]
            r = m.rhs(pol, seed=0)
            z = m.precond(r, pol)
            ts = []
            for _ in range(max(a.reps, 3)):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                nb.nb_precond_apply(m.h, pol, nb.NB_PC_SCHWARZ, r, z)
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            us = 1e3 * statistics.median(ts)
            print(json.dumps({"case": c, "policy": name, "apply_us": us, "ns_per_dof": 1e3 * us / m.n_local,
                              "n_local": m.n_local}), flush=True)
        m.close()


if __name__ == "__main__":
    main()
