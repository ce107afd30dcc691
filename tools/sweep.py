#!/usr/bin/env python3
"""Throughput sweep (BASELINE.json configs[4] style): fixed-iteration CG solves (rtol = 0) on
cube / box meshes, every policy; prints one JSON line per point with DOF*iter/s and the
per-phase device times (block-0 globaltimer stamps of the megakernel, or CUDA events of the
graph driver's kernels) and their algorithmic HBM bandwidth.

    python tools/sweep.py --cases 16x16x16p7 32x32x32p7 --iters 200 [--policies mixed fp64]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_02134_b200 as nb  # noqa: E402

SV = {0: 8, 1: 4, 2: 4, 3: 4}
SJ = {0: 8, 1: 4, 2: 8, 3: 4}
POL = {"fp64": nb.NB_FP64, "fp32": nb.NB_FP32, "mixed": nb.NB_MIXED, "fp32_dot2": nb.NB_FP32_DOT2}


def parse(c):
    d = 0.0
    if c.endswith("d"):
        c, d = c[:-1], 0.1
    dims, p = c.split("p")
    return [int(v) for v in dims.split("x")], int(p), d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", nargs="+", default=["16x16x16p7"])
    ap.add_argument("--policies", nargs="+", default=["fp64", "fp32", "mixed"])
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--standalone", action="store_true", help="also time nb_ax (local) and nb_dssum")
    ap.add_argument("--configs4", action="store_true", help="BASELINE configs[4]: cubes 10..50, p 7/9/11, "
                    "undeformed and deformed")
    a = ap.parse_args()
    if a.configs4:
        a.cases = [f"{s}x{s}x{s}p{p}{d}" for p in (7, 9, 11) for s in (10, 13, 16, 20, 25, 32, 40, 50)
                   for d in ("", "d")]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for c in a.cases:
        nel, p, d = parse(c)
        m = nb.Mesh(*nel, p, deform=d)
        NL = m.n_local
        for name in a.policies:
            pol = POL[name]
            b = m.rhs(pol, seed=0)
            x = m.empty(pol)
            nb.nb_cg(m.h, b, x, pol, a.iters, 0.0, history=False)          # warm-up
            best = None
            for _ in range(a.reps):
                flush.zero_()
                rep, _ = nb.nb_cg(m.h, b, x, pol, a.iters, 0.0, history=False)
                if best is None or rep.solve_ms < best.solve_ms:
                    best = rep
            it = best.iterations
            k1 = 1e3 * best.k_ax_ms / it
            k2 = 1e3 * best.k_upd_ms / it
            kg = 1e3 * best.k_gs_ms / it
            b1 = (12 * SV[pol]) * NL
            b2 = (4 * SV[pol] + SJ[pol]) * NL
            extra = {}
            if a.standalone:
                st = torch.cuda.current_stream()
                wv = m.empty(pol)
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                for what in ("ax", "dssum"):
                    fn = (lambda: nb.nb_ax(m.h, pol, b, wv, nb.NB_AX_LOCAL)) if what == "ax" else \
                         (lambda: nb.nb_dssum(m.h, pol, nb.NB_GS_CONSISTENT, wv))
                    fn()
                    ev0.record(st)
                    for _ in range(10):
                        fn()
                    ev1.record(st)
                    ev1.synchronize()
                    us = 1e3 * ev0.elapsed_time(ev1) / 10
                    byts = (8 * SV[pol]) * NL if what == "ax" else \
                        m.info.n_shared_copies * (2 * SV[pol] + 4) + (m.info.n_shared_global + 1) * 4
                    extra[what + "_us"] = us
                    extra[what + "_GBps"] = byts / (us * 1e-6) / 1e9
            print(json.dumps({**extra, "case": c, "policy": name, "n_local": NL, "iters": it, "solve_ms": best.solve_ms,
                              "dof_iter_per_s": NL * it / (best.solve_ms * 1e-3),
                              "us_per_iter": 1e3 * best.solve_ms / it, "phaseA_us": k1, "phaseS_us": kg,
                              "phaseB_us": k2, "A_GBps": b1 / (k1 * 1e-6) / 1e9 if k1 else None,
                              "B_GBps": b2 / (k2 * 1e-6) / 1e9 if k2 else None}), flush=True)
        m.close()


if __name__ == "__main__":
    main()
