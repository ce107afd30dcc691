#!/usr/bin/env python3
"""fp32 vs fp32+Dot2 vs mixed at full size (BASELINE.json configs[2], configs[3]; consistent and
per-copy GS orders): does compensating the dot products let single precision reach the tolerance?
("only marginal improvement".)  One JSON line per run.

    python tools/dot2_full_size.py > profiles/r1_dot2_full_size.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_02134_b200 as nb  # noqa: E402

CASES = [("configs[2]", (32, 32, 32), 9, 0.1, nb.NB_RHS_UNIFORM, 1e-8),
         ("configs[3]", (64, 32, 32), 11, 0.0, nb.NB_RHS_MANUFACTURED, 1e-10)]
for name, nel, p, d, kind, rtol in CASES:
    m = nb.Mesh(*nel, p, deform=d, seed=0)
    for order_name, order in (("consistent", nb.NB_GS_CONSISTENT), ("per_copy", nb.NB_GS_PER_COPY)):
        for pol_name, pol in (("fp32", nb.NB_FP32), ("fp32_dot2", nb.NB_FP32_DOT2), ("mixed", nb.NB_MIXED)):
            b = m.rhs(pol, kind, noise=1e-3, seed=0)
            _, r = m.cg(b, pol, max_iter=6000, rtol=rtol, gs_order=order)
            st = {nb.NB_CONVERGED: "converged", nb.NB_MAXITER: "max_iter", nb.NB_STAGNATED: "stagnated",
                  nb.NB_BROKEDOWN: "breakdown"}[r.status]
            print(json.dumps({"config": name, "gs_order": order_name, "policy": pol_name, "rtol": rtol,
                              "status": st, "iterations": r.iterations, "rel_res_min": r.rel_res_min,
                              "rel_res_final": r.rel_res_final, "time_ms": r.solve_ms}), flush=True)
            del b
    m.close()
