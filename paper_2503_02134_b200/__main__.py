"""Command line: one Jacobi-PCG solve on the GPU, JSON report on stdout.

    python -m paper_2503_02134_b200 solve --nel 16 16 16 --p 7 --policy mixed --rtol 1e-8
    python -m paper_2503_02134_b200 solve --nel 16 16 16 --p 7 --policy fp32 --gs-order per_copy

Exit codes follow SPEC.md's CLI contract (External Interfaces): 0 converged (or a fixed-iteration
run that finished), 1 usage / setup error, 2 stagnated, 3 numeric breakdown.
Every step runs in the CUDA library through include/nb.h; there is no CPU path.
"""
from __future__ import annotations

import argparse
import json
import sys

POLICIES = {"fp64": 0, "fp32": 1, "mixed": 2, "fp32_dot2": 3}
ORDERS = {"consistent": 0, "per_copy": 1}
PRECONDS = {"jacobi": 0, "identity": 1, "jacobi_f32": 2}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2503_02134_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="Jacobi-PCG solve of the SEM Poisson problem on a box")
    s.add_argument("--nel", type=int, nargs=3, default=[16, 16, 16], metavar=("NX", "NY", "NZ"))
    s.add_argument("--p", type=int, default=7, help="polynomial order (1..15)")
    s.add_argument("--deform", type=float, default=0.0, help="vertex deformation amplitude / element size")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--policy", choices=list(POLICIES), default="mixed")
    s.add_argument("--rtol", type=float, default=1e-8, help="0: run exactly --max-iter iterations")
    s.add_argument("--max-iter", type=int, default=4000)
    s.add_argument("--gs-order", choices=list(ORDERS), default="consistent")
    s.add_argument("--rhs", choices=["uniform", "manufactured"], default="uniform")
    s.add_argument("--noise", type=float, default=1e-3)
    s.add_argument("--precond", choices=list(PRECONDS), default="jacobi")
    s.add_argument("--x64", action="store_true", help="mixed policy: accumulate x in fp64")
    s.add_argument("--slabs", type=int, default=1,
                   help="split the box into this many z-slabs solved together in one launch (multi-rank path)")
    s.add_argument("--history", action="store_true", help="include the residual history")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 1 if e.code else 0
    import paper_2503_02134_b200 as nb
    pol = POLICIES[a.policy]
    kind = nb.NB_RHS_UNIFORM if a.rhs == "uniform" else nb.NB_RHS_MANUFACTURED
    try:
        if a.slabs > 1:
            meshes = [nb.Mesh(*a.nel, a.p, deform=a.deform, seed=a.seed, slab=nb.slab_bounds(a.nel[2], a.slabs, r))
                      for r in range(a.slabs)]
        else:
            meshes = [nb.Mesh(*a.nel, a.p, deform=a.deform, seed=a.seed)]
        bs = [m.rhs(pol, kind, noise=a.noise, seed=a.seed) for m in meshes]
        if a.slabs > 1:
            if a.gs_order != "consistent":
                raise ValueError("--slabs needs --gs-order consistent")
            _, rs = nb.cg_group(meshes, bs, pol, max_iter=a.max_iter, rtol=a.rtol, precond=PRECONDS[a.precond],
                                x64=a.x64)
            r = rs[0]
        else:
            _, r = meshes[0].cg(bs[0], pol, max_iter=a.max_iter, rtol=a.rtol, gs_order=ORDERS[a.gs_order],
                                precond=PRECONDS[a.precond], x64=a.x64)
    except (nb.NbError, ValueError) as e:
        print(json.dumps({"error": str(e)}), file=sys.stderr)
        return 1
    n_local = sum(m.n_local for m in meshes)
    status = {nb.NB_CONVERGED: "converged", nb.NB_MAXITER: "max_iter", nb.NB_STAGNATED: "stagnated",
              nb.NB_BROKEDOWN: "breakdown"}[r.status]
    out = {"schema": "nb-run-report/1", "nel": a.nel, "p": a.p, "deform": a.deform, "policy": a.policy,
           "gs_order": a.gs_order, "precond": a.precond, "x64": a.x64, "slabs": a.slabs, "rhs": a.rhs,
           "n_local": n_local, "iterations": r.iterations,
           "status": status, "rel_res_final": r.rel_res_final, "rel_res_min": r.rel_res_min,
           "solve_ms": r.solve_ms, "dof_iter_per_s": n_local * r.iterations / (r.solve_ms * 1e-3)
           if r.solve_ms > 0 else None}
    if a.history:
        out["history"] = [float(v) for v in r.history]
    print(json.dumps(out))
    for m in meshes:
        m.close()
    if r.status == nb.NB_STAGNATED:
        return 2
    if r.status == nb.NB_BROKEDOWN:
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
