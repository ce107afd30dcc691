#!/usr/bin/env python3
"""Small profiling driver: one mesh, a few CG iterations in direct-launch mode (so ncu can
see every kernel), plus standalone nb_ax / nb_dssum launches.

    python tools/prof_cg.py --nel 16 16 16 --p 7 --policy mixed --iters 20
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_02134_b200 as nb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nel", type=int, nargs=3, default=[16, 16, 16])
ap.add_argument("--p", type=int, default=7)
ap.add_argument("--deform", type=float, default=0.0)
ap.add_argument("--policy", default="mixed", choices=["fp64", "fp32", "mixed"])
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--gs", default="consistent", choices=["consistent", "per_copy"])
ap.add_argument("--standalone", type=int, default=3)
a = ap.parse_args()
pol = {"fp64": nb.NB_FP64, "fp32": nb.NB_FP32, "mixed": nb.NB_MIXED}[a.policy]
order = nb.NB_GS_CONSISTENT if a.gs == "consistent" else nb.NB_GS_PER_COPY
m = nb.Mesh(*a.nel, a.p, deform=a.deform)
b = m.rhs(pol, seed=0)
x = m.empty(pol)
rep, _ = nb.nb_cg(m.h, b, x, pol, a.iters, 0.0, gs_order=order)
print(f"iters={rep.iterations} k1={1e3 * rep.k_ax_ms / rep.iterations:.2f}us gs={1e3 * rep.k_gs_ms / rep.iterations:.2f}us "
      f"k2={1e3 * rep.k_upd_ms / rep.iterations:.2f}us")
w = m.empty(pol)
for _ in range(a.standalone):
    nb.nb_ax(m.h, pol, b, w, nb.NB_AX_LOCAL)
    nb.nb_dssum(m.h, pol, order, w)
torch.cuda.synchronize()
m.close()
