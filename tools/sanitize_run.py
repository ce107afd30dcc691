#!/usr/bin/env python3
"""Small workload touching every kernel of the library, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_02134_b200 as nb  # noqa: E402

for (nel, p, d) in [((2, 2, 2), 7, 0.0), ((3, 2, 2), 4, 0.1)]:
    m = nb.Mesh(*nel, p, deform=d, seed=1)
    for pol in (nb.NB_FP64, nb.NB_FP32, nb.NB_MIXED):
        b = m.rhs(pol, nb.NB_RHS_UNIFORM, seed=0)
        bm = m.rhs(pol, nb.NB_RHS_MANUFACTURED, noise=1e-3, seed=0)
        w = m.ax(b, pol)
        wl = m.ax(bm, pol, local=True)
        for order in (nb.NB_GS_CONSISTENT, nb.NB_GS_PER_COPY):
            m.dssum(wl, pol, order)
            x, r = m.cg(b, pol, max_iter=6, rtol=0.0, gs_order=order)
    nb.nb_export_maps(m.h)
    nb.nb_export_geom(m.h)
    m.close()
torch.cuda.synchronize()
print("sanitize workload done")
