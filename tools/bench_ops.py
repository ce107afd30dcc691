#!/usr/bin/env python3
"""Standalone nb_ax (local) / nb_dssum timing (the metric's "Ax/dssum HBM GB/s"), algorithmic
bytes per SURVEY.md §8(d): Ax u + 6 g -> w; dssum f_sh (2 s_v + 4) + f_g 4 (copies + CSR indices).

    python tools/bench_ops.py --cases 32x32x32p9d 50x50x50p7 --policies mixed fp64 [--reps 20]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_02134_b200 as nb  # noqa: E402

SV = {0: 8, 1: 4, 2: 4}
POL = {"fp64": 0, "fp32": 1, "mixed": 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", nargs="+", default=["32x32x32p9d"])
    ap.add_argument("--policies", nargs="+", default=["mixed", "fp64"])
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    peak = 6545.3
    try:
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for c in a.cases:
        d = 0.1 if c.endswith("d") else 0.0
        dims, p = c.rstrip("d").split("p")
        m = nb.Mesh(*[int(v) for v in dims.split("x")], int(p), deform=d)
        info = m.info
        for name in a.policies:
            pol = POL[name]
            u = m.rhs(pol, seed=3)
            w = m.empty(pol)
            out = {"case": c, "policy": name, "n_local": m.n_local}
            for what in ("ax", "dssum"):
                fn = (lambda: nb.nb_ax(m.h, pol, u, w, nb.NB_AX_LOCAL)) if what == "ax" else \
                     (lambda: nb.nb_dssum(m.h, pol, nb.NB_GS_CONSISTENT, w))
                fn()
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    fn()
                    e1.record(st)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                us = 1e3 * statistics.median(ts)
                byts = 8 * SV[pol] * m.n_local if what == "ax" else \
                    info.n_shared_copies * (2 * SV[pol] + 4) + (info.n_shared_global + 1) * 4
                out[what + "_us"] = us
                out[what + "_GBps"] = byts / (us * 1e-6) / 1e9
                out[what + "_frac"] = out[what + "_GBps"] / peak
            print(json.dumps(out), flush=True)
        m.close()


if __name__ == "__main__":
    main()
