"""Compare sweep logs of A/B library variants: python tools/ab_table.py gpurun_out/r2/ab1 prev nb"""
import json
import sys
from collections import defaultdict

pre, vs = sys.argv[1], sys.argv[2:]
res = defaultdict(lambda: defaultdict(list))
for v in vs:
    for rep in (1, 2, 3):
        try:
            for ln in open(f"{pre}_{rep}_{v}.log"):
                if ln.startswith("{"):
                    d = json.loads(ln)
                    res[(d["case"], d["policy"])][v].append((d["us_per_iter"], d["phaseA_us"], d["phaseB_us"],
                                                             d.get("A_GBps"), d.get("B_GBps")))
        except FileNotFoundError:
            pass
print(f"{'case':16s} {'pol':6s} " + " ".join(f"{v + ' it/A/B us':>28s}" for v in vs) + "   B GB/s")
for k, d in res.items():
    row = []
    for v in vs:
        if d[v]:
            it = min(x[0] for x in d[v]); a = min(x[1] for x in d[v]); b = min(x[2] for x in d[v])
            row.append(f"{it:9.1f}/{a:8.1f}/{b:8.1f}")
        else:
            row.append(" " * 28)
    bg = " ".join(f"{max(x[4] for x in d[v]):7.0f}" for v in vs if d[v])
    print(f"{k[0]:16s} {k[1]:6s} " + " ".join(row) + "   " + bg)
