#!/usr/bin/env python3
"""Write profiles/ncu_traffic.json (DRAM bytes per CG iteration of the solve megakernel) and a
text summary from an ncu --set full capture of one configs[1] solve.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep --policy mixed --iterations 587 --tag r1
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--policy", default="mixed")
ap.add_argument("--iterations", type=int, required=True)
ap.add_argument("--tag", default="r1")
a = ap.parse_args()
rows = [d for d in ncu_summary.rows(a.rep) if "k_cg_mega" in d["kernel"]]
d = rows[0]
tr = d["dram_rd"] + d["dram_wr"]
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
js = {}
if os.path.exists(path):
    js = json.load(open(path))
js[f"{a.policy}_configs1_dram_bytes_per_iteration"] = tr / a.iterations
js[f"{a.policy}_configs1_source"] = f"{os.path.basename(a.rep)}: {d['kernel']}, {d['us']:.1f} us, {a.iterations} iterations"
json.dump(js, open(path, "w"), indent=1)
print(json.dumps(js, indent=1))
