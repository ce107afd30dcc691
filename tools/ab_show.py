#!/usr/bin/env python3
"""Condensed view of sweep.py logs: python tools/ab_show.py gpurun_out/abe_*.log"""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        ex = " ".join(f"{k}={d[k]:.1f}" for k in ("ax_us", "dssum_us") if k in d)
        print(f"{f.split('/')[-1]:28s} {d['case']:14s} {d['policy']:6s} it={d['us_per_iter']:8.1f} A={d['phaseA_us']:8.1f} "
              f"S={d['phaseS_us']:7.1f} B={d['phaseB_us']:8.1f} {ex}")
