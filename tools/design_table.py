#!/usr/bin/env python3
"""Markdown rows of DESIGN.md §6.0's roofline table from a bench.py JSON line
(`hbm_roofline_point`: configs[2], event-timed launch, globaltimer phase split, ncu DRAM bytes).

    python tools/design_table.py profiles/r2_bench_v8.jsonl
"""
import json
import sys

PEAK = 6545.0
NLOC = 32768000
PHASE_BYTES = {"mixed": (48, 24), "fp64": (96, 40)}


def main():
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    h = d["hbm_roofline_point"]["policies"]
    for pol in ("mixed", "fp64"):
        r = h[pol]
        impl = r["impl_bytes_per_dof_iter"]
        dram = r["ncu_dram_bytes_per_iteration"]
        print(f"| whole solve | {pol} | {r['launch_ms']:.1f} ms | {r['survey_bytes_per_dof_iter']:.1f} | "
              f"{r['achieved_GBps']:.0f} GB/s | **{r['achieved_GBps'] / PEAK:.3f}** | {impl} | "
              f"{r['achieved_impl_GBps'] / PEAK:.3f} | {dram / 1e9:.2f} GB ({dram / (impl * NLOC):.2f}× impl) | "
              f"{r['ncu_dram_GBps_at_this_launch_time']:.0f} (**{r['ncu_dram_GBps_at_this_launch_time'] / PEAK:.3f}**) |")
        for ph, b in zip("AB", PHASE_BYTES[pol]):
            us = r[f"phase{ph}_us"]
            dr = r[f"ncu_phase{ph}_dram_bytes_per_iteration"]
            print(f"| phase {ph} | {pol} | {us:.0f} µs/it | — | — | — | {b} | {r[f'phase{ph}_frac']:.3f} | "
                  f"{dr / 1e9:.2f} GB ({dr / (b * NLOC):.2f}×) | {dr / us / 1e3:.0f} ({r[f'ncu_phase{ph}_dram_frac']:.3f}) |")


if __name__ == "__main__":
    main()
